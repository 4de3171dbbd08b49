// acceptance.cpp criterion 8 through the product C-ABI: 10000 random
// queries, best of five, cold = sp_choose_method, warm = sp_model_cache_choose.
// Prints "<cold_s> <warm_s> <agree>".
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include "stridepack_b200.h"

int main(int argc, char **argv) {
  sp_profile p = nullptr;
  if (argc < 2 || sp_profile_load(argv[1], &p) != SP_OK) return 2;
  sp_model_cache c = nullptr;
  sp_model_cache_create(p, &c);
  std::mt19937_64 rng(0x8badf00d);
  std::vector<std::pair<int64_t, int64_t>> q;
  for (int i = 0; i < 10000; ++i) {
    const int64_t o = 1 + static_cast<int64_t>(rng() % (4 << 20));
    q.emplace_back(o, 1 + static_cast<int64_t>(rng() % o));
  }
  int agree = 1;
  for (auto &[o, b] : q) {
    int a = -1, w = -2;
    sp_choose_method(p, o, b, &a);
    sp_model_cache_choose(c, o, b, &w);
    agree &= a == w;
  }
  double cold = 1e9, warm = 1e9;
  volatile int sink = 0;
  for (int rep = 0; rep < 5; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    for (auto &[o, b] : q) {
      int m;
      sp_choose_method(p, o, b, &m);
      sink = sink + m;
    }
    auto t1 = std::chrono::steady_clock::now();
    for (auto &[o, b] : q) {
      int m;
      sp_model_cache_choose(c, o, b, &m);
      sink = sink + m;
    }
    auto t2 = std::chrono::steady_clock::now();
    cold = std::min(cold, std::chrono::duration<double>(t1 - t0).count());
    warm = std::min(warm, std::chrono::duration<double>(t2 - t1).count());
  }
  std::printf("%.9f %.9f %d\n", cold, warm, agree);
  sp_model_cache_free(c);
  sp_profile_free(p);
  return 0;
}
