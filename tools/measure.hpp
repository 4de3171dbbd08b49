// tools/measure.hpp -- B200 machine-profile measurement shared by
// tools/measure_profile (standalone) and `stridepack profile-gen`
// (tools/stridepack_cli.cpp). See measure_profile.cpp for what is measured.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "stridepack_b200.h"

#define CK(x)                                                                                          \
  do {                                                                                                 \
    if ((x) != 0) {                                                                                    \
      std::fprintf(stderr, "%s failed: %s\n", #x, sp_last_error());                                    \
      std::exit(1);                                                                                    \
    }                                                                                                  \
  } while (0)

template <class F> inline double median_s(F &&f, int reps) {
  for (int i = 0; i < 3; ++i) f();
  std::vector<double> t;
  for (int i = 0; i < reps; ++i) {
    const auto a = std::chrono::steady_clock::now();
    f();
    t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

// measures every curve and surface on device 0 and writes `out_path`;
// returns 0, or 1 when the file cannot be written
inline int measure_profile(const char *out_path, int reps, bool report) {
  std::vector<int64_t> objects, blocks = {1, 4, 16, 64, 256, 1024, 4096}, sizes;
  for (int k = 10; k <= 26; k += 2) objects.push_back(int64_t{1} << k);
  for (int k = 0; k <= 20; ++k) sizes.push_back(int64_t{64} << k);
  const int64_t big = objects.back();
  cudaSetDevice(0);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  uint8_t *src, *packed, *hpacked, *dev, *dev2, *h1, *h2, *peer = nullptr;
  cudaMalloc(&src, 2 * big);
  cudaMemset(src, 3, 2 * big);
  cudaMalloc(&packed, big);
  cudaHostAlloc(&hpacked, big, cudaHostAllocMapped | cudaHostAllocPortable);
  const int64_t maxn = sizes.back();
  cudaMalloc(&dev, maxn);
  cudaMalloc(&dev2, maxn);
  cudaHostAlloc(&h1, maxn, cudaHostAllocPortable);
  cudaHostAlloc(&h2, maxn, cudaHostAllocPortable);
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  if (ndev > 1) {
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, 0, 1);
    cudaSetDevice(1);
    cudaMalloc(&peer, maxn);
    cudaSetDevice(0);
    if (ok) cudaDeviceEnablePeerAccess(1, 0);
  }
  sp_type byte;
  CK(sp_type_named(SP_BYTE, &byte));
  sp_profile prof;
  CK(sp_profile_create(&prof));
  std::vector<double> ox(objects.begin(), objects.end()), bx(blocks.begin(), blocks.end());
  for (int surf = 0; surf < 4; ++surf) {
    const bool to_host = surf >= 2, unpack = surf % 2 == 1;
    std::vector<double> t;
    for (int64_t o : objects)
      for (int64_t b0 : blocks) {
        const int64_t b = std::min(b0, o);
        sp_type row, t2;
        CK(sp_type_contiguous(b, byte, &row));
        CK(sp_type_hvector(o / b, 1, 2 * b, row, &t2));
        CK(sp_type_commit(t2));
        uint8_t *pk = to_host ? hpacked : packed;
        t.push_back(median_s(
            [&] {
              int64_t pos = 0;
              if (unpack) {
                CK(sp_unpack(pk, big, &pos, t2, 1, src, 2 * big, s));
              } else {
                CK(sp_pack(src, 2 * big, t2, 1, pk, big, &pos, s));
              }
              cudaStreamSynchronize(s);
            },
            reps));
        sp_type_free(row);
        sp_type_free(t2);
      }
    CK(sp_profile_set_surface(prof, surf, ox.data(), ox.size(), bx.data(), bx.size(), t.data()));
  }
  // B200 extension: the DIRECT method's one typed-copy launch, probe layout
  // -> the same layout in another buffer on this GPU (gpu_direct) and in a
  // buffer on device 1 over NVLink (gpu_direct_peer, when visible)
  uint8_t *dst_local = nullptr, *dst_peer = nullptr;
  cudaMalloc(&dst_local, 2 * big);
  if (peer) {
    cudaSetDevice(1);
    cudaMalloc(&dst_peer, 2 * big);
    cudaSetDevice(0);
  }
  for (int surf : {SP_SURF_GPU_DIRECT, SP_SURF_GPU_DIRECT_PEER}) {
    uint8_t *dst = surf == SP_SURF_GPU_DIRECT ? dst_local : dst_peer;
    if (!dst) continue;
    std::vector<double> t;
    for (int64_t o : objects)
      for (int64_t b0 : blocks) {
        const int64_t b = std::min(b0, o);
        sp_type row, t2;
        CK(sp_type_contiguous(b, byte, &row));
        CK(sp_type_hvector(o / b, 1, 2 * b, row, &t2));
        CK(sp_type_commit(t2));
        const sp_copy_job job{src, static_cast<uint64_t>(2 * big), t2, 1, dst, static_cast<uint64_t>(2 * big), t2, 1};
        t.push_back(median_s(
            [&] {
              CK(sp_copy(&job, s));
              cudaStreamSynchronize(s);
            },
            reps));
        sp_type_free(row);
        sp_type_free(t2);
      }
    CK(sp_profile_set_surface(prof, surf, ox.data(), ox.size(), bx.data(), bx.size(), t.data()));
  }
  std::vector<double> sx(sizes.begin(), sizes.end());
  auto curve = [&](int which, auto &&copy) {
    std::vector<double> t;
    for (int64_t n : sizes) t.push_back(median_s([&] { copy(n); }, reps));
    CK(sp_profile_set_curve(prof, which, sx.data(), t.data(), static_cast<int64_t>(t.size())));
  };
  curve(SP_CURVE_D2H, [&](int64_t n) {
    cudaMemcpyAsync(h1, dev, n, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  });
  curve(SP_CURVE_H2D, [&](int64_t n) {
    cudaMemcpyAsync(dev, h1, n, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
  });
  curve(SP_CURVE_GPU_GPU, [&](int64_t n) {
    if (peer) {
      cudaMemcpyPeerAsync(peer, 1, dev, 0, n, s);
    } else {
      cudaMemcpyAsync(dev2, dev, n, cudaMemcpyDeviceToDevice, s);
    }
    cudaStreamSynchronize(s);
  });
  curve(SP_CURVE_CPU_CPU, [&](int64_t n) { std::memcpy(h2, h1, static_cast<size_t>(n)); });
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, 0);
  const std::string header =
      std::string("B200 machine profile measured by tools/measure_profile on ") + prop.name +
      "\nsurfaces: median wall time of synchronous sp_pack/sp_unpack (enqueue + completion)," +
      " probe hvector(o/b,1,2b,contiguous(b,BYTE))\n" +
      (peer ? "gpu_gpu: cudaMemcpyPeerAsync device 0 -> 1\n" : "gpu_gpu: same-device copy (one GPU visible)\n") +
      "cpu_cpu: pinned host memcpy; d2h/h2d: cudaMemcpyAsync pinned\n" +
      "gpu_direct: synchronous sp_copy probe layout -> same layout, same GPU (the DIRECT method, B200 extension)" +
      (peer ? "\ngpu_direct_peer: the same copy into device 1 over NVLink" : "");
  int64_t len = 0;
  CK(sp_profile_save(prof, header.c_str(), nullptr, 0, &len));
  std::string text(static_cast<size_t>(len) + 1, '\0');
  CK(sp_profile_save(prof, header.c_str(), text.data(), len + 1, &len));
  FILE *f = std::fopen(out_path, "w");
  if (!f) return 1;
  std::fwrite(text.data(), 1, static_cast<size_t>(len), f);
  std::fclose(f);
  if (!report) return 0;
  const int64_t q[][2] = {{1 << 10, 16}, {1 << 16, 8}, {1 << 20, 64}, {4 << 20, 16}, {64 << 20, 4096}};
  const char *names[4] = {"oneshot", "device", "staged", "direct"};
  for (auto &qq : q) {
    int m = -1, m4 = -1;
    double t4[4];
    CK(sp_choose_method(prof, qq[0], qq[1], &m));
    CK(sp_choose_method_b200(prof, qq[0], qq[1], 1, &m4, t4));
    std::printf("object %lld block %lld -> %s (b200, same GPU: %s)  device %.3e oneshot %.3e staged %.3e direct %.3e\n",
                (long long)qq[0], (long long)qq[1], names[m], names[m4], t4[0], t4[1], t4[2], t4[3]);
  }
  return 0;
}
