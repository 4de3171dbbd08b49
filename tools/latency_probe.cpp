// tools/latency_probe.cpp -- host-side cost of the pieces of a small
// message on this node (median of 2000 calls each): the CUDA runtime calls
// the engine makes per message, an sp_pack of a small type, and a complete
// self-send (sp_rt_isend + sp_rt_irecv + waits) for each method.
//   latency_probe            (one B200; prints one line per probe)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "stridepack_b200.h"

template <class F> static double med_us(F &&f, int reps = 2000) {
  for (int i = 0; i < 50; ++i) f();
  std::vector<double> t;
  for (int i = 0; i < reps; ++i) {
    const auto a = std::chrono::steady_clock::now();
    f();
    t.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count());
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

__global__ void k_empty() {}

#define CK(x)                                                                                                  \
  do {                                                                                                         \
    if ((x) != 0) {                                                                                            \
      std::printf("%s failed: %s\n", #x, sp_last_error());                                                     \
      return 1;                                                                                                \
    }                                                                                                          \
  } while (0)

int main() {
  cudaSetDevice(0);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  uint8_t *d = nullptr, *d2 = nullptr;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&d2, 1 << 20);
  cudaPointerAttributes at{};
  std::printf("cudaPointerGetAttributes   %8.2f us\n", med_us([&] { cudaPointerGetAttributes(&at, d + 64); }));
  cudaIpcMemHandle_t h;
  std::printf("cudaIpcGetMemHandle        %8.2f us\n", med_us([&] { cudaIpcGetMemHandle(&h, d); }));
  int ndev = 0;
  std::printf("cudaGetDeviceCount         %8.2f us\n", med_us([&] { cudaGetDeviceCount(&ndev); }));
  std::printf("launch empty (enqueue)     %8.2f us\n", med_us([&] { k_empty<<<1, 32, 0, s>>>(); }));
  cudaStreamSynchronize(s);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  std::printf("launch empty + sync        %8.2f us\n", med_us([&] {
                k_empty<<<1, 32, 0, s>>>();
                cudaStreamSynchronize(s);
              }));
  std::printf("launch + event poll        %8.2f us\n", med_us([&] {
                k_empty<<<1, 32, 0, s>>>();
                cudaEventRecord(ev, s);
                while (cudaEventQuery(ev) == cudaErrorNotReady) {
                }
              }));
  sp_type byte, row, t;
  CK(sp_type_named(SP_BYTE, &byte));
  CK(sp_type_contiguous(64, byte, &row));
  CK(sp_type_hvector(16, 1, 1024, row, &t)); // 1 KiB of 64-B rows
  CK(sp_type_commit(t));
  int64_t pos = 0;
  std::printf("sp_pack 1 KiB (enqueue)    %8.2f us\n", med_us([&] {
                pos = 0;
                sp_pack(d, 1 << 20, t, 1, d2, 1 << 20, &pos, s);
              }));
  cudaStreamSynchronize(s);
  std::printf("sp_pack 1 KiB + sync       %8.2f us\n", med_us([&] {
                pos = 0;
                sp_pack(d, 1 << 20, t, 1, d2, 1 << 20, &pos, s);
                cudaStreamSynchronize(s);
              }));
  // enqueue cost of batch launches: the job table travels as a kernel
  // parameter (k_batchp), ~224 B per job
  for (int nj : {1, 8, 26}) {
    std::vector<sp_copy_job> jobs;
    for (int i = 0; i < nj; ++i) jobs.push_back(sp_copy_job{d, uint64_t{1} << 20, t, 1, d2 + 1024 * i, (uint64_t{1} << 20) - 1024 * uint64_t(i), t, 1});
    sp_batch b = nullptr;
    CK(sp_copy_batch_create(jobs.data(), nj, &b));
    std::printf("copy batch %2d jobs enqueue %8.2f us\n", nj, med_us([&] { sp_batch_execute(b, s); }));
    cudaStreamSynchronize(s);
    std::printf("copy batch %2d jobs + sync %8.2f us\n", nj, med_us([&] {
                  sp_batch_execute(b, s);
                  cudaStreamSynchronize(s);
                }));
    sp_batch_free(b);
  }
  CK(sp_rt_init(0, 1, "latprobe", 0, 8 << 20, 8 << 20));
  for (int m : {SP_METHOD_DIRECT, SP_METHOD_DEVICE, SP_METHOD_ONESHOT, SP_METHOD_STAGED}) {
    int tag = 0;
    const double us = med_us(
        [&] {
          sp_request r, q;
          sp_rt_irecv(d2, 1 << 20, 1, t, 0, tag, &r);
          sp_rt_isend(d, 1 << 20, 1, t, 0, tag, m, &q);
          sp_rt_wait(q, nullptr);
          sp_rt_wait(r, nullptr);
          ++tag;
        },
        500);
    std::printf("self send 1 KiB method %d   %8.2f us\n", m, us);
  }
  // the 1x1x1 halo through MPI_Neighbor_alltoallw (26 region types on the
  // padded 260^3 x 32 B allocation, every neighbour is this rank) against
  // the same 26 typed copies as a prebuilt batch: the difference is the
  // collective's host-side cost per call
  {
    sp_halo_config hc{{1, 1, 1}, {256, 256, 256}, 2, 32};
    sp_type hs[26], hr[26];
    int dir[78];
    int64_t cells[26];
    CK(sp_halo_types(&hc, hs, hr, dir, cells));
    const uint64_t pad = uint64_t{260} * 260 * 260 * 32;
    uint8_t *a = nullptr;
    cudaMalloc(&a, pad);
    cudaMemset(a, 0, pad);
    int64_t one[26], zero[26];
    int nb[26];
    sp_type rtyp[26];
    std::vector<sp_copy_job> jobs;
    for (int k = 0; k < 26; ++k) {
      one[k] = 1;
      zero[k] = 0;
      nb[k] = 0;
      rtyp[k] = hr[25 - k];
      jobs.push_back(sp_copy_job{a, pad, hs[k], 1, a, pad, hr[25 - k], 1});
    }
    sp_batch b = nullptr;
    CK(sp_copy_batch_create(jobs.data(), 26, &b));
    std::printf("halo copy batch + sync     %8.2f us\n", med_us(
                                                              [&] {
                                                                sp_batch_execute(b, s);
                                                                cudaStreamSynchronize(s);
                                                              },
                                                              500));
    auto call = [&] {
      sp_rt_neighbor_alltoallw(a, one, zero, hs, 26, nb, a, one, zero, rtyp, 26, nb);
    };
    std::printf("halo alltoallw (1 rank)    %8.2f us\n", med_us(call, 500));
    // the distributed plan's DIRECT exchange, enqueue only (a time loop's
    // host cost per iteration), against enqueueing the same 26 typed copies
    {
      sp_halo_plan plan = nullptr;
      CK(sp_halo_plan_create(&hc, a, SP_HALO_DIRECT, &plan));
      void *rs = nullptr;
      CK(sp_rt_stream(&rs));
      std::printf("halo plan exchange enqueue %8.2f us\n",
                  med_us([&] { sp_halo_plan_exchange(plan, nullptr); }, 300));
      cudaStreamSynchronize(static_cast<cudaStream_t>(rs));
      std::printf("halo copy batch enqueue    %8.2f us\n", med_us([&] { sp_batch_execute(b, s); }, 300));
      cudaStreamSynchronize(s);
      sp_halo_plan_free(plan);
    }
    // the same two with a cold L2 (a 512 MiB memset before each call, waited
    // for and not timed), as bench.py measures them; and the kernel alone
    // by events, so host cost = wall - kernel
    {
      uint8_t *fl = nullptr;
      cudaMalloc(&fl, size_t{512} << 20);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto cold_med = [&](auto &&f, int reps) {
        std::vector<double> t;
        for (int i = 0; i < reps + 5; ++i) {
          cudaMemsetAsync(fl, i & 0xff, size_t{512} << 20, s);
          cudaStreamSynchronize(s);
          const auto t0 = std::chrono::steady_clock::now();
          f();
          const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
          if (i >= 5) t.push_back(us);
        }
        std::sort(t.begin(), t.end());
        return t[t.size() / 2];
      };
      std::printf("cold: copy batch + sync    %8.2f us\n", cold_med([&] {
                    sp_batch_execute(b, s);
                    cudaStreamSynchronize(s);
                  }, 100));
      std::vector<double> kt;
      for (int i = 0; i < 105; ++i) {
        cudaMemsetAsync(fl, i & 0xff, size_t{512} << 20, s);
        cudaEventRecord(e0, s);
        sp_batch_execute(b, s);
        cudaEventRecord(e1, s);
        cudaStreamSynchronize(s);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 5) kt.push_back(ms * 1e3);
      }
      std::sort(kt.begin(), kt.end());
      std::printf("cold: copy batch (events)  %8.2f us\n", kt[kt.size() / 2]);
      std::printf("cold: alltoallw (1 rank)   %8.2f us\n", cold_med(call, 100));
      cudaFree(fl);
    }
    sp_batch_free(b);
    // host side only: the same call with every count zero launches no copy
    std::printf("alltoallw, zero counts     %8.2f us\n", med_us(
                                                              [&] {
                                                                sp_rt_neighbor_alltoallw(a, zero, zero, hs, 26, nb, a,
                                                                                         zero, zero, rtyp, 26, nb);
                                                              },
                                                              500));
    cudaFree(a);
  }
  CK(sp_rt_finalize());
  return 0;
}
