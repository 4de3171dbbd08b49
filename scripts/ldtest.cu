// Microbenchmark: gather ROW-byte rows at PITCH-byte pitch with different
// global-load flavors, to find which one fetches only the touched sectors.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldtest scripts/ldtest.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int F> __device__ __forceinline__ uint2 ld8(const uint2 *p) {
  uint2 r;
  if (F == 0) { r = *p; }
  else if (F == 1) { r = __ldcs(p); }
  else if (F == 2) { r = __ldcg(p); }
  else if (F == 3) { r = __ldg(p); }
  else if (F == 4) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else if (F == 5) {
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else if (F == 6) {
    asm volatile("ld.global.cg.L2::64B.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else if (F == 7) {
    asm volatile("ld.global.cv.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else if (F == 8) {
    asm volatile("ld.relaxed.gpu.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  }
  return r;
}

// each thread: 2 rows of 8 B -> one 16 B store
template <int F> __global__ void gather8(const uint8_t *src, uint4 *dst, uint32_t nrows, uint32_t pitch) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t step = gridDim.x * blockDim.x;
  for (; 2 * t < nrows; t += step) {
    uint2 a = ld8<F>(reinterpret_cast<const uint2 *>(src + (uint64_t)(2 * t) * pitch));
    uint2 b = ld8<F>(reinterpret_cast<const uint2 *>(src + (uint64_t)(2 * t + 1) * pitch));
    dst[t] = make_uint4(a.x, a.y, b.x, b.y);
  }
}

template <int F> float run(const uint8_t *src, uint4 *dst, uint32_t nrows, uint32_t pitch, uint8_t *flush, size_t fl) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaMemsetAsync(flush, r, fl);
    cudaEventRecord(a);
    gather8<F><<<148 * 8, 256>>>(src, dst, nrows, pitch);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const uint32_t pitch = 1024, nrows = 1u << 22; // 4M rows x 8 B = 32 MiB
  uint8_t *src, *flush;
  uint4 *dst;
  cudaMalloc(&src, (size_t)nrows * pitch);
  cudaMalloc(&dst, (size_t)nrows * 8);
  size_t fl = 512ull << 20;
  cudaMalloc(&flush, fl);
  const char *names[] = {"plain", "ldcs", "ldcg", "ldg(nc)", "nc.L1::no_allocate", "L1::no_allocate",
                         "cg.L2::64B", "cv", "relaxed.gpu"};
  float t[9];
  t[0] = run<0>(src, dst, nrows, pitch, flush, fl);
  t[1] = run<1>(src, dst, nrows, pitch, flush, fl);
  t[2] = run<2>(src, dst, nrows, pitch, flush, fl);
  t[3] = run<3>(src, dst, nrows, pitch, flush, fl);
  t[4] = run<4>(src, dst, nrows, pitch, flush, fl);
  t[5] = run<5>(src, dst, nrows, pitch, flush, fl);
  t[6] = run<6>(src, dst, nrows, pitch, flush, fl);
  t[7] = run<7>(src, dst, nrows, pitch, flush, fl);
  t[8] = run<8>(src, dst, nrows, pitch, flush, fl);
  for (int i = 0; i < 9; ++i)
    printf("%-22s %8.1f us  %7.1f GB/s algorithmic\n", names[i], t[i] * 1e3, 2.0 * nrows * 8 / (t[i] * 1e-3) / 1e9);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
