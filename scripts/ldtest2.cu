// Microbenchmark 2: scattered-row gather under different L2 fetch
// granularities (cudaLimitMaxL2FetchGranularity) and pitches.
//   each thread loads two ROW-byte rows (ROW in {8,32}) at PITCH and stores
//   them contiguously; reports event time and GB/s of algorithmic bytes.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int ROW> struct V;
template <> struct V<8> { using T = uint2; };
template <> struct V<16> { using T = uint4; };

template <int ROW>
__global__ void gather(const uint8_t *src, uint8_t *dst, uint32_t nrows, uint32_t pitch) {
  using T = typename V<ROW>::T;
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x, step = gridDim.x * blockDim.x;
  for (; 2 * t < nrows; t += step) {
    T a = *reinterpret_cast<const T *>(src + (uint64_t)(2 * t) * pitch);
    T b = *reinterpret_cast<const T *>(src + (uint64_t)(2 * t + 1) * pitch);
    reinterpret_cast<T *>(dst)[2 * t] = a;
    reinterpret_cast<T *>(dst)[2 * t + 1] = b;
  }
}

template <int ROW>
float run(const uint8_t *src, uint8_t *dst, uint32_t nrows, uint32_t pitch, uint8_t *flush, size_t fl) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaMemsetAsync(flush, r, fl);
    cudaEventRecord(a);
    gather<ROW><<<148 * 8, 256>>>(src, dst, nrows, pitch);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  uint8_t *src, *dst, *flush;
  size_t fl = 512ull << 20;
  cudaMalloc(&src, 17ull << 30);
  cudaMalloc(&dst, 64ull << 20);
  cudaMalloc(&flush, fl);
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
  printf("default cudaLimitMaxL2FetchGranularity = %zu\n", cur);
  for (int gran : {32, 64, 128, 0}) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
    printf("--- granularity set %d -> %zu (%s)\n", gran, cur, cudaGetErrorString(e));
    for (uint32_t pitch : {32u, 64u, 128u, 256u, 1024u, 4096u}) {
      const uint32_t n8 = 4u << 20;  // 4M rows of 8 B
      const uint32_t n16 = 2u << 20; // 2M rows of 16 B
      float t8 = run<8>(src, dst, n8, pitch, flush, fl);
      float t16 = pitch >= 16 ? run<16>(src, dst, n16, pitch, flush, fl) : 0;
      printf("pitch %5u: 8B rows %7.1f us (%6.1f Grows/s, %6.1f GB/s)   16B rows %7.1f us (%6.1f Grows/s, %6.1f GB/s)\n",
             pitch, t8 * 1e3, n8 / (t8 * 1e-3) / 1e9, 2.0 * n8 * 8 / (t8 * 1e-3) / 1e9, t16 * 1e3,
             n16 / (t16 * 1e-3) / 1e9, 2.0 * n16 * 16 / (t16 * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
