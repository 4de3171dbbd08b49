// Microbenchmark: the E0=1 unpack store pattern (one byte per 1 KiB row, 64M
// rows over 64 GiB) with different lane -> row mappings and store flavours,
// to see whether the DRAM read-modify-write rate depends on the order.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scatter_order scripts/scatter_order.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// M=0: lane owns 16 consecutive rows (k_smallrow today: row = 16*t + j)
// M=1: warp owns 512 rows, lane l writes rows base + 32*j + l
// M=2: block owns 4096 rows, thread writes rows base + 256*j + tid
template <int M, int F>
__global__ void scatter(const uint4 *__restrict__ packed, uint8_t *__restrict__ out, uint64_t pitch, uint32_t nchunks) {
  const uint32_t step = gridDim.x * blockDim.x;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nchunks; t += step) {
    const uint4 v = __ldcs(packed + t);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint64_t row0;
    uint32_t rstep;
    if (M == 0) {
      row0 = uint64_t(t) * 16;
      rstep = 1;
    } else if (M == 1) {
      const uint32_t lane = t & 31, warp = t >> 5;
      row0 = uint64_t(warp) * 512 + lane;
      rstep = 32;
    } else {
      const uint32_t tid = t & 255, blk = t >> 8;
      row0 = uint64_t(blk) * 4096 + tid;
      rstep = 256;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      uint8_t *p = out + (row0 + uint64_t(j) * rstep) * pitch;
      const uint8_t b = uint8_t(w[j >> 2] >> ((j & 3) * 8));
      if (F == 0) {
        __stcs(reinterpret_cast<char *>(p), char(b));
      } else {
        *p = b;
      }
    }
  }
}

// the E0 = 1 PACK pattern: 16 one-byte loads at 1 KiB pitch -> one 16-B store
__global__ void gather(const uint8_t *__restrict__ in, uint4 *__restrict__ packed, uint64_t pitch, uint32_t nchunks) {
  const uint32_t step = gridDim.x * blockDim.x;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nchunks; t += step) {
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint8_t b = uint8_t(__ldcs(reinterpret_cast<const char *>(in + (uint64_t(t) * 16 + j) * pitch)));
      w[j >> 2] |= uint32_t(b) << ((j & 3) * 8);
    }
    __stcs(packed + t, make_uint4(w[0], w[1], w[2], w[3]));
  }
}

template <int M, int F> float run(const uint4 *pk, uint8_t *out, uint64_t pitch, uint32_t nchunks, uint8_t *flush) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cudaMemset(flush, r, 512u << 20);
    cudaEventRecord(a);
    scatter<M, F><<<148 * 8, 256>>>(pk, out, pitch, nchunks);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const uint64_t pitch = 1024, rows = uint64_t(64) << 20; // 64M rows: 64 GiB
  const uint32_t nchunks = uint32_t(rows / 16);
  uint8_t *out, *flush;
  uint4 *pk;
  if (cudaMalloc(&out, rows * pitch) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&pk, rows);
  cudaMalloc(&flush, 512u << 20);
  cudaMemset(pk, 7, rows);
  const double bytes = 2.0 * rows; // algorithmic: packed read + described bytes written
  printf("M0 stcs %.1f GB/s\n", bytes / run<0, 0>(pk, out, pitch, nchunks, flush) / 1e6);
  printf("M0 st   %.1f GB/s\n", bytes / run<0, 1>(pk, out, pitch, nchunks, flush) / 1e6);
  printf("M1 stcs %.1f GB/s\n", bytes / run<1, 0>(pk, out, pitch, nchunks, flush) / 1e6);
  printf("M1 st   %.1f GB/s\n", bytes / run<1, 1>(pk, out, pitch, nchunks, flush) / 1e6);
  printf("M2 stcs %.1f GB/s\n", bytes / run<2, 0>(pk, out, pitch, nchunks, flush) / 1e6);
  printf("M2 st   %.1f GB/s\n", bytes / run<2, 1>(pk, out, pitch, nchunks, flush) / 1e6);
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaMemset(flush, r, 512u << 20);
      cudaEventRecord(a);
      gather<<<148 * 8, 256>>>(out, pk, pitch, nchunks);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("gather (pack pattern) %.1f GB/s\n", bytes / best / 1e6);
  }
  return 0;
}
