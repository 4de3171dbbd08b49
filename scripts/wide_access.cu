// Study: do 256-bit accesses (LDG.256 / STG.256, sm_100) move cfg2 rows
// faster than the 128-bit words k_words uses? Gather (pack) and scatter
// (unpack) of K cfg2 objects (E0 x E1 x E2 in a 1024^3-byte allocation per
// object), one L2 flush before every timed kernel, CUDA events around the
// kernel alone. Prints one JSON line per (E0, direction, W, U).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wide_access wide_access.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>

struct alignas(32) W32 {
  uint4 a, b;
};

template <int W> struct Acc;
template <> struct Acc<16> {
  using T = uint4;
  static __device__ __forceinline__ T ld(const void *p) {
    T v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
  }
  static __device__ __forceinline__ void st(void *p, const T &v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
};
template <> struct Acc<32> {
  using T = W32;
  static __device__ __forceinline__ T ld(const void *p) {
    T v;
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.a.x), "=r"(v.a.y), "=r"(v.a.z), "=r"(v.a.w), "=r"(v.b.x), "=r"(v.b.y), "=r"(v.b.z),
                   "=r"(v.b.w)
                 : "l"(p));
    return v;
  }
  static __device__ __forceinline__ void st(void *p, const T &v) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.a.x), "r"(v.a.y), "r"(v.a.z),
                 "r"(v.a.w), "r"(v.b.x), "r"(v.b.y), "r"(v.b.z), "r"(v.b.w)
                 : "memory");
  }
};

struct G {
  uint32_t wpr_sh;  // log2(words per row)
  uint32_t e1_sh;   // log2(rows per plane)
  uint32_t obj_sh;  // log2(rows per object)
  uint32_t words;
};

// every cfg2 dimension is a power of two: shifts, no division
__device__ __forceinline__ int64_t strided_off(uint32_t q, const G &g, int W) {
  const uint32_t row = q >> g.wpr_sh;
  const uint32_t col = q & ((1u << g.wpr_sh) - 1);
  const uint32_t obj = row >> g.obj_sh;
  const uint32_t r = row & ((1u << g.obj_sh) - 1);
  const uint32_t plane = r >> g.e1_sh, rr = r & ((1u << g.e1_sh) - 1);
  return (static_cast<int64_t>(obj) << 30) + (static_cast<int64_t>(plane) << 20) + (rr << 10) + col * W;
}

template <int W, int U, bool PACK>
__global__ void __launch_bounds__(256) k(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, G g) {
  using A = Acc<W>;
  typename A::T v[U];
  const uint32_t step = gridDim.x * 256 * U;
  for (uint32_t base = blockIdx.x * 256 * U + threadIdx.x; base < g.words; base += step) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = base + u * 256;
      if (q < g.words) v[u] = A::ld(in + (PACK ? strided_off(q, g, W) : static_cast<int64_t>(q) * W));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = base + u * 256;
      if (q < g.words) A::st(out + (PACK ? static_cast<int64_t>(q) * W : strided_off(q, g, W)), v[u]);
    }
  }
}

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));           \
      std::exit(1);                                                           \
    }                                                                         \
  } while (0)

__global__ void k_fill(uint8_t *p, size_t n, int v) {
  for (size_t i = blockIdx.x * 256ull + threadIdx.x; i < n / 16; i += gridDim.x * 256ull)
    reinterpret_cast<uint4 *>(p)[i] = make_uint4(v, v, v, v);
}

// read the flush buffer back so the timed kernel starts on a cold CLEAN L2
// (no dirty lines of the flush left to write back inside the timed region)
__global__ void k_read(const uint8_t *p, size_t n, unsigned *sink) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * 256ull + threadIdx.x; i < n / 16; i += gridDim.x * 256ull) {
    const uint4 v = reinterpret_cast<const uint4 *>(p)[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void k_iota(uint8_t *p, size_t n) {
  for (size_t i = blockIdx.x * 256ull + threadIdx.x; i < n / 4; i += gridDim.x * 256ull)
    reinterpret_cast<uint32_t *>(p)[i] = static_cast<uint32_t>(i * 2654435761u);
}

template <int W, int U, bool PACK>
float run(const uint8_t *in, uint8_t *out, G g, uint8_t *flush, size_t flush_n, int reps) {
  int occ = 0, sms = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<W, U, PACK>, 256, 0));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t blocks = (g.words + 256 * U - 1) / (256 * U);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(blocks, static_cast<uint64_t>(sms) * occ));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  std::vector<float> ts;
  for (int i = 0; i < reps + 2; ++i) {
    k_fill<<<sms * 8, 256>>>(flush, flush_n, i);
    k_read<<<sms * 8, 256>>>(flush, flush_n, reinterpret_cast<unsigned *>(flush));
    CK(cudaEventRecord(a));
    k<W, U, PACK><<<grid, 256>>>(in, out, g);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (i >= 2) ts.push_back(ms);
  }
  CK(cudaGetLastError());
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main(int argc, char **argv) {
  const int K = argc > 1 ? std::atoi(argv[1]) : 64;
  const int reps = 7;
  uint8_t *strided = nullptr, *packed = nullptr, *packed2 = nullptr, *flush = nullptr;
  const size_t flush_n = size_t{512} << 20;
  CK(cudaMalloc(&strided, static_cast<size_t>(K) << 30));
  CK(cudaMalloc(&packed, static_cast<size_t>(K) << 20));
  CK(cudaMalloc(&packed2, static_cast<size_t>(K) << 20));
  CK(cudaMalloc(&flush, flush_n));
  k_iota<<<1184, 256>>>(strided, static_cast<size_t>(K) << 30);
  CK(cudaDeviceSynchronize());
  for (int e0 : {32, 64, 128, 256, 512}) {
    // cfg2 dims: E2 = 2^ceil(log2(2^20/E0)/2), E1 = 2^20 / (E0 E2)
    int lg = 0;
    while ((1 << lg) < (1 << 20) / e0) ++lg;
    const int e2 = 1 << ((lg + 1) / 2), e1 = (1 << 20) / (e0 * e2);
    const double bytes = 2.0 * K * (1 << 20);
    auto line = [&](const char *dir, int w, int u, float ms) {
      std::printf("{\"E0\": %d, \"dir\": \"%s\", \"W\": %d, \"U\": %d, \"us\": %.2f, \"GBps\": %.1f}\n", e0, dir, w, u,
                  ms * 1e3, bytes / (ms * 1e-3) / 1e9);
      std::fflush(stdout);
    };
    for (int w : {16, 32}) {
      if (e0 % w) continue;
      auto lg2 = [](uint32_t v) { return static_cast<uint32_t>(__builtin_ctz(v)); };
      G g{lg2(e0 / w), lg2(e1), lg2(e1 * e2), static_cast<uint32_t>(static_cast<uint64_t>(K) * (1 << 20) / w)};
      if (w == 16) {
        line("pack", 16, 4, run<16, 4, true>(strided, packed, g, flush, flush_n, reps));
        line("pack", 16, 8, run<16, 8, true>(strided, packed, g, flush, flush_n, reps));
        line("unpack", 16, 4, run<16, 4, false>(packed, strided, g, flush, flush_n, reps));
      } else {
        line("pack", 32, 2, run<32, 2, true>(strided, packed2, g, flush, flush_n, reps));
        line("pack", 32, 4, run<32, 4, true>(strided, packed2, g, flush, flush_n, reps));
        line("unpack", 32, 2, run<32, 2, false>(packed2, strided, g, flush, flush_n, reps));
        line("unpack", 32, 4, run<32, 4, false>(packed2, strided, g, flush, flush_n, reps));
      }
    }
    // the two word sizes packed the same bytes
    std::vector<uint8_t> h1(1 << 20), h2(1 << 20);
    CK(cudaMemcpy(h1.data(), packed + (static_cast<size_t>(K - 1) << 20), 1 << 20, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), packed2 + (static_cast<size_t>(K - 1) << 20), 1 << 20, cudaMemcpyDeviceToHost));
    if (e0 % 32 == 0 && h1 != h2) std::printf("{\"E0\": %d, \"error\": \"W=32 pack differs from W=16\"}\n", e0);
  }
  return 0;
}
