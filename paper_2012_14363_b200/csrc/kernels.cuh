// kernels.cuh -- device helpers and host launch helpers shared by the
// single-object kernels (pack.cu) and the batch / typed-copy kernels
// (batch.cu). Internal to the engine.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <vector>

#include "core.hpp"

namespace spb {

// ------------------------------------------------------------ fast divmod
// Granlund-Montgomery round-up division for runtime-invariant divisors.
struct FastDiv {
  uint32_t d = 1, m = 1, s1 = 0, s2 = 0;
};

inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  int l = 0;
  while ((uint64_t{1} << l) < d) ++l;
  f.m = static_cast<uint32_t>(((uint64_t{1} << 32) * ((uint64_t{1} << l) - d)) / d + 1);
  f.s1 = l > 0 ? 1 : 0;
  f.s2 = l > 0 ? l - 1 : 0;
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
  const uint32_t t = __umulhi(f.m, n);
  return (t + ((n - t) >> f.s1)) >> f.s2;
}

// ------------------------------------------------------------ geometry
constexpr int KMAX = 12; // row dims a kernel carries (incl. the object dim)

struct Geom {
  int nd;             // row dims
  uint32_t wpr;       // words per row (c0 / W)
  FastDiv wdiv;       // divides by wpr
  uint32_t cnt[KMAX]; // row-dim counts, dim 0 fastest
  FastDiv div[KMAX];
  int64_t str[KMAX];  // row-dim byte strides on the strided side
  int64_t back[KMAX]; // cnt[k]*str[k], for carry-increment walks
  uint64_t total;     // work items (words, or 16-B chunks for smallrow)
  uint64_t rows;      // total rows
  // smallrow only: packed-side 16-byte grid
  uint64_t head;      // bytes before the first 16-B aligned packed address
};

// strided-side byte offset of row r (r < rows)
__device__ __forceinline__ int64_t row_offset(uint32_t r, const Geom &g) {
  int64_t off = 0;
#pragma unroll 1
  for (int k = 0; k < g.nd - 1; ++k) {
    const uint32_t q = fdiv(r, g.div[k]);
    off += static_cast<int64_t>(r - q * g.cnt[k]) * g.str[k];
    r = q;
  }
  if (g.nd > 0) off += static_cast<int64_t>(r) * g.str[g.nd - 1];
  return off;
}

template <int W> struct Word;
template <> struct Word<1> { using T = uint8_t; };
template <> struct Word<2> { using T = uint16_t; };
template <> struct Word<4> { using T = uint32_t; };
template <> struct Word<8> { using T = uint2; };
template <> struct Word<16> { using T = uint4; };

// streaming loads/stores: every byte is touched once, keep it out of L1
template <class T> __device__ __forceinline__ T ld_stream(const T *p) { return __ldcs(p); }
template <> __device__ __forceinline__ uint8_t ld_stream(const uint8_t *p) {
  return static_cast<uint8_t>(__ldcs(reinterpret_cast<const char *>(p)));
}
template <> __device__ __forceinline__ uint16_t ld_stream(const uint16_t *p) {
  return static_cast<uint16_t>(__ldcs(reinterpret_cast<const unsigned short *>(p)));
}
template <class T> __device__ __forceinline__ void st_stream(T *p, T v) { __stcs(p, v); }
template <> __device__ __forceinline__ void st_stream(uint8_t *p, uint8_t v) {
  __stcs(reinterpret_cast<char *>(p), static_cast<char>(v));
}
template <> __device__ __forceinline__ void st_stream(uint16_t *p, uint16_t v) {
  __stcs(reinterpret_cast<unsigned short *>(p), static_cast<unsigned short>(v));
}


// ------------------------------------------------------------ host helpers
extern std::atomic<int64_t> g_launches; // kernels launched by this process (sp_kernel_launch_count)

struct RowDims {
  int64_t c0 = 0;
  std::vector<int64_t> cnt, str; // dim 0 fastest
};
// Row geometry of `count` objects; contiguous-in-row-order dims merged.
RowDims row_dims(const Committed &ct, int64_t count);
// largest power of two <= 16 dividing v
int pow2_align(uint64_t v);

enum class MemKind { Device, Pinned, Pageable };
struct Resolved {
  MemKind kind;
  uint8_t *dptr; // device-accessible address (for Device/Pinned)
};
Resolved resolve(const void *p);
int sm_count();
// grid cap for kernels touching pinned host memory (set by execute())
extern thread_local unsigned t_host_grid_cap;
constexpr unsigned kHostGridCap = 48;

} // namespace spb
