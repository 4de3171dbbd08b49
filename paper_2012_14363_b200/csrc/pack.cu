// pack.cu -- sm_100a pack/unpack kernels and their launcher.
//
// The reference executes a committed StridedBlock on the host
// (pack.hpp:47-60 walk_words: object-major, dimension 1 fastest, one
// memcpy of `word` bytes at a time). On B200 the same byte order is produced
// by kernels that see the object as ROWS of c0 = counts[0] bytes:
//
//   packed[pos + R*c0 + b] = strided[start + sum_k i_k * str_k + b]
//
// where R enumerates the row multi-index (i_0 fastest) and the object count
// is just one more row dimension with stride = extent. Row dimensions that
// are contiguous in row order are merged on the host, so a kernel only ever
// walks the irreducible geometry.
//
// Kernels:
//   k_words<W,PACK>    one W-byte word per work item; consecutive lanes own
//                      consecutive packed words, so the packed side is fully
//                      coalesced and the strided side is coalesced within a
//                      row. Index math is fast-divmod (mul-hi), no division.
//   k_smallrow<C0,PACK> rows of 1/2/4/8 bytes: each lane assembles 16/C0
//                      rows into one 16-byte packed word (one STG.128 per
//                      lane, or one LDG.128 for unpack) and walks the rows by
//                      carry-increment instead of re-dividing.
//   k_blocklist<PACK>  definition-order run table on the device, for forms
//                      without a strided canon (zero-stride "Unsupported"
//                      types) or with more row dims than a kernel carries.
// W is the largest power of two <= 16 dividing the row length, every row
// stride, and BOTH buffer addresses (the reference's select_word_size,
// plan.hpp:47-64, plus the address alignment a GPU load needs).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "core.hpp"
#include "tma.hpp"

namespace spb {

static std::atomic<int64_t> g_launches{0};
static thread_local sp_launch_info t_last{};

void set_last_launch(const sp_launch_info &li) { t_last = li; }

void cuda_check(int err, const char *what) {
  const cudaError_t e = static_cast<cudaError_t>(err);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(SP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(SP_ERR_NO_DEVICE, "no CUDA device: the B200 kernels are the only execution path");
  }
}

// ------------------------------------------------------------ fast divmod
// Granlund-Montgomery round-up division for runtime-invariant divisors.
struct FastDiv {
  uint32_t d = 1, m = 1, s1 = 0, s2 = 0;
};

static FastDiv make_fastdiv(uint32_t d) {
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

// ------------------------------------------------------------ k_words
// strided: base of the strided side (already offset by start)
// packed:  base of the packed side (already offset by position)
template <int W, bool PACK, int U>
__global__ void __launch_bounds__(256) k_words(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                               const Geom g) {
  using T = typename Word<W>::T;
  const uint32_t total = static_cast<uint32_t>(g.total);
  const uint32_t step = gridDim.x * blockDim.x * U;
  for (uint32_t base = blockIdx.x * blockDim.x * U + threadIdx.x; base < total; base += step) {
    T v[U];
    int64_t soff[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = base + u * blockDim.x;
      if (q < total) {
        const uint32_t row = fdiv(q, g.wdiv);
        const uint32_t col = q - row * g.wpr;
        soff[u] = row_offset(row, g) + static_cast<int64_t>(col) * W;
        if (PACK) {
          v[u] = ld_stream(reinterpret_cast<const T *>(in + soff[u]));
        } else {
          v[u] = ld_stream(reinterpret_cast<const T *>(in) + q);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = base + u * blockDim.x;
      if (q < total) {
        if (PACK) {
          st_stream(reinterpret_cast<T *>(out) + q, v[u]);
        } else {
          st_stream(reinterpret_cast<T *>(out + soff[u]), v[u]);
        }
      }
    }
  }
}

// 64-bit fallback for > 4 Gi words or > 4 Gi rows (plain division; rare)
template <int W, bool PACK>
__global__ void __launch_bounds__(256) k_words64(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                 const Geom g, const uint64_t *cnt64) {
  using T = typename Word<W>::T;
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < g.total; q += step) {
    uint64_t row = q / g.wpr;
    const uint64_t col = q - row * g.wpr;
    int64_t off = static_cast<int64_t>(col) * W;
    for (int k = 0; k < g.nd; ++k) {
      const uint64_t c = cnt64[k];
      const uint64_t i = (k == g.nd - 1) ? row : row % c;
      off += static_cast<int64_t>(i) * g.str[k];
      row = (k == g.nd - 1) ? 0 : row / c;
    }
    if (PACK) {
      st_stream(reinterpret_cast<T *>(out) + q, ld_stream(reinterpret_cast<const T *>(in + off)));
    } else {
      st_stream(reinterpret_cast<T *>(out + off), ld_stream(reinterpret_cast<const T *>(in) + q));
    }
  }
}

// ------------------------------------------------------------ k_smallrow
// Packed side seen as 16-byte aligned chunks; chunk t covers packed bytes
// [16t - head, 16t - head + 16). Rows are C0 bytes and C0-aligned on both
// sides, so a row never straddles a chunk. Interior chunks move with one
// 16-byte access on the packed side; the (at most two) edge chunks fall back
// to per-row C0-byte accesses.
template <int C0, bool PACK>
__global__ void __launch_bounds__(256) k_smallrow(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                  const Geom g) {
  using T = typename Word<C0>::T;
  constexpr int R = 16 / C0;
  const uint32_t nchunks = static_cast<uint32_t>(g.total);
  const uint32_t rows = static_cast<uint32_t>(g.rows);
  const uint32_t head_rows = static_cast<uint32_t>(g.head / C0);
  const uint32_t step = gridDim.x * blockDim.x;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nchunks; t += step) {
    // rows [r0, r1) live in this chunk
    const int64_t first = static_cast<int64_t>(t) * R - head_rows;
    const uint32_t r0 = first < 0 ? 0u : static_cast<uint32_t>(first);
    const int64_t lastrow = first + R < static_cast<int64_t>(rows) ? first + R : static_cast<int64_t>(rows);
    const uint32_t r1 = static_cast<uint32_t>(lastrow);
    if (r0 >= r1) continue;
    // decompose r0 once, then carry-increment
    uint32_t idx[KMAX];
    int64_t off = 0;
    {
      uint32_t r = r0;
      for (int k = 0; k < g.nd - 1; ++k) {
        const uint32_t q = fdiv(r, g.div[k]);
        idx[k] = r - q * g.cnt[k];
        off += static_cast<int64_t>(idx[k]) * g.str[k];
        r = q;
      }
      if (g.nd > 0) {
        idx[g.nd - 1] = r;
        off += static_cast<int64_t>(r) * g.str[g.nd - 1];
      }
    }
    auto advance = [&]() {
      for (int k = 0; k < g.nd; ++k) {
        off += g.str[k];
        if (++idx[k] < g.cnt[k] || k == g.nd - 1) return;
        idx[k] = 0;
        off -= g.back[k];
      }
    };
    const bool full = (first >= 0) && (r1 - r0 == R);
    if (full) {
      union {
        uint4 v;
        T e[R];
      } buf;
      if (PACK) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          buf.e[j] = ld_stream(reinterpret_cast<const T *>(in + off));
          if (j + 1 < R) advance();
        }
        st_stream(reinterpret_cast<uint4 *>(out + static_cast<int64_t>(r0) * C0), buf.v);
      } else {
        buf.v = ld_stream(reinterpret_cast<const uint4 *>(in + static_cast<int64_t>(r0) * C0));
#pragma unroll
        for (int j = 0; j < R; ++j) {
          st_stream(reinterpret_cast<T *>(out + off), buf.e[j]);
          if (j + 1 < R) advance();
        }
      }
    } else {
      for (uint32_t r = r0; r < r1; ++r) {
        if (PACK) {
          st_stream(reinterpret_cast<T *>(out + static_cast<int64_t>(r) * C0),
                    ld_stream(reinterpret_cast<const T *>(in + off)));
        } else {
          st_stream(reinterpret_cast<T *>(out + off),
                    ld_stream(reinterpret_cast<const T *>(in + static_cast<int64_t>(r) * C0)));
        }
        if (r + 1 < r1) advance();
      }
    }
  }
}

// ------------------------------------------------------------ k_shift
// Rows (c0 >= 16 B) whose strided-side addresses or strides are not word
// aligned (e.g. a subarray starting at byte 3) would force W = 1 in k_words.
// The shift kernels keep 16-B accesses by aligning the work to the 16-B grid
// of the side that is WRITTEN and funnel-shifting what is read:
//   k_shift_pack   : lane = one aligned 16-B packed chunk (touches <= 2 rows,
//                    since c0 >= 16), built from the aligned source blocks
//                    that hold its bytes -> one STG.128;
//   k_shift_unpack : lane = one aligned 16-B block of a destination row
//                    (ceil(c0/16)+1 slots per row, empty ones skip), read
//                    from the packed blocks that hold its bytes -> one
//                    STG.128 inside the row, masked u32/u8 stores at its ends.
// Only aligned blocks that contain described bytes are loaded or stored, so
// no access leaves the blocks the layout touches.
// Auto-selection, from scripts/shift_bench.py on B200 (profiles/r01_shift_bench.json):
//   pack  : 4.0-5.1 TB/s against 1.26 (W=1) and 3.6-4.4 (W=4, c0 % 16 == 0);
//           at W=4 with c0 % 16 != 0 the word kernel stays ahead;
//   unpack: 1.6-2.5 TB/s against 1.33 (W=1) for c0 >= 128; shorter rows lose
//           to W=1 because the row-end partial blocks become per-lane
//           scattered sub-word stores.
// below this the LDG/STG kernel wins the TMA unpack (1 MiB single objects:
// 6.1 vs 8.1 us, bench.py single_object); the sweep's 64 MiB calls keep TMA
constexpr uint64_t kTmaMinBytes = uint64_t{8} << 20;

static bool shift_wins(bool pack, int w, int64_t c0) {
  if (pack) return w <= 2 || (w == 4 && c0 % 16 == 0);
  return w <= 2 && c0 >= 128;
}

// the 16 bytes starting at (window), of which only [lo, hi) are meaningful;
// aligned 16-B blocks not intersecting [lo, hi) are never read
__device__ __forceinline__ uint4 load_window(const uint8_t *window, const uint8_t *lo, const uint8_t *hi) {
  const uintptr_t w = reinterpret_cast<uintptr_t>(window);
  const uintptr_t b0 = w & ~uintptr_t{15}, b1 = b0 + 16;
  const uintptr_t l = reinterpret_cast<uintptr_t>(lo), h = reinterpret_cast<uintptr_t>(hi);
  uint4 x0 = make_uint4(0, 0, 0, 0), x1 = make_uint4(0, 0, 0, 0);
  if (l < b0 + 16 && h > b0) x0 = ld_stream(reinterpret_cast<const uint4 *>(b0));
  const unsigned d = static_cast<unsigned>(w & 15);
  if (d && l < b1 + 16 && h > b1) x1 = ld_stream(reinterpret_cast<const uint4 *>(b1));
  const uint32_t W[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
  const unsigned q = d >> 2, sh = (d & 3) * 8;
  uint32_t v[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) { // v[k] = W[k + q], selects instead of local memory
    const uint32_t a = k + 0 < 8 ? W[k] : 0, b = k + 1 < 8 ? W[k + 1] : 0;
    const uint32_t c = k + 2 < 8 ? W[k + 2] : 0, e = k + 3 < 8 ? W[k + 3] : 0;
    v[k] = q == 0 ? a : q == 1 ? b : q == 2 ? c : e;
  }
  return make_uint4(__funnelshift_r(v[0], v[1], sh), __funnelshift_r(v[1], v[2], sh),
                    __funnelshift_r(v[2], v[3], sh), __funnelshift_r(v[3], v[4], sh));
}

__device__ __forceinline__ uint4 merge_bytes(uint4 a, uint4 b, unsigned n) { // bytes [0,n) of a, rest of b
  uint32_t r[4];
  const uint32_t A[4] = {a.x, a.y, a.z, a.w}, B[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int lo = static_cast<int>(n) - 4 * k; // bytes of word k taken from a
    const uint32_t m = lo >= 4 ? 0xffffffffu : lo <= 0 ? 0u : (0xffffffffu >> (32 - 8 * lo));
    r[k] = (A[k] & m) | (B[k] & ~m);
  }
  return make_uint4(r[0], r[1], r[2], r[3]);
}

// bytes [lo, hi) of the aligned 16-B block at blk: whole u32 words where
// covered, single bytes at the two ends
__device__ __forceinline__ void store_masked(uint8_t *blk, uint4 z, unsigned lo, unsigned hi) {
  const uint32_t Z[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
  for (unsigned i = 0; i < 4; ++i) {
    if (lo <= 4 * i && 4 * i + 4 <= hi) {
      st_stream(reinterpret_cast<uint32_t *>(blk) + i, Z[i]);
    } else {
#pragma unroll
      for (unsigned b = 0; b < 4; ++b) {
        const unsigned k = 4 * i + b;
        if (lo <= k && k < hi) st_stream(blk + k, static_cast<uint8_t>(Z[i] >> (8 * b)));
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_shift_pack(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                    const Geom g, uint32_t c0, FastDiv c0div) {
  const uint32_t nchunks = static_cast<uint32_t>(g.total);
  const uint64_t T = g.rows * c0;
  const uint32_t step = gridDim.x * blockDim.x;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nchunks; t += step) {
    const int64_t lo = static_cast<int64_t>(t) * 16 - static_cast<int64_t>(g.head);
    if (lo >= 0 && static_cast<uint64_t>(lo) + 16 <= T) {
      const uint32_t p = static_cast<uint32_t>(lo);
      const uint32_t r = fdiv(p, c0div), col = p - r * c0;
      const unsigned n1 = min(16u, c0 - col);
      const uint8_t *a = in + row_offset(r, g) + col;
      uint4 v = load_window(a, a, a + n1);
      if (n1 < 16) { // the chunk continues at the start of row r + 1
        const uint8_t *b = in + row_offset(r + 1, g);
        v = merge_bytes(v, load_window(b - n1, b, b + (16 - n1)), n1);
      }
      st_stream(reinterpret_cast<uint4 *>(out + p), v);
    } else { // first / last chunk: byte by byte over its valid range
      const int64_t b0 = lo < 0 ? 0 : lo;
      const int64_t b1 = static_cast<int64_t>(T) < lo + 16 ? static_cast<int64_t>(T) : lo + 16;
      for (int64_t p = b0; p < b1; ++p) {
        const uint32_t pp = static_cast<uint32_t>(p);
        const uint32_t r = fdiv(pp, c0div), col = pp - r * c0;
        out[p] = in[row_offset(r, g) + col];
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_shift_unpack(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                      const Geom g, uint32_t c0, uint32_t slots, FastDiv sdiv) {
  const uint32_t nitems = static_cast<uint32_t>(g.total);
  const uint32_t step = gridDim.x * blockDim.x;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nitems; t += step) {
    const uint32_t r = fdiv(t, sdiv), j = t - r * slots;
    const uintptr_t A = reinterpret_cast<uintptr_t>(out + row_offset(r, g)); // row start
    const uintptr_t B = (A & ~uintptr_t{15}) + 16 * uintptr_t{j};           // this lane's block
    const uintptr_t vlo = B > A ? B : A, vhi = B + 16 < A + c0 ? B + 16 : A + c0;
    if (vlo >= vhi) continue;
    const uint8_t *P = in + static_cast<uint64_t>(r) * c0; // packed row start
    const uint4 z = load_window(P + static_cast<intptr_t>(B - A), P + (vlo - A), P + (vhi - A));
    uint8_t *blk = reinterpret_cast<uint8_t *>(B);
    const unsigned lo = static_cast<unsigned>(vlo - B), hi = static_cast<unsigned>(vhi - B);
    if (lo == 0 && hi == 16) {
      st_stream(reinterpret_cast<uint4 *>(blk), z);
    } else {
      store_masked(blk, z, lo, hi);
    }
  }
}

// ------------------------------------------------------------ k_blocklist
// One thread per (object, run): byte loop over the run. Used only for
// definition-order gathers (Unsupported forms, pack.hpp:123-135) and for
// strided forms with more row dimensions than KMAX.
template <bool PACK>
__global__ void __launch_bounds__(256) k_blocklist(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                   const int64_t *__restrict__ rsrc,
                                                   const int64_t *__restrict__ rdst,
                                                   const int64_t *__restrict__ rlen, int64_t nruns,
                                                   int64_t nobj, int64_t extent, int64_t size) {
  const int64_t total = nruns * nobj;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += step) {
    const int64_t j = t / nruns, k = t - j * nruns;
    const int64_t so = j * extent + rsrc[k], po = j * size + rdst[k], n = rlen[k];
    for (int64_t b = 0; b < n; ++b) {
      if (PACK) {
        out[po + b] = in[so + b];
      } else {
        out[so + b] = in[po + b];
      }
    }
  }
}

// ============================================================ host side

Committed::~Committed() {
  if (dev.d_src) {
    int cur = -1;
    cudaGetDevice(&cur);
    if (dev.device >= 0) cudaSetDevice(dev.device);
    cudaFree(dev.d_src);
    cudaFree(dev.d_dst);
    cudaFree(dev.d_len);
    if (cur >= 0) cudaSetDevice(cur);
  }
}

namespace {

struct RowDims {
  int64_t c0 = 0;
  std::vector<int64_t> cnt, str; // dim 0 fastest
};

// Row geometry of `count` objects; contiguous-in-row-order dims merged.
RowDims row_dims(const Committed &ct, int64_t count) {
  RowDims r;
  const StridedBlock &sb = ct.sb;
  r.c0 = sb.counts[0];
  std::vector<std::pair<int64_t, int64_t>> dims;
  for (int d = 1; d < sb.ndims(); ++d) dims.emplace_back(sb.counts[d], sb.strides[d]);
  dims.emplace_back(count, ct.extent);
  for (auto &[c, s] : dims) {
    if (c == 1) continue;
    if (r.cnt.empty() && s == r.c0) { // rows abut: one longer row
      r.c0 *= c;
      continue;
    }
    if (!r.cnt.empty() && s == r.cnt.back() * r.str.back()) {
      r.cnt.back() *= c;
      continue;
    }
    r.cnt.push_back(c);
    r.str.push_back(s);
  }
  return r;
}

int pow2_align(uint64_t v) {
  int w = 16;
  while (w > 1 && (v % static_cast<uint64_t>(w))) w >>= 1;
  return w;
}

enum class MemKind { Device, Pinned, Pageable };

struct Resolved {
  MemKind kind;
  uint8_t *dptr; // device-accessible address (for Device/Pinned)
};

Resolved resolve(const void *p) {
  cudaPointerAttributes at{};
  const cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return {MemKind::Pageable, nullptr};
  }
  switch (at.type) {
  case cudaMemoryTypeDevice:
  case cudaMemoryTypeManaged:
    return {MemKind::Device, static_cast<uint8_t *>(const_cast<void *>(p))};
  case cudaMemoryTypeHost:
    return {MemKind::Pinned, static_cast<uint8_t *>(at.devicePointer)};
  default:
    return {MemKind::Pageable, nullptr};
  }
}

int sm_count() {
  static thread_local int dev = -1, sms = 148;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) {
    dev = cur;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// Kernels that read or write pinned host memory are PCIe-bound (~55 GB/s
// per direction): a few CTAs keep enough bytes in flight, and leaving the
// other SMs free lets an inbound and an outbound transfer run concurrently
// (PCIe is full duplex). Set by execute() for the duration of one launch.
thread_local unsigned t_host_grid_cap = 0;
constexpr unsigned kHostGridCap = 48;
constexpr int64_t kDmaStageMin = int64_t{1} << 20; // pinned packed messages >= 1 MiB move by DMA

// Persistent per-(device, stream) staging buffers for DMA'd messages. Work
// on one stream is ordered, so reuse by the next call on that stream is
// safe; a pool allocation freed on one stream and reused on another would
// make the stream-ordered allocator insert a cross-stream dependency and
// serialise the inbound and outbound legs of a pipelined exchange.
uint8_t *stage_buffer(cudaStream_t s, size_t bytes) {
  struct Stage {
    uint8_t *p = nullptr;
    size_t n = 0;
  };
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, Stage> stages;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  Stage &st = stages[{dev, s}];
  if (st.n < bytes) {
    if (st.p) cuda_check(cudaFreeAsync(st.p, s), "cudaFreeAsync(stage)");
    const size_t n = std::max(bytes, st.n * 2);
    cuda_check(cudaMallocAsync(reinterpret_cast<void **>(&st.p), n, s), "cudaMallocAsync(stage)");
    st.n = n;
  }
  return st.p;
}

unsigned grid_for(uint64_t items, int per_thread) {
  const uint64_t blocks = (items + 256ull * per_thread - 1) / (256ull * per_thread);
  uint64_t cap = static_cast<uint64_t>(sm_count()) * 8; // 8 x 256 = 2048 threads/SM
  if (t_host_grid_cap) cap = std::min<uint64_t>(cap, t_host_grid_cap);
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(blocks, cap)));
}

template <int W, bool PACK>
void launch_words(const uint8_t *in, uint8_t *out, const Geom &g, cudaStream_t s, sp_launch_info &li) {
  const bool big = g.total >= static_cast<uint64_t>(sm_count()) * 2048 * 4;
  unsigned grid = grid_for(g.total, big ? 4 : 1);
  if (big) {
    k_words<W, PACK, 4><<<grid, 256, 0, s>>>(in, out, g);
  } else {
    k_words<W, PACK, 1><<<grid, 256, 0, s>>>(in, out, g);
  }
  li.grid = grid;
  li.block = 256;
}

template <bool PACK>
void dispatch_words(int w, const uint8_t *in, uint8_t *out, const Geom &g, cudaStream_t s, sp_launch_info &li) {
  switch (w) {
  case 16: launch_words<16, PACK>(in, out, g, s, li); break;
  case 8: launch_words<8, PACK>(in, out, g, s, li); break;
  case 4: launch_words<4, PACK>(in, out, g, s, li); break;
  case 2: launch_words<2, PACK>(in, out, g, s, li); break;
  default: launch_words<1, PACK>(in, out, g, s, li); break;
  }
}

template <bool PACK>
void dispatch_smallrow(int c0, const uint8_t *in, uint8_t *out, const Geom &g, cudaStream_t s,
                       sp_launch_info &li) {
  const unsigned grid = grid_for(g.total, 1);
  switch (c0) {
  case 1: k_smallrow<1, PACK><<<grid, 256, 0, s>>>(in, out, g); break;
  case 2: k_smallrow<2, PACK><<<grid, 256, 0, s>>>(in, out, g); break;
  case 4: k_smallrow<4, PACK><<<grid, 256, 0, s>>>(in, out, g); break;
  default: k_smallrow<8, PACK><<<grid, 256, 0, s>>>(in, out, g); break;
  }
  li.grid = grid;
  li.block = 256;
}

template <bool PACK>
void dispatch_words64(int w, const uint8_t *in, uint8_t *out, const Geom &g, const uint64_t *cnt64,
                      cudaStream_t s, sp_launch_info &li) {
  const unsigned grid = grid_for(g.total, 1);
  switch (w) {
  case 16: k_words64<16, PACK><<<grid, 256, 0, s>>>(in, out, g, cnt64); break;
  case 8: k_words64<8, PACK><<<grid, 256, 0, s>>>(in, out, g, cnt64); break;
  case 4: k_words64<4, PACK><<<grid, 256, 0, s>>>(in, out, g, cnt64); break;
  case 2: k_words64<2, PACK><<<grid, 256, 0, s>>>(in, out, g, cnt64); break;
  default: k_words64<1, PACK><<<grid, 256, 0, s>>>(in, out, g, cnt64); break;
  }
  li.grid = grid;
  li.block = 256;
}

// upload the run table of a committed type to the current device (cached)
const DeviceRuns &device_runs(const Committed &ct, const std::vector<Run> &runs) {
  std::lock_guard<std::mutex> lk(ct.dev_mu);
  int cur = 0;
  cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
  if (ct.dev.d_src && ct.dev.device == cur) return ct.dev;
  if (ct.dev.d_src) {
    cudaFree(ct.dev.d_src);
    cudaFree(ct.dev.d_dst);
    cudaFree(ct.dev.d_len);
    ct.dev = DeviceRuns{};
  }
  const size_t n = runs.size();
  std::vector<int64_t> hs(n), hd(n), hl(n);
  int64_t acc = 0;
  for (size_t k = 0; k < n; ++k) {
    hs[k] = runs[k].off;
    hd[k] = acc;
    hl[k] = runs[k].len;
    acc += runs[k].len;
  }
  DeviceRuns d;
  d.device = cur;
  d.n = static_cast<int64_t>(n);
  const size_t bytes = std::max<size_t>(n, 1) * sizeof(int64_t);
  cuda_check(cudaMalloc(&d.d_src, bytes), "cudaMalloc(runs)");
  cuda_check(cudaMalloc(&d.d_dst, bytes), "cudaMalloc(runs)");
  cuda_check(cudaMalloc(&d.d_len, bytes), "cudaMalloc(runs)");
  cuda_check(cudaMemcpy(d.d_src, hs.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice), "upload runs");
  cuda_check(cudaMemcpy(d.d_dst, hd.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice), "upload runs");
  cuda_check(cudaMemcpy(d.d_len, hl.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice), "upload runs");
  ct.dev = d;
  return ct.dev;
}

// runs of a strided form, for row geometries too deep for the kernels
std::vector<Run> strided_runs(const StridedBlock &sb) {
  std::vector<Run> out;
  std::vector<int64_t> idx(sb.ndims(), 0);
  for (;;) {
    int64_t off = sb.start;
    for (int d = 1; d < sb.ndims(); ++d) off += idx[d] * sb.strides[d];
    out.push_back({off, sb.counts[0]});
    int d = 1;
    while (d < sb.ndims() && ++idx[d] == sb.counts[d]) idx[d++] = 0;
    if (d >= sb.ndims()) break;
  }
  return out;
}

// Launch on device-accessible pointers. strided: object base (no start);
// packed: packed buffer base + position.
void launch(const Committed &ct, int64_t count, const uint8_t *strided_in, uint8_t *strided_out,
            const uint8_t *packed_in, uint8_t *packed_out, bool pack, cudaStream_t s,
            const sp_pack_options &opt, sp_launch_info &li) {
  const uint8_t *in = pack ? strided_in : packed_in;
  uint8_t *out = pack ? packed_out : strided_out;
  const uint64_t strided_addr = reinterpret_cast<uint64_t>(pack ? strided_in : strided_out);
  const uint64_t packed_addr = reinterpret_cast<uint64_t>(pack ? packed_out : packed_in);

  bool blocklist = ct.form != SP_FORM_STRIDED || opt.kernel == SP_KERNEL_BLOCKLIST;
  RowDims rd;
  if (!blocklist) {
    rd = row_dims(ct, count);
    if (static_cast<int>(rd.cnt.size()) > KMAX) blocklist = true;
  }
  if (blocklist) {
    std::vector<Run> tmp;
    const std::vector<Run> *runs = &ct.runs;
    if (ct.form == SP_FORM_STRIDED) {
      tmp = strided_runs(ct.sb);
      runs = &tmp;
    }
    const DeviceRuns &dr = device_runs(ct, *runs);
    const unsigned grid = grid_for(static_cast<uint64_t>(dr.n * count), 1);
    if (pack) {
      k_blocklist<true><<<grid, 256, 0, s>>>(in, out, dr.d_src, dr.d_dst, dr.d_len, dr.n, count, ct.extent,
                                             ct.size);
    } else {
      k_blocklist<false><<<grid, 256, 0, s>>>(in, out, dr.d_src, dr.d_dst, dr.d_len, dr.n, count,
                                              ct.extent, ct.size);
    }
    cuda_check(cudaGetLastError(), "k_blocklist launch");
    li.kernel = SP_KERNEL_BLOCKLIST;
    li.word = 1;
    li.launches = 1;
    li.grid = grid;
    li.block = 256;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return;
  }

  // alignment-derived word
  uint64_t g_or = static_cast<uint64_t>(rd.c0) | (strided_addr + ct.sb.start) | packed_addr;
  for (int64_t st : rd.str) g_or |= static_cast<uint64_t>(st);
  int w = pow2_align(g_or);
  if (opt.force_word) {
    if (opt.force_word > w || (opt.force_word & (opt.force_word - 1)))
      fail(SP_ERR_INVALID_ARGUMENT, "force_word is not legal for these buffers");
    w = opt.force_word;
  }
  // strided side offset by the StridedBlock start
  const uint8_t *sin = pack ? in + ct.sb.start : in;
  uint8_t *sout = pack ? out : out + ct.sb.start;

  uint64_t rows = 1;
  for (int64_t c : rd.cnt) rows *= static_cast<uint64_t>(c);
  const uint64_t total_bytes = rows * static_cast<uint64_t>(rd.c0);

  Geom g{};
  g.nd = static_cast<int>(rd.cnt.size());
  bool fits32 = rows < (1ull << 32) && total_bytes / static_cast<uint64_t>(w) < (1ull << 32);
  for (int k = 0; k < g.nd; ++k) {
    fits32 = fits32 && rd.cnt[k] < (int64_t{1} << 32);
    g.str[k] = rd.str[k];
    g.back[k] = rd.cnt[k] * rd.str[k];
  }
  g.rows = rows;

  const bool smallrow_ok = (rd.c0 == 1 || rd.c0 == 2 || rd.c0 == 4 || rd.c0 == 8) && w >= rd.c0 && fits32;
  int kernel = opt.kernel;
  if (kernel == SP_KERNEL_AUTO) kernel = smallrow_ok && !opt.force_word ? SP_KERNEL_SMALLROW : SP_KERNEL_WORDS;
  if (!fits32 || kernel == SP_KERNEL_WORDS64) {
    fits32 = false;
    kernel = SP_KERNEL_WORDS64;
  }
  if (kernel == SP_KERNEL_SMALLROW && !smallrow_ok) fail(SP_ERR_INVALID_ARGUMENT, "smallrow kernel not applicable");
  // misaligned long rows: the word would be < kShiftBelow only because of
  // addresses / strides, the shift kernel keeps 16-B packed-side accesses
  const bool shift_ok = rd.c0 >= 16 && fits32 && total_bytes < (1ull << 32);
  if (kernel == SP_KERNEL_WORDS && opt.kernel == SP_KERNEL_AUTO && !opt.force_word && shift_ok &&
      shift_wins(pack, w, rd.c0))
    kernel = SP_KERNEL_SHIFT;
  if (kernel == SP_KERNEL_SHIFT && !shift_ok) fail(SP_ERR_INVALID_ARGUMENT, "shift kernel not applicable");
  // unpack of rows >= 64 B: the TMA store path measured 6-9% ahead of the
  // LDG/STG kernel at c0 = 64 and 128 (profiles/r01_tma_vs_words.txt) and
  // ties above; at 32 B it loses; pack ties or loses everywhere
  if (kernel == SP_KERNEL_WORDS && opt.kernel == SP_KERNEL_AUTO && !pack && !opt.force_word && rd.c0 >= 64 &&
      g.nd <= 4 && t_host_grid_cap == 0 /* device memory on both sides */ &&
      total_bytes >= kTmaMinBytes /* the TMA ring's pipeline fill costs ~2 us on a 1 MiB object */) {
    TmaGeometry probe{};
    probe.c0 = rd.c0;
    probe.nd = g.nd;
    for (int k = 0; k < g.nd; ++k) {
      probe.cnt[k] = rd.cnt[k];
      probe.str[k] = rd.str[k];
    }
    probe.strided_addr = strided_addr + ct.sb.start;
    probe.packed_addr = packed_addr;
    if (tma_applicable(probe)) kernel = SP_KERNEL_TMA;
  }
  if (kernel == SP_KERNEL_TMA) {
    TmaGeometry tg{};
    tg.c0 = rd.c0;
    tg.nd = g.nd;
    if (tg.nd > 4) fail(SP_ERR_INVALID_ARGUMENT, "TMA path: more than 4 row dimensions");
    for (int k = 0; k < tg.nd; ++k) {
      tg.cnt[k] = rd.cnt[k];
      tg.str[k] = rd.str[k];
    }
    tg.strided_addr = strided_addr + ct.sb.start;
    tg.packed_addr = packed_addr;
    int64_t grid = 0;
    tma_launch(tg, pack ? sin : sout, pack ? out : const_cast<uint8_t *>(in), pack, s, &grid);
    li.kernel = SP_KERNEL_TMA;
    li.word = 16;
    li.launches = 1;
    li.grid = grid;
    li.block = 32;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return;
  }

  if (fits32) {
    for (int k = 0; k < g.nd; ++k) {
      g.cnt[k] = static_cast<uint32_t>(rd.cnt[k]);
      g.div[k] = make_fastdiv(g.cnt[k]);
    }
  }
  if (kernel == SP_KERNEL_SMALLROW) {
    // packed side on the 16-byte grid: chunk t spans packed offsets
    // [16t - head, 16t - head + 16), head = packed address mod 16
    g.head = packed_addr & 15;
    g.total = (total_bytes + g.head + 15) / 16;
    if (pack) {
      dispatch_smallrow<true>(static_cast<int>(rd.c0), sin, out, g, s, li);
    } else {
      dispatch_smallrow<false>(static_cast<int>(rd.c0), in, sout, g, s, li);
    }
    li.word = rd.c0;
  } else if (kernel == SP_KERNEL_SHIFT) {
    unsigned grid = 0;
    if (pack) { // aligned 16-B packed chunks
      g.head = packed_addr & 15;
      g.total = (total_bytes + g.head + 15) / 16;
      grid = grid_for(g.total, 1);
      k_shift_pack<<<grid, 256, 0, s>>>(sin, out, g, static_cast<uint32_t>(rd.c0),
                                        make_fastdiv(static_cast<uint32_t>(rd.c0)));
    } else { // aligned 16-B destination blocks, ceil(c0/16)+1 slots per row
      const uint32_t slots = static_cast<uint32_t>((rd.c0 + 15) / 16 + 1);
      g.total = rows * slots;
      grid = grid_for(g.total, 1);
      k_shift_unpack<<<grid, 256, 0, s>>>(in, sout, g, static_cast<uint32_t>(rd.c0), slots, make_fastdiv(slots));
    }
    li.grid = grid;
    li.block = 256;
    li.word = 16;
  } else if (fits32) {
    g.wpr = static_cast<uint32_t>(rd.c0 / w);
    g.wdiv = make_fastdiv(g.wpr);
    g.total = total_bytes / static_cast<uint64_t>(w);
    if (pack) {
      dispatch_words<true>(w, sin, out, g, s, li);
    } else {
      dispatch_words<false>(w, in, sout, g, s, li);
    }
    li.word = w;
  } else {
    g.wpr = static_cast<uint32_t>(std::min<int64_t>(rd.c0 / w, 0xffffffff));
    if (rd.c0 / w >= (int64_t{1} << 32)) fail(SP_ERR_UNSUPPORTED, "row longer than 64 GiB words");
    g.total = total_bytes / static_cast<uint64_t>(w);
    uint64_t *cnt64 = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void **>(&cnt64), KMAX * sizeof(uint64_t), s), "cudaMallocAsync");
    uint64_t hc[KMAX] = {0};
    for (int k = 0; k < g.nd; ++k) hc[k] = static_cast<uint64_t>(rd.cnt[k]);
    cuda_check(cudaMemcpyAsync(cnt64, hc, sizeof(hc), cudaMemcpyHostToDevice, s), "cudaMemcpyAsync");
    if (pack) {
      dispatch_words64<true>(w, sin, out, g, cnt64, s, li);
    } else {
      dispatch_words64<false>(w, in, sout, g, cnt64, s, li);
    }
    cuda_check(cudaFreeAsync(cnt64, s), "cudaFreeAsync");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize"); // hc lifetime
    li.word = w;
  }
  cuda_check(cudaGetLastError(), "pack kernel launch");
  li.kernel = kernel;
  li.launches = 1;
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

} // namespace

// ============================================================ batches
// A persistent list of jobs executed by ONE launch per word size. A job is
//   PACK   (type, count, strided src) -> packed dst
//   UNPACK packed src -> (type, count, strided dst)
//   COPY   (type S, count, strided src) -> (type D, count', strided dst),
//          byte k of S's pack order lands on byte k of D's: a typed copy
//          with no packed intermediate (halo ghost writes, alltoallw).
// Destinations may be peer-GPU memory mapped over NVLink (CUDA IPC), which
// turns the batch into a fused pack-to-peer / copy-to-peer.
//
// Work distribution: the words of all jobs form one index space, split into
// equal contiguous ranges, one per CTA of a single resident wave (grid =
// SMs x resident CTAs per SM). Each thread moves U words per round with all
// U loads issued before the first store, so a CTA's whole range is usually
// one or two DRAM round trips and no CTA waits on a straggler chunk. Within
// a round a thread finds its job by walking forward from the CTA's first
// job (ranges rarely cross a job boundary); the job descriptors are read
// through the read-only path and stay L1-resident.
constexpr int kBatchU = 4;                            // words in flight per thread
constexpr uint32_t kBatchChunk = 256 * kBatchU;       // words per unit of work
enum : int { kModeUnpack = 0, kModePack = 1, kModeCopy = 2 };

struct BatchJob {
  Geom gs;           // strided-side geometry of the source (PACK, COPY)
  Geom gd;           // strided-side geometry of the destination (UNPACK, COPY)
  const uint8_t *in; // source base (strided sources already at start)
  uint8_t *out;      // destination base
  uint64_t begin;    // first word of this job in the launch's index space
  uint32_t q0;       // first word of the job's own stream this launch moves
                     // (non-zero for one chunk of a pipelined message)
  int same;          // COPY with gd == gs: destination offset = source offset
};

// Optional in-kernel completion protocol (distributed halo): every block
// first waits until each `wait` flag (local memory, written by peers over
// NVLink) reaches wait_value; after the last word, the LAST block to finish
// publishes signal_value to each `signal` flag (peer memory) with a
// system-scope release store, after fences by every block.
constexpr int kMaxSig = 32;
struct BatchSig {
  const unsigned long long *wait[kMaxSig];
  unsigned long long *signal[kMaxSig];
  unsigned long long wait_value, signal_value;
  unsigned *done; // block-completion counter of this launch (device memory)
  int n_wait, n_signal;
  int sys_scope;  // some destination lives on another GPU: system-scope fences
  // published by block 0 BEFORE waiting (consumer-side "ready" flags: the
  // stream order guarantees everything before this launch has completed)
  unsigned long long *pre[kMaxSig];
  unsigned long long pre_value;
  int n_pre;
  // waited for by the LAST block after it signalled (completion of the
  // peers' writes into this rank's memory folded into the same launch)
  const unsigned long long *post[kMaxSig];
  unsigned long long post_value;
  int n_post;
  // per-target values (neighbour collectives count calls per peer pair);
  // used instead of signal_value / post_value when per_target is set
  unsigned long long signal_vals[kMaxSig], post_vals[kMaxSig];
  int per_target;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// byte offset of word q on a strided side
template <int W> __device__ __forceinline__ int64_t word_offset(uint32_t q, const Geom &g) {
  const uint32_t row = fdiv(q, g.wdiv);
  return row_offset(row, g) + static_cast<int64_t>(q - row * g.wpr) * W;
}

// words of chunk `c` (job-local) of job J: U per thread, all U loads issued
// before the first store; geometry read from J (shared or param memory)
template <int W, int MODE> __device__ __forceinline__ void move_chunk(const BatchJob &J, uint32_t c, uint32_t words) {
  using T = typename Word<W>::T;
  const uint32_t base = c * kBatchChunk + threadIdx.x;
  T v[kBatchU];
  int64_t doff[kBatchU];
#pragma unroll
  for (int u = 0; u < kBatchU; ++u) {
    const uint32_t q = base + u * 256;
    if (q < words) {
      const uint32_t ql = q + J.q0;
      if (MODE == kModeUnpack) {
        v[u] = ld_stream(reinterpret_cast<const T *>(J.in) + ql);
        doff[u] = word_offset<W>(ql, J.gd);
      } else {
        const int64_t so = word_offset<W>(ql, J.gs);
        v[u] = ld_stream(reinterpret_cast<const T *>(J.in + so));
        if (MODE == kModePack) {
          doff[u] = static_cast<int64_t>(ql) * W;
        } else {
          doff[u] = J.same ? so : word_offset<W>(ql, J.gd);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kBatchU; ++u)
    if (base + u * 256 < words) st_stream(reinterpret_cast<T *>(J.out + doff[u]), v[u]);
}

__device__ __forceinline__ void batch_prologue(const BatchSig &sig) {
  if (sig.n_pre && blockIdx.x == 0 && threadIdx.x < static_cast<unsigned>(sig.n_pre))
    st_release_sys(sig.pre[threadIdx.x], sig.pre_value);
  if (sig.n_wait) {
    if (threadIdx.x < static_cast<unsigned>(sig.n_wait))
      while (ld_acquire_sys(sig.wait[threadIdx.x]) < sig.wait_value) __nanosleep(64);
    __syncthreads();
  }
}

__device__ __forceinline__ void batch_epilogue(const BatchSig &sig) {
  if (sig.n_signal || sig.n_post) {
    // bar.sync orders every thread's stores before thread 0 (CTA scope);
    // thread 0's fence is cumulative over them: GPU scope when every
    // destination is on this device, system scope when some were written
    // over NVLink into a peer GPU
    __syncthreads();
    if (threadIdx.x == 0) {
      if (sig.sys_scope) {
        __threadfence_system();
      } else {
        __threadfence();
      }
    }
    __shared__ int last;
    if (threadIdx.x == 0) last = atomicAdd(sig.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
      if (threadIdx.x == 0) {
        __threadfence_system();
        for (int i = 0; i < sig.n_signal; ++i)
          st_release_sys(sig.signal[i], sig.per_target ? sig.signal_vals[i] : sig.signal_value);
        atomicExch(sig.done, 0u); // ready for the next launch on this stream
      }
      // every other block of this launch has finished, so waiting here
      // cannot starve them; the peers publish before they wait, so the
      // ranks' last blocks cannot wait on each other in a cycle
      if (threadIdx.x < static_cast<unsigned>(sig.n_post))
        while (ld_acquire_sys(sig.post[threadIdx.x]) <
               (sig.per_target ? sig.post_vals[threadIdx.x] : sig.post_value))
          __nanosleep(32);
    }
  }
}

__device__ __forceinline__ uint32_t job_words(const BatchJob &J, int mode) {
  return static_cast<uint32_t>(mode == kModeUnpack ? J.gd.total : J.gs.total);
}

// Every chunk (kBatchChunk words of one job) is a unit of work; CTAs walk
// the chunks grid-stride, so each CTA sees chunks of every job (the slow
// 64-B-row regions of a halo spread over the whole grid) and the grid stays
// one resident wave at full occupancy. The chunk's job is found by binary
// search on the jobs' first-chunk indices and staged in shared memory.
template <int W, int MODE>
__global__ void __launch_bounds__(256) k_batch(const BatchJob *__restrict__ jobs, int njobs, uint32_t nchunks,
                                               const BatchSig sig) {
  batch_prologue(sig);
  __shared__ BatchJob sj;
  int loaded = -1;
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    int a = 0, b = njobs - 1;
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (jobs[m].begin <= c) {
        a = m;
      } else {
        b = m - 1;
      }
    }
    if (a != loaded) {
      __syncthreads();
      const uint32_t *src = reinterpret_cast<const uint32_t *>(jobs + a);
      uint32_t *dst = reinterpret_cast<uint32_t *>(&sj);
      for (uint32_t i = threadIdx.x; i < sizeof(BatchJob) / 4; i += blockDim.x) dst[i] = src[i];
      __syncthreads();
      loaded = a;
    }
    move_chunk<W, MODE>(sj, c - static_cast<uint32_t>(sj.begin), job_words(sj, MODE) - sj.q0);
  }
  batch_epilogue(sig);
}

// one job passed by value (param space): a single message or message chunk
// launches without uploading a descriptor; `words` from q0 on
template <int W, int MODE>
__global__ void __launch_bounds__(256) k_job(const __grid_constant__ BatchJob job, uint32_t words) {
  const uint32_t nchunks = (words + kBatchChunk - 1) / kBatchChunk;
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) move_chunk<W, MODE>(job, c, words);
}

// ---- compact job tables in kernel-parameter space
// A batch of up to kParamJobs jobs whose geometries have at most 3 row dims
// (every halo region, every cfg1-cfg4 object) travels by value: the
// chunk -> job search and every descriptor read hit the constant cache, so
// a chunk starts with no dependent global load and no barrier, and word
// offsets are computed from registers.
constexpr int kParamJobs = 32;
struct CGeom {
  uint32_t wpr, c0, c1;
  int32_t nd;
  FastDiv wdiv, d0, d1;
  int64_t s0, s1, s2;
  uint32_t total; // words of the job's stream
  uint32_t pad;
};
struct CJob {
  const uint8_t *in;
  uint8_t *out;
  CGeom gs, gd;
  uint32_t begin; // first chunk
  uint32_t q0;
  int32_t same;
  int32_t pad;
};
struct CTable {
  CJob jobs[kParamJobs];
  int32_t njobs;
  uint32_t nchunks;
};

template <int W> __device__ __forceinline__ int64_t c_offset(uint32_t q, const CGeom &r) {
  const uint32_t row = fdiv(q, r.wdiv);
  int64_t off = static_cast<int64_t>(q - row * r.wpr) * W;
  if (r.nd <= 1) return r.nd == 1 ? off + static_cast<int64_t>(row) * r.s0 : off;
  const uint32_t q1 = fdiv(row, r.d0);
  off += static_cast<int64_t>(row - q1 * r.c0) * r.s0;
  if (r.nd == 2) return off + static_cast<int64_t>(q1) * r.s1;
  const uint32_t q2 = fdiv(q1, r.d1);
  return off + static_cast<int64_t>(q1 - q2 * r.c1) * r.s1 + static_cast<int64_t>(q2) * r.s2;
}

template <int W, int MODE>
__global__ void __launch_bounds__(256) k_batchp(const __grid_constant__ CTable t, const BatchSig sig) {
  using T = typename Word<W>::T;
  batch_prologue(sig);
  for (uint32_t c = blockIdx.x; c < t.nchunks; c += gridDim.x) {
    int a = 0, b = t.njobs - 1;
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (t.jobs[m].begin <= c) {
        a = m;
      } else {
        b = m - 1;
      }
    }
    const CJob &J = t.jobs[a];
    const uint32_t words = (MODE == kModeUnpack ? J.gd.total : J.gs.total) - J.q0;
    const uint32_t base = (c - J.begin) * kBatchChunk + threadIdx.x;
    T v[kBatchU];
    int64_t doff[kBatchU];
#pragma unroll
    for (int u = 0; u < kBatchU; ++u) {
      const uint32_t q = base + u * 256;
      if (q < words) {
        const uint32_t ql = q + J.q0;
        if (MODE == kModeUnpack) {
          v[u] = ld_stream(reinterpret_cast<const T *>(J.in) + ql);
          doff[u] = c_offset<W>(ql, J.gd);
        } else {
          const int64_t so = c_offset<W>(ql, J.gs);
          v[u] = ld_stream(reinterpret_cast<const T *>(J.in + so));
          if (MODE == kModePack) {
            doff[u] = static_cast<int64_t>(ql) * W;
          } else {
            doff[u] = J.same ? so : c_offset<W>(ql, J.gd);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kBatchU; ++u)
      if (base + u * 256 < words) st_stream(reinterpret_cast<T *>(J.out + doff[u]), v[u]);
  }
  batch_epilogue(sig);
}

struct BatchGroup {
  int w = 0, mode = 0;
  BatchJob *d_jobs = nullptr;
  int njobs = 0;
  uint32_t nchunks = 0;
  std::shared_ptr<CTable> table; // set when the jobs fit kernel-parameter space
};

struct Batch {
  int device = -1;
  std::vector<BatchGroup> groups;
  int64_t bytes = 0; // payload bytes moved per execution
  ~Batch() {
    for (auto &g : groups) cudaFree(g.d_jobs);
  }
};

namespace {

Geom batch_geom(const RowDims &rd, int w) {
  if (static_cast<int>(rd.cnt.size()) > KMAX) fail(SP_ERR_UNSUPPORTED, "batch: too many row dimensions");
  uint64_t rows = 1;
  for (int64_t c : rd.cnt) rows *= static_cast<uint64_t>(c);
  const uint64_t words = rows * static_cast<uint64_t>(rd.c0) / static_cast<uint64_t>(w);
  if (words >= (1ull << 32) || rows >= (1ull << 32) || rd.c0 / w >= (int64_t{1} << 32))
    fail(SP_ERR_UNSUPPORTED, "batch: job larger than 2^32 words");
  Geom g{};
  g.nd = static_cast<int>(rd.cnt.size());
  for (int k = 0; k < g.nd; ++k) {
    g.cnt[k] = static_cast<uint32_t>(rd.cnt[k]);
    g.div[k] = make_fastdiv(g.cnt[k]);
    g.str[k] = rd.str[k];
    g.back[k] = rd.cnt[k] * rd.str[k];
  }
  g.wpr = static_cast<uint32_t>(rd.c0 / w);
  g.wdiv = make_fastdiv(g.wpr);
  g.total = words;
  g.rows = rows;
  return g;
}

uint64_t align_bits(const RowDims &rd, uint64_t base) {
  uint64_t g_or = static_cast<uint64_t>(rd.c0) | base;
  for (int64_t st : rd.str) g_or |= static_cast<uint64_t>(st);
  return g_or;
}

bool same_geom(const RowDims &a, const RowDims &b) { return a.c0 == b.c0 && a.cnt == b.cnt && a.str == b.str; }

// device-accessible address of a batch buffer (device, pinned or peer-mapped)
const uint8_t *batch_ptr(const void *p) {
  const Resolved r = resolve(p);
  if (r.kind == MemKind::Pageable)
    fail(SP_ERR_INVALID_ARGUMENT, "batch: buffers must be device, pinned or peer-mapped memory");
  return r.dptr;
}

Batch *build_batch(std::vector<BatchJob> (&by_w)[5], int mode, int64_t bytes) {
  auto b = std::make_unique<Batch>();
  cuda_check(cudaGetDevice(&b->device), "cudaGetDevice");
  b->bytes = bytes;
  for (int wi = 4; wi >= 0; --wi) {
    auto &jobs = by_w[wi];
    if (jobs.empty()) continue;
    BatchGroup g;
    g.w = 1 << wi;
    g.mode = mode;
    uint64_t chunks = 0;
    for (BatchJob &j : jobs) {
      j.begin = chunks; // first chunk of the job
      chunks += ((mode == kModeUnpack ? j.gd.total : j.gs.total) + kBatchChunk - 1) / kBatchChunk;
      if (chunks >= (1ull << 32)) fail(SP_ERR_UNSUPPORTED, "batch: too much work for one launch");
    }
    g.njobs = static_cast<int>(jobs.size());
    g.nchunks = static_cast<uint32_t>(chunks);
    bool compact = jobs.size() <= static_cast<size_t>(kParamJobs);
    for (const BatchJob &j : jobs) {
      const bool needs_s = mode != kModeUnpack, needs_d = mode == kModeUnpack || (mode == kModeCopy && !j.same);
      compact = compact && (!needs_s || j.gs.nd <= 3) && (!needs_d || j.gd.nd <= 3);
    }
    if (compact) {
      auto t = std::make_shared<CTable>();
      std::memset(t.get(), 0, sizeof(CTable));
      auto cg = [](const Geom &g) {
        CGeom c{};
        c.nd = g.nd;
        c.wpr = g.wpr;
        c.wdiv = g.wdiv;
        c.c0 = g.cnt[0];
        c.c1 = g.cnt[1];
        c.d0 = g.div[0];
        c.d1 = g.div[1];
        c.s0 = g.str[0];
        c.s1 = g.str[1];
        c.s2 = g.str[2];
        c.total = static_cast<uint32_t>(g.total);
        return c;
      };
      for (size_t i = 0; i < jobs.size(); ++i) {
        CJob &c = t->jobs[i];
        c.in = jobs[i].in;
        c.out = jobs[i].out;
        c.gs = cg(jobs[i].gs);
        c.gd = cg(jobs[i].gd);
        c.begin = static_cast<uint32_t>(jobs[i].begin);
        c.q0 = jobs[i].q0;
        c.same = jobs[i].same;
      }
      t->njobs = g.njobs;
      t->nchunks = g.nchunks;
      g.table = t;
    }
    cuda_check(cudaMalloc(&g.d_jobs, jobs.size() * sizeof(BatchJob)), "cudaMalloc(batch)");
    b->groups.push_back(g);
    cuda_check(cudaMemcpy(g.d_jobs, jobs.data(), jobs.size() * sizeof(BatchJob), cudaMemcpyHostToDevice),
               "upload batch");
  }
  return b.release();
}

} // namespace

namespace {

// validated job of one (type, count, buffers) pack or unpack; `align` is
// OR-ed into the word-size choice (chunk boundaries of a pipelined message).
// Returns false for an Empty form (nothing to move).
bool make_pack_job(const BatchSpec &s, bool unpack, uint64_t align, BatchJob &j, int &w) {
  const Committed &ct = *s.ct;
  // argument checks in the reference's precedence (pack.hpp:102-126 / :146-159)
  if (s.count < 1 || s.position < 0) fail(SP_ERR_INVALID_ARGUMENT, "batch: count must be positive, position >= 0");
  if (unpack && ct.overlapping) fail(SP_ERR_OVERLAPPING_LAYOUT, "batch: unpack layout describes overlapping bytes");
  const uint64_t packed_need = static_cast<uint64_t>(s.position + s.count * ct.size);
  if (packed_need > (unpack ? s.src_bytes : s.dst_bytes)) fail(SP_ERR_BUFFER_TOO_SMALL, "batch: packed buffer too small");
  if (ct.form == SP_FORM_EMPTY) return false;
  const uint64_t strided_need = static_cast<uint64_t>((s.count - 1) * ct.extent + ct.span);
  if (strided_need > (unpack ? s.dst_bytes : s.src_bytes)) fail(SP_ERR_BUFFER_TOO_SMALL, "batch: strided buffer too small");
  if (ct.form != SP_FORM_STRIDED) fail(SP_ERR_UNSUPPORTED, "batch: only strided forms can be batched");
  const uint8_t *strided = batch_ptr(unpack ? s.dst : s.src) + ct.sb.start;
  const uint8_t *packed = batch_ptr(unpack ? s.src : s.dst) + s.position;
  const RowDims rd = row_dims(ct, s.count);
  w = pow2_align(align_bits(rd, reinterpret_cast<uint64_t>(strided)) | reinterpret_cast<uint64_t>(packed) | align);
  j = BatchJob{};
  const Geom g = batch_geom(rd, w);
  if (unpack) {
    j.gd = g;
  } else {
    j.gs = g;
  }
  j.in = unpack ? packed : strided;
  j.out = const_cast<uint8_t *>(unpack ? strided : packed);
  return true;
}

bool make_copy_job(const CopySpec &s, uint64_t align, BatchJob &j, int &w) {
  const Committed &sc = *s.sct, &dc = *s.dct;
  if (s.scount < 0 || s.dcount < 0) fail(SP_ERR_INVALID_ARGUMENT, "copy: counts must be >= 0");
  if (s.scount * sc.size != s.dcount * dc.size)
    fail(SP_ERR_INVALID_ARGUMENT, "copy: source and destination describe different byte counts");
  if (dc.overlapping) fail(SP_ERR_OVERLAPPING_LAYOUT, "copy: destination layout describes overlapping bytes");
  if (s.scount * sc.size == 0) return false;
  if (static_cast<uint64_t>((s.scount - 1) * sc.extent + sc.span) > s.src_bytes)
    fail(SP_ERR_BUFFER_TOO_SMALL, "copy: source too small");
  if (static_cast<uint64_t>((s.dcount - 1) * dc.extent + dc.span) > s.dst_bytes)
    fail(SP_ERR_BUFFER_TOO_SMALL, "copy: destination too small");
  if (sc.form != SP_FORM_STRIDED || dc.form != SP_FORM_STRIDED)
    fail(SP_ERR_UNSUPPORTED, "copy: only strided forms can be batched");
  const uint8_t *src = batch_ptr(s.src) + sc.sb.start;
  const uint8_t *dst = batch_ptr(s.dst) + dc.sb.start;
  const RowDims rs = row_dims(sc, s.scount), rd = row_dims(dc, s.dcount);
  w = pow2_align(align_bits(rs, reinterpret_cast<uint64_t>(src)) | align_bits(rd, reinterpret_cast<uint64_t>(dst)) |
                 align);
  j = BatchJob{};
  j.gs = batch_geom(rs, w);
  j.gd = batch_geom(rd, w);
  j.same = same_geom(rs, rd) ? 1 : 0;
  j.in = src;
  j.out = const_cast<uint8_t *>(dst);
  return true;
}

} // namespace

Batch *batch_create(const std::vector<BatchSpec> &specs, bool unpack) {
  require_device();
  std::vector<BatchJob> by_w[5]; // W = 1, 2, 4, 8, 16
  int64_t bytes = 0;
  for (const BatchSpec &s : specs) {
    BatchJob j;
    int w = 1;
    if (!make_pack_job(s, unpack, 0, j, w)) continue;
    by_w[__builtin_ctz(static_cast<unsigned>(w))].push_back(j);
    bytes += s.count * s.ct->size;
  }
  return build_batch(by_w, unpack ? kModeUnpack : kModePack, bytes);
}

Batch *copy_batch_create(const std::vector<CopySpec> &specs) {
  require_device();
  std::vector<BatchJob> by_w[5];
  int64_t bytes = 0;
  for (const CopySpec &s : specs) {
    BatchJob j;
    int w = 1;
    if (!make_copy_job(s, 0, j, w)) continue;
    by_w[__builtin_ctz(static_cast<unsigned>(w))].push_back(j);
    bytes += s.scount * s.sct->size;
  }
  return build_batch(by_w, kModeCopy, bytes);
}

namespace {

template <int W, int MODE> void launch_batch(const BatchGroup &g, const BatchSig &sig, cudaStream_t s, unsigned &grid) {
  static thread_local int occ_dev = -1, occ = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (occ_dev != dev) {
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_batch<W, MODE>, 256, 0), "occupancy");
    occ = std::max(occ, 1);
    occ_dev = dev;
  }
  grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(g.nchunks, static_cast<uint64_t>(sm_count()) * occ)));
  if (g.table) {
    k_batchp<W, MODE><<<grid, 256, 0, s>>>(*g.table, sig);
  } else {
    k_batch<W, MODE><<<grid, 256, 0, s>>>(g.d_jobs, g.njobs, g.nchunks, sig);
  }
}

template <int W> void launch_batch_w(const BatchGroup &g, const BatchSig &sig, cudaStream_t s, unsigned &grid) {
  switch (g.mode) {
  case kModePack: launch_batch<W, kModePack>(g, sig, s, grid); break;
  case kModeUnpack: launch_batch<W, kModeUnpack>(g, sig, s, grid); break;
  default: launch_batch<W, kModeCopy>(g, sig, s, grid); break;
  }
}

void batch_launch(const Batch &b, void *stream, const BatchSignal *bs) {
  sp_launch_info li{};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (size_t gi = 0; gi < b.groups.size(); ++gi) {
    const BatchGroup &g = b.groups[gi];
    BatchSig sig{};
    if (bs) { // pre-signal and wait in the first kernel, signal from the last
      if (bs->wait.size() > static_cast<size_t>(kMaxSig) || bs->signal.size() > static_cast<size_t>(kMaxSig) ||
          bs->pre.size() > static_cast<size_t>(kMaxSig))
        fail(SP_ERR_UNSUPPORTED, "batch signalling: more than 32 peers");
      if (gi == 0) {
        sig.n_pre = static_cast<int>(bs->pre.size());
        for (int i = 0; i < sig.n_pre; ++i) sig.pre[i] = reinterpret_cast<unsigned long long *>(bs->pre[i]);
        sig.pre_value = bs->pre_value;
        sig.n_wait = static_cast<int>(bs->wait.size());
        for (int i = 0; i < sig.n_wait; ++i) sig.wait[i] = reinterpret_cast<const unsigned long long *>(bs->wait[i]);
        sig.wait_value = bs->wait_value;
      }
      if (gi + 1 == b.groups.size()) {
        sig.n_signal = static_cast<int>(bs->signal.size());
        for (int i = 0; i < sig.n_signal; ++i) sig.signal[i] = reinterpret_cast<unsigned long long *>(bs->signal[i]);
        sig.signal_value = bs->signal_value;
        sig.done = bs->done;
        sig.sys_scope = bs->sys_scope ? 1 : 0;
        if (bs->post.size() > static_cast<size_t>(kMaxSig)) fail(SP_ERR_UNSUPPORTED, "batch signalling: more than 32 peers");
        sig.n_post = static_cast<int>(bs->post.size());
        for (int i = 0; i < sig.n_post; ++i) sig.post[i] = reinterpret_cast<const unsigned long long *>(bs->post[i]);
        sig.post_value = bs->post_value;
        if (!bs->signal_values.empty() || !bs->post_values.empty()) {
          if (bs->signal_values.size() != bs->signal.size() || bs->post_values.size() != bs->post.size())
            fail(SP_ERR_INTERNAL, "batch signalling: per-target values do not match the targets");
          sig.per_target = 1;
          for (int i = 0; i < sig.n_signal; ++i) sig.signal_vals[i] = bs->signal_values[i];
          for (int i = 0; i < sig.n_post; ++i) sig.post_vals[i] = bs->post_values[i];
        }
      }
    }
    unsigned grid = 0;
    switch (g.w) {
    case 16: launch_batch_w<16>(g, sig, s, grid); break;
    case 8: launch_batch_w<8>(g, sig, s, grid); break;
    case 4: launch_batch_w<4>(g, sig, s, grid); break;
    case 2: launch_batch_w<2>(g, sig, s, grid); break;
    default: launch_batch_w<1>(g, sig, s, grid); break;
    }
    cuda_check(cudaGetLastError(), "k_batch launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    li.kernel = SP_KERNEL_BATCH;
    li.launches += 1;
    li.grid = grid;
    li.block = 256;
  }
  set_last_launch(li);
}
} // namespace


namespace {

template <int W, int MODE> void launch_job(const BatchJob &j, uint32_t words, cudaStream_t s) {
  static thread_local int occ_dev = -1, occ = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (occ_dev != dev) {
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_job<W, MODE>, 256, 0), "occupancy");
    occ = std::max(occ, 1);
    occ_dev = dev;
  }
  const uint64_t want = (static_cast<uint64_t>(words) + kBatchChunk - 1) / kBatchChunk;
  uint64_t cap = static_cast<uint64_t>(sm_count()) * occ;
  if (t_host_grid_cap) cap = std::min<uint64_t>(cap, t_host_grid_cap);
  const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, cap)));
  k_job<W, MODE><<<grid, 256, 0, s>>>(j, words);
  cuda_check(cudaGetLastError(), "k_job launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  sp_launch_info li{};
  li.kernel = SP_KERNEL_BATCH;
  li.word = W;
  li.launches = 1;
  li.grid = grid;
  li.block = 256;
  set_last_launch(li);
}

template <int MODE> void launch_job_w(int w, const BatchJob &j, uint32_t words, cudaStream_t s) {
  switch (w) {
  case 16: launch_job<16, MODE>(j, words, s); break;
  case 8: launch_job<8, MODE>(j, words, s); break;
  case 4: launch_job<4, MODE>(j, words, s); break;
  case 2: launch_job<2, MODE>(j, words, s); break;
  default: launch_job<1, MODE>(j, words, s); break;
  }
}

// words [lo/w, hi/w) of a job's stream in one launch
void launch_range(int mode, int w, BatchJob j, uint64_t total_bytes, uint64_t lo, uint64_t hi, cudaStream_t s) {
  if (hi > total_bytes || lo > hi) fail(SP_ERR_INVALID_ARGUMENT, "range outside the message");
  if (lo == hi) return;
  if ((hi - lo) / w >= (1ull << 32) || hi / w >= (1ull << 32)) fail(SP_ERR_UNSUPPORTED, "range larger than 2^32 words");
  j.begin = 0;
  j.q0 = static_cast<uint32_t>(lo / w);
  const uint32_t words = static_cast<uint32_t>((hi - lo) / w);
  switch (mode) {
  case kModePack: launch_job_w<kModePack>(w, j, words, s); break;
  case kModeUnpack: launch_job_w<kModeUnpack>(w, j, words, s); break;
  default: launch_job_w<kModeCopy>(w, j, words, s); break;
  }
}

// chunk boundaries strictly inside the message carry alignment; the end of
// the message is a whole number of words by construction
uint64_t range_align(uint64_t lo, uint64_t hi, uint64_t total) { return lo | (hi == total ? 0 : hi); }

} // namespace

bool range_capable(const Committed &ct, int64_t count, const void *strided, const void *packed) {
  if (ct.form != SP_FORM_STRIDED || count < 1) return false;
  if (static_cast<int>(row_dims(ct, count).cnt.size()) > KMAX) return false;
  const Resolved a = resolve(strided), b = resolve(packed);
  return a.kind != MemKind::Pageable && b.kind != MemKind::Pageable;
}

void range_execute(const BatchSpec &spec, bool unpack, uint64_t lo, uint64_t hi, void *stream) {
  require_device();
  const uint64_t total = static_cast<uint64_t>(spec.count * spec.ct->size);
  BatchJob j;
  int w = 1;
  if (!make_pack_job(spec, unpack, range_align(lo, hi, total), j, w)) return;
  launch_range(unpack ? kModeUnpack : kModePack, w, j, total, lo, hi, static_cast<cudaStream_t>(stream));
}

void copy_execute(const CopySpec &spec, uint64_t lo, uint64_t hi, void *stream) {
  require_device();
  const uint64_t total = static_cast<uint64_t>(spec.scount * spec.sct->size);
  BatchJob j;
  int w = 1;
  if (!make_copy_job(spec, range_align(lo, hi, total), j, w)) return;
  launch_range(kModeCopy, w, j, total, lo, hi, static_cast<cudaStream_t>(stream));
}

// one warp: release-store each signal, then wait for each post flag; the
// completion protocol of a neighbour call that moves no bytes
__global__ void k_flag_signal_wait(const BatchSig sig) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int i = 0; i < sig.n_signal; ++i)
      st_release_sys(sig.signal[i], sig.per_target ? sig.signal_vals[i] : sig.signal_value);
  }
  if (threadIdx.x < static_cast<unsigned>(sig.n_post))
    while (ld_acquire_sys(sig.post[threadIdx.x]) < (sig.per_target ? sig.post_vals[threadIdx.x] : sig.post_value))
      __nanosleep(32);
}

void flags_signal_wait(const BatchSignal &bs, void *stream) {
  if (bs.signal.size() > static_cast<size_t>(kMaxSig) || bs.post.size() > static_cast<size_t>(kMaxSig))
    fail(SP_ERR_UNSUPPORTED, "flag signalling: more than 32 peers");
  if (bs.signal.empty() && bs.post.empty()) return;
  BatchSig sig{};
  sig.n_signal = static_cast<int>(bs.signal.size());
  sig.n_post = static_cast<int>(bs.post.size());
  for (int i = 0; i < sig.n_signal; ++i) sig.signal[i] = reinterpret_cast<unsigned long long *>(bs.signal[i]);
  for (int i = 0; i < sig.n_post; ++i) sig.post[i] = reinterpret_cast<const unsigned long long *>(bs.post[i]);
  sig.signal_value = bs.signal_value;
  sig.post_value = bs.post_value;
  if (!bs.signal_values.empty() || !bs.post_values.empty()) {
    sig.per_target = 1;
    for (int i = 0; i < sig.n_signal; ++i) sig.signal_vals[i] = bs.signal_values[i];
    for (int i = 0; i < sig.n_post; ++i) sig.post_vals[i] = bs.post_values[i];
  }
  k_flag_signal_wait<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(sig);
  cuda_check(cudaGetLastError(), "k_flag_signal_wait launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void batch_execute(const Batch &b, void *stream) { batch_launch(b, stream, nullptr); }

void batch_execute_signaled(const Batch &b, void *stream, const BatchSignal &sig) {
  if (b.groups.empty()) fail(SP_ERR_UNSUPPORTED, "batch signalling needs at least one non-empty job");
  batch_launch(b, stream, &sig);
}

void batch_destroy(Batch *b) { delete b; }

int64_t batch_bytes(const Batch &b) { return b.bytes; }

// check_user_buffer (pack.hpp:85-91), same message
static void need_bytes(uint64_t have, int64_t need, const char *what) {
  if (static_cast<uint64_t>(need) > have)
    fail(SP_ERR_BUFFER_TOO_SMALL, std::string(what) + ": need " + std::to_string(need) + " bytes, have " +
                                      std::to_string(have));
}

// Validation order follows pack.hpp:102-126 / :146-159 exactly.
int64_t execute(const PackArgs &a) {
  const Committed &ct = *a.ct;
  sp_launch_info li{};
  if (a.pack) {
    if (a.count < 1 || a.position < 0) fail(SP_ERR_INVALID_ARGUMENT, "pack: incount must be positive, position >= 0");
    need_bytes(a.dst_bytes, a.position + a.count * ct.size, "pack: destination");
    if (ct.form == SP_FORM_EMPTY) {
      set_last_launch(li);
      return a.position;
    }
    need_bytes(a.src_bytes, (a.count - 1) * ct.extent + ct.span, "pack: source");
    if (ct.form == SP_FORM_UNSUPPORTED && !a.opt.allow_fallback)
      fail(SP_ERR_UNSUPPORTED, "pack: type has no strided form");
  } else {
    if (a.count < 1 || a.position < 0) fail(SP_ERR_INVALID_ARGUMENT, "unpack: outcount must be positive, position >= 0");
    if (ct.overlapping) fail(SP_ERR_OVERLAPPING_LAYOUT, "unpack: layout describes overlapping bytes");
    need_bytes(a.src_bytes, a.position + a.count * ct.size, "unpack: source");
    if (ct.form == SP_FORM_EMPTY) {
      set_last_launch(li);
      return a.position;
    }
    need_bytes(a.dst_bytes, (a.count - 1) * ct.extent + ct.span, "unpack: destination");
    if (ct.form == SP_FORM_UNSUPPORTED && !a.opt.allow_fallback)
      fail(SP_ERR_UNSUPPORTED, "unpack: type has no strided form");
  }
  require_device();
  cudaStream_t s = static_cast<cudaStream_t>(a.stream);
  const int64_t strided_len = (a.count - 1) * ct.extent + ct.span;
  const int64_t packed_len = a.count * ct.size;

  const void *strided_user = a.pack ? a.src : a.dst;
  const Resolved rs = resolve(strided_user);
  const Resolved rp = a.pack ? resolve(static_cast<uint8_t *>(a.dst) + a.position)
                             : resolve(static_cast<const uint8_t *>(a.src) + a.position);
  uint8_t *strided_dev = rs.dptr;
  uint8_t *packed_dev = rp.dptr; // already at position
  // A large packed message in pinned host memory moves by DMA: the copy
  // engine streams it over PCIe while the kernel runs on device memory with
  // the whole GPU (zero-copy kernels would hold SMs hostage to PCIe latency,
  // and two streams could not overlap inbound and outbound traffic). Small
  // messages keep the zero-copy one-shot path (lowest latency).
  const bool dma_packed = rp.kind == MemKind::Pinned && packed_len >= kDmaStageMin;
  struct CapGuard {
    explicit CapGuard(bool on) { t_host_grid_cap = on ? kHostGridCap : 0; }
    ~CapGuard() { t_host_grid_cap = 0; }
  } cap_guard(rs.kind == MemKind::Pinned || (rp.kind == MemKind::Pinned && !dma_packed));
  uint8_t *scratch_s = nullptr, *scratch_p = nullptr;
  bool staged = false, must_sync = false;
  uint8_t *dma_stage = nullptr;
  if (dma_packed) {
    staged = true;
    dma_stage = scratch_p = stage_buffer(s, static_cast<size_t>(packed_len));
    if (!a.pack)
      cuda_check(cudaMemcpyAsync(scratch_p, static_cast<const uint8_t *>(a.src) + a.position,
                                 static_cast<size_t>(packed_len), cudaMemcpyHostToDevice, s),
                 "dma packed H2D");
    packed_dev = scratch_p;
  }
  if (rs.kind == MemKind::Pageable) {
    staged = must_sync = true;
    cuda_check(cudaMallocAsync(reinterpret_cast<void **>(&scratch_s), static_cast<size_t>(strided_len), s),
               "cudaMallocAsync(stage)");
    // pack reads the span; unpack must preserve bytes outside the layout
    cuda_check(cudaMemcpyAsync(scratch_s, strided_user, static_cast<size_t>(strided_len), cudaMemcpyHostToDevice, s),
               "stage strided H2D");
    strided_dev = scratch_s;
  }
  if (rp.kind == MemKind::Pageable) {
    staged = must_sync = true;
    cuda_check(cudaMallocAsync(reinterpret_cast<void **>(&scratch_p), static_cast<size_t>(packed_len), s),
               "cudaMallocAsync(stage)");
    if (!a.pack)
      cuda_check(cudaMemcpyAsync(scratch_p, static_cast<const uint8_t *>(a.src) + a.position,
                                 static_cast<size_t>(packed_len), cudaMemcpyHostToDevice, s),
                 "stage packed H2D");
    packed_dev = scratch_p;
  }
  if (a.pack) {
    launch(ct, a.count, strided_dev, nullptr, nullptr, packed_dev, true, s, a.opt, li);
  } else {
    launch(ct, a.count, nullptr, strided_dev, packed_dev, nullptr, false, s, a.opt, li);
  }
  if (staged) {
    if (a.pack && scratch_p)
      cuda_check(cudaMemcpyAsync(static_cast<uint8_t *>(a.dst) + a.position, scratch_p,
                                 static_cast<size_t>(packed_len), cudaMemcpyDeviceToHost, s),
                 "stage packed D2H");
    if (!a.pack && scratch_s)
      cuda_check(cudaMemcpyAsync(a.dst, scratch_s, static_cast<size_t>(strided_len), cudaMemcpyDeviceToHost, s),
                 "stage strided D2H");
    if (scratch_s) cuda_check(cudaFreeAsync(scratch_s, s), "cudaFreeAsync");
    if (scratch_p && scratch_p != dma_stage) cuda_check(cudaFreeAsync(scratch_p, s), "cudaFreeAsync");
    // pageable memory is only safe once the copies completed; pinned DMA
    // staging stays stream-ordered like every other call
    if (must_sync) cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(stage)");
  }
  li.staged = staged;
  set_last_launch(li);
  return a.position + packed_len;
}

} // namespace spb

extern "C" sp_status sp_last_launch(sp_launch_info *out) {
  if (!out) return SP_ERR_INVALID_ARGUMENT;
  *out = spb::t_last;
  return SP_OK;
}

extern "C" int64_t sp_kernel_launch_count(void) { return spb::g_launches.load(); }
