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
//   k_runs<W, PACK>    definition-order run table on the device, for forms
//                      without a strided canon (zero-stride "Unsupported"
//                      types, irregular indexed/struct types) or with more
//                      row dims than a kernel carries; one thread per packed
//                      word, run found by binary search.
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
#include "kernels.cuh"
#include "tma.hpp"

namespace spb {

std::atomic<int64_t> g_launches{0};
static thread_local sp_launch_info t_last{};

void set_last_launch(const sp_launch_info &li) { t_last = li; }

void cuda_check(int err, const char *what) {
  const cudaError_t e = static_cast<cudaError_t>(err);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(SP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

void copy_sync(void *dst, const void *src, size_t n, const char *what) {
  if (n == 0) return;
  // one private non-blocking stream per host thread and device
  thread_local cudaStream_t streams[64] = {};
  int cur = 0;
  cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
  cudaStream_t &st = streams[cur & 63];
  if (!st) cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate(copy_sync)");
  cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, st), what);
  cuda_check(cudaStreamSynchronize(st), what);
}

cudaMemPool_t engine_pool() {
  // one pool per device for the engine's stream-ordered scratch (staging
  // buffers, STAGED transfers): its release threshold keeps the memory
  // mapped across synchronisations. The default pool returns it to the
  // driver at every sync, so a 64 MiB STAGED message re-mapped its scratch
  // each time (0.3-10 ms of variance per message).
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  cudaMemPool_t &p = pools[dev & 63];
  if (!p) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cuda_check(cudaMemPoolCreate(&p, &props), "cudaMemPoolCreate");
    uint64_t keep = uint64_t{4} << 30; // up to 4 GiB stays mapped between uses
    cuda_check(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep), "cudaMemPoolSetAttribute");
  }
  return p;
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(SP_ERR_NO_DEVICE, "no CUDA device: the B200 kernels are the only execution path");
  }
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
// mean run length from which misaligned runs (word < 8) take k_runs_shift
// (scripts/runs_bench.py --misaligned: pack wins from 32 B; unpack, whose
// run ends are masked stores, from 1 KiB -- at 256 B the byte-word kernel
// still ties or wins)
constexpr int64_t kRunsShiftMinPack = 32, kRunsShiftMinUnpack = 512;

static bool shift_wins(bool pack, int w, int64_t c0) {
  if (pack) return w <= 2 || (w == 4 && c0 % 16 == 0);
  return w <= 2 && c0 >= 128;
}

// the 16 bytes starting d bytes into x0, continuing into x1 (d < 16): a
// switch on the word offset d >> 2 picks compile-time word indices, so each
// output word is one funnel shift (no select chain; when the offset is
// uniform across a warp -- one shift per run -- there is no divergence)
__device__ __forceinline__ uint4 funnel16(const uint4 &x0, const uint4 &x1, unsigned d) {
  const unsigned sh = (d & 3) * 8;
  switch (d >> 2) {
  case 0:
    return make_uint4(__funnelshift_r(x0.x, x0.y, sh), __funnelshift_r(x0.y, x0.z, sh),
                      __funnelshift_r(x0.z, x0.w, sh), __funnelshift_r(x0.w, x1.x, sh));
  case 1:
    return make_uint4(__funnelshift_r(x0.y, x0.z, sh), __funnelshift_r(x0.z, x0.w, sh),
                      __funnelshift_r(x0.w, x1.x, sh), __funnelshift_r(x1.x, x1.y, sh));
  case 2:
    return make_uint4(__funnelshift_r(x0.z, x0.w, sh), __funnelshift_r(x0.w, x1.x, sh),
                      __funnelshift_r(x1.x, x1.y, sh), __funnelshift_r(x1.y, x1.z, sh));
  default:
    return make_uint4(__funnelshift_r(x0.w, x1.x, sh), __funnelshift_r(x1.x, x1.y, sh),
                      __funnelshift_r(x1.y, x1.z, sh), __funnelshift_r(x1.z, x1.w, sh));
  }
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
  return funnel16(x0, x1, d); // a warp whose rows disagree on d >> 2 runs the cases in turn
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

// ------------------------------------------------------------ k_runs
// Run-table kernel for forms without a strided canon (the reference's
// zero-stride "Unsupported" types, irregular indexed/struct types) and for
// strided forms with more row dims than KMAX. The table holds the runs in
// definition order as pieces (<= kPieceMax bytes). A group of G = 2^lg
// lanes takes one (object, piece) item at a time, grid-stride, prefetching
// the next item's descriptor, and moves its W-byte words lane-strided with
// four loads in flight per lane: both sides of a piece are contiguous, so a
// group's accesses coalesce. G is the largest power of two <= the mean
// piece length in words, capped at 16 (measured best from 16-B to 4-KiB
// runs: scripts/runs_bench.py, profiles/r01_runs_kernel.md). Duplicated
// source bytes pack with their multiplicity (pack.hpp:123-135).
template <int W, bool PACK>
__global__ void __launch_bounds__(256) k_runs(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                              const int64_t *__restrict__ psrc, const int64_t *__restrict__ pdst,
                                              int64_t npieces, int64_t nobj, int64_t extent, int64_t size, int lg) {
  using T = typename Word<W>::T;
  const int g = 1 << lg;
  const int lane = static_cast<int>(threadIdx.x) & (g - 1);
  const int64_t groups = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> lg;
  const int64_t total = npieces * nobj;
  int64_t p = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> lg;
  if (p >= total) return;
  // the next item's descriptor is loaded before this item's words move
  int64_t k = p % npieces;
  int64_t ns = __ldg(psrc + k), nd = __ldg(pdst + k), ne = __ldg(pdst + k + 1);
  for (; p < total; p += groups) {
    const int64_t j = p / npieces;
    const int64_t s0 = ns, d0 = nd, words = (ne - nd) / W;
    if (p + groups < total) {
      k = (p + groups) % npieces;
      ns = __ldg(psrc + k);
      nd = __ldg(pdst + k);
      ne = __ldg(pdst + k + 1);
    }
    const T *sw = reinterpret_cast<const T *>(PACK ? in + j * extent + s0 : in + j * size + d0);
    T *dw = reinterpret_cast<T *>(PACK ? out + j * size + d0 : out + j * extent + s0);
    int64_t w = lane;
    for (; w + 3 * g < words; w += 4 * g) { // four loads in flight before the stores
      const T a = ld_stream(sw + w), b = ld_stream(sw + w + g), c = ld_stream(sw + w + 2 * g),
              e = ld_stream(sw + w + 3 * g);
      st_stream(dw + w, a);
      st_stream(dw + w + g, b);
      st_stream(dw + w + 2 * g, c);
      st_stream(dw + w + 3 * g, e);
    }
    for (; w < words; w += g) st_stream(dw + w, ld_stream(sw + w));
  }
}

__device__ __forceinline__ uint4 shfl_down4(unsigned mask, const uint4 &x, int width) {
  return make_uint4(__shfl_down_sync(mask, x.x, 1, width), __shfl_down_sync(mask, x.y, 1, width),
                    __shfl_down_sync(mask, x.z, 1, width), __shfl_down_sync(mask, x.w, 1, width));
}

// Runs whose offsets only allow 1-, 2- or 4-byte words (byte-granular
// hindexed / struct displacements): the shift technique of k_shift_* per
// piece. A group of G lanes takes an (object, piece) item; lane l of the
// group owns aligned 16-B block c*G + l of the WRITTEN side. Consecutive
// written blocks read consecutive aligned 16-B blocks of the read side at
// one fixed byte shift, so each lane loads ONE aligned read block and takes
// the next one from its neighbour lane (a shuffle; the group's last lane
// loads its own), then assembles its 16 bytes with funnel shifts. Only read
// blocks that intersect the run are loaded; the blocks at the two ends of a
// run are stored masked. Every lane of a group runs the same trip count,
// so the shuffles name just the group's lanes.
// one run of `len` bytes from src to dst by a group of g lanes (lane l of
// the group, `gmask` names the group's lanes in the warp): the body of
// k_runs_shift and k_runs_multi_shift
__device__ __forceinline__ void shift_run(const uint8_t *src, uint8_t *dst, int64_t len, int g, int lane,
                                          unsigned gmask) {
  const uint4 zero = make_uint4(0, 0, 0, 0);
  const uintptr_t A = reinterpret_cast<uintptr_t>(dst), E = A + static_cast<uintptr_t>(len);
  const uintptr_t S = reinterpret_cast<uintptr_t>(src), SE = S + static_cast<uintptr_t>(len);
  const uintptr_t first = A & ~uintptr_t{15};
  const int64_t nblk = static_cast<int64_t>(((E + 15) & ~uintptr_t{15}) - first) / 16;
  // read address of written block B is B + (S - A): a fixed byte shift
  const uintptr_t r0 = first + (S - A);
  const unsigned d = static_cast<unsigned>(r0 & 15);
  // written block b: its aligned read block, the next one (neighbour lane
  // or own load), the assembled 16 bytes, the (masked) store
  auto load = [&](int64_t b, uint4 &x0, uint4 &x1) {
    const uintptr_t rb = (r0 & ~uintptr_t{15}) + 16 * static_cast<uintptr_t>(b);
    x0 = b < nblk && rb < SE && rb + 16 > S ? ld_stream(reinterpret_cast<const uint4 *>(rb)) : zero;
    const uintptr_t nb = rb + 16;
    const bool own = lane == g - 1 || b + 1 >= nblk;
    x1 = own && b < nblk && d && nb < SE && nb + 16 > S ? ld_stream(reinterpret_cast<const uint4 *>(nb)) : zero;
  };
  auto put = [&](int64_t b, const uint4 &x0, uint4 x1, const uint4 &nx) {
    if (!(lane == g - 1 || b + 1 >= nblk)) x1 = nx;
    if (b >= nblk) return;
    const uint4 z = d ? funnel16(x0, x1, d) : x0;
    const uintptr_t B = first + 16 * static_cast<uintptr_t>(b);
    const uintptr_t vlo = B > A ? B : A, vhi = B + 16 < E ? B + 16 : E;
    uint8_t *blk = reinterpret_cast<uint8_t *>(B);
    if (vlo == B && vhi == B + 16) {
      st_stream(reinterpret_cast<uint4 *>(blk), z);
    } else {
      store_masked(blk, z, static_cast<unsigned>(vlo - B), static_cast<unsigned>(vhi - B));
    }
  };
  int64_t c = 0;
  for (; c + g < nblk; c += 2 * g) { // two chunks of G blocks: up to four loads in flight per lane
    uint4 a0, a1, b0, b1;
    load(c + lane, a0, a1);
    load(c + g + lane, b0, b1);
    const uint4 na = shfl_down4(gmask, a0, g), nb = shfl_down4(gmask, b0, g);
    put(c + lane, a0, a1, na);
    put(c + g + lane, b0, b1, nb);
  }
  if (c < nblk) {
    uint4 a0, a1;
    load(c + lane, a0, a1);
    const uint4 na = shfl_down4(gmask, a0, g);
    put(c + lane, a0, a1, na);
  }
}

__device__ __forceinline__ unsigned group_mask(int g) {
  return (g == 32 ? 0xffffffffu : ((1u << g) - 1u)) << ((threadIdx.x & 31) & ~(g - 1));
}

// Runs whose offsets only allow 1-, 2- or 4-byte words (byte-granular
// hindexed / struct displacements): the shift technique of k_shift_* per
// piece. A group of G lanes takes an (object, piece) item; lane l of the
// group owns aligned 16-B block c*G + l of the WRITTEN side. Consecutive
// written blocks read consecutive aligned 16-B blocks of the read side at
// one fixed byte shift, so each lane loads ONE aligned read block and takes
// the next one from its neighbour lane (a shuffle; the group's last lane
// loads its own), then assembles its 16 bytes with funnel shifts. Only read
// blocks that intersect the run are loaded; the blocks at the two ends of a
// run are stored masked. Every lane of a group runs the same trip count,
// so the shuffles name just the group's lanes.
template <bool PACK>
__global__ void __launch_bounds__(256) k_runs_shift(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                    const int64_t *__restrict__ psrc,
                                                    const int64_t *__restrict__ pdst, int64_t npieces, int64_t nobj,
                                                    int64_t extent, int64_t size, int lg) {
  const int g = 1 << lg;
  const int lane = static_cast<int>(threadIdx.x) & (g - 1);
  const unsigned gmask = group_mask(g);
  const int64_t groups = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> lg;
  const int64_t total = npieces * nobj;
  for (int64_t p = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> lg; p < total; p += groups) {
    const int64_t j = p / npieces, k = p - j * npieces;
    const int64_t s0 = __ldg(psrc + k), d0 = __ldg(pdst + k), len = __ldg(pdst + k + 1) - d0;
    shift_run(PACK ? in + j * extent + s0 : in + j * size + d0, PACK ? out + j * size + d0 : out + j * extent + s0,
              len, g, lane, gmask);
  }
}

// Several run-table packs in one launch (the irregular edges of a
// neighbour collective): the edge table travels in kernel-parameter space,
// an item (edge, object, piece) finds its edge by binary search over the
// edges' first-item indices (constant cache), then moves like k_runs.
constexpr int kRunEdges = 32;
struct RunEdge {
  const int64_t *psrc, *pdst;
  int64_t npieces, nobj, extent, size, item0;
  const uint8_t *in;
  uint8_t *out;
  int64_t unpack; // 0: gather into packed `out`; 1: scatter packed `in`
};
struct RunTable {
  RunEdge e[kRunEdges];
  int n;
  int64_t total;
};

template <int W>
__global__ void __launch_bounds__(256) k_runs_multi(const __grid_constant__ RunTable t, int lg) {
  using T = typename Word<W>::T;
  const int g = 1 << lg;
  const int lane = static_cast<int>(threadIdx.x) & (g - 1);
  const int64_t groups = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> lg;
  for (int64_t p = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> lg; p < t.total; p += groups) {
    int a = 0, b = t.n - 1;
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (t.e[m].item0 <= p) {
        a = m;
      } else {
        b = m - 1;
      }
    }
    const RunEdge &e = t.e[a];
    const int64_t local = p - e.item0;
    const int64_t j = local / e.npieces, k = local - j * e.npieces;
    const int64_t s0 = __ldg(e.psrc + k), d0 = __ldg(e.pdst + k), words = (__ldg(e.pdst + k + 1) - d0) / W;
    const T *sw = reinterpret_cast<const T *>(e.unpack ? e.in + j * e.size + d0 : e.in + j * e.extent + s0);
    T *dw = reinterpret_cast<T *>(e.unpack ? e.out + j * e.extent + s0 : e.out + j * e.size + d0);
    int64_t w = lane;
    for (; w + 3 * g < words; w += 4 * g) {
      const T v0 = ld_stream(sw + w), v1 = ld_stream(sw + w + g), v2 = ld_stream(sw + w + 2 * g),
              v3 = ld_stream(sw + w + 3 * g);
      st_stream(dw + w, v0);
      st_stream(dw + w + g, v1);
      st_stream(dw + w + 2 * g, v2);
      st_stream(dw + w + 3 * g, v3);
    }
    for (; w < words; w += g) st_stream(dw + w, ld_stream(sw + w));
  }
}

// k_runs_multi with the shift technique: misaligned irregular edges of a
// neighbour collective (byte-granular runs, mean >= kRunsShiftMin*)
__global__ void __launch_bounds__(256) k_runs_multi_shift(const __grid_constant__ RunTable t, int lg) {
  const int g = 1 << lg;
  const int lane = static_cast<int>(threadIdx.x) & (g - 1);
  const unsigned gmask = group_mask(g);
  const int64_t groups = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> lg;
  for (int64_t p = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> lg; p < t.total; p += groups) {
    int a = 0, b = t.n - 1;
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (t.e[m].item0 <= p) {
        a = m;
      } else {
        b = m - 1;
      }
    }
    const RunEdge &e = t.e[a];
    const int64_t local = p - e.item0;
    const int64_t j = local / e.npieces, k = local - j * e.npieces;
    const int64_t s0 = __ldg(e.psrc + k), d0 = __ldg(e.pdst + k), len = __ldg(e.pdst + k + 1) - d0;
    shift_run(e.unpack ? e.in + j * e.size + d0 : e.in + j * e.extent + s0,
              e.unpack ? e.out + j * e.extent + s0 : e.out + j * e.size + d0, len, g, lane, gmask);
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
    if (cur >= 0) cudaSetDevice(cur);
  }
}

// (row_dims, pow2_align, resolve, sm_count, t_host_grid_cap: kernels.cuh)
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
constexpr int64_t kDmaStageMin = int64_t{1} << 20; // pinned packed messages >= 1 MiB move by DMA

namespace {

// Persistent per-(device, stream) staging buffers for DMA'd messages. Work
// on one stream is ordered, so reuse by the next call on that stream is
// safe; a pool allocation freed on one stream and reused on another would
// make the stream-ordered allocator insert a cross-stream dependency and
// serialise the inbound and outbound legs of a pipelined exchange.
constexpr size_t kStagePad = 32;

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
  if (st.n < bytes + kStagePad) {
    if (st.p) cuda_check(cudaFreeAsync(st.p, s), "cudaFreeAsync(stage)");
    const size_t n = std::max(bytes + kStagePad, st.n * 2);
    cuda_check(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&st.p), n, engine_pool(), s), "cudaMallocAsync(stage)");
    st.n = n;
  }
  return st.p;
}

// A DMA lane beside a caller's stream: a copy stream and a ring of events,
// so the PCIe leg of a large pinned-host message overlaps its kernels chunk
// by chunk (H2D of chunk k+1 while chunk k unpacks; D2H of chunk k while
// chunk k+1 packs). One per (device, caller stream), like the stage buffers.
constexpr int kLaneEvents = 64;
// packed bytes per pipelined chunk (TEMPI_DMA_CHUNK overrides, >= 64 KiB)
int64_t dma_chunk() {
  static const int64_t c = [] {
    const char *e = std::getenv("TEMPI_DMA_CHUNK");
    const int64_t v = e && *e ? std::atoll(e) : 0;
    return v >= (int64_t{64} << 10) ? v : int64_t{8} << 20;
  }();
  return c;
}
struct DmaLane {
  cudaStream_t cs = nullptr;
  cudaEvent_t ev[kLaneEvents] = {};
  int next = 0;
  cudaEvent_t take() {
    cudaEvent_t e = ev[next];
    next = (next + 1) % kLaneEvents;
    return e;
  }
};

DmaLane &dma_lane(cudaStream_t s) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, DmaLane> lanes;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  DmaLane &l = lanes[{dev, s}];
  if (!l.cs) {
    cuda_check(cudaStreamCreateWithFlags(&l.cs, cudaStreamNonBlocking), "cudaStreamCreate(dma lane)");
    for (cudaEvent_t &e : l.ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  }
  return l;
}

unsigned grid_for(uint64_t items, int per_thread) {
  const uint64_t blocks = (items + 256ull * per_thread - 1) / (256ull * per_thread);
  uint64_t cap = static_cast<uint64_t>(sm_count()) * 8; // 8 x 256 = 2048 threads/SM
  if (t_host_grid_cap) cap = std::min<uint64_t>(cap, t_host_grid_cap);
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(blocks, cap)));
}

// grid of 256-thread CTAs for `items` threads of work, capped at one
// resident wave of kernel K (occupancy queried once per kernel and device;
// the template parameter is the kernel itself, so every instantiation has
// its own cache)
template <auto K> unsigned resident_grid(uint64_t items) {
  static thread_local int dev = -1, occ = 0;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) {
    dev = cur;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, K, 256, 0) != cudaSuccess || occ < 1) occ = 1;
  }
  const uint64_t blocks = (items + 255) / 256;
  const uint64_t cap = static_cast<uint64_t>(sm_count()) * static_cast<uint64_t>(occ);
  const uint64_t hcap = t_host_grid_cap ? std::min<uint64_t>(cap, t_host_grid_cap) : cap;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(blocks, hcap)));
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
    ct.dev = DeviceRuns{};
  }
  std::vector<int64_t> hs, hd;
  hs.reserve(runs.size());
  hd.reserve(runs.size() + 1);
  int64_t acc = 0;
  uint64_t align_or = 0;
  for (const Run &r : runs) {
    align_or |= static_cast<uint64_t>(r.off) | static_cast<uint64_t>(r.len);
    for (int64_t o = 0; o < r.len; o += kPieceMax) {
      hs.push_back(r.off + o);
      hd.push_back(acc + o);
    }
    acc += r.len;
  }
  hd.push_back(acc);
  DeviceRuns d;
  d.device = cur;
  d.n = static_cast<int64_t>(hs.size());
  d.align_or = align_or;
  cuda_check(cudaMalloc(&d.d_src, std::max<size_t>(hs.size(), 1) * sizeof(int64_t)), "cudaMalloc(runs)");
  cuda_check(cudaMalloc(&d.d_dst, hd.size() * sizeof(int64_t)), "cudaMalloc(runs)");
  copy_sync(d.d_src, hs.data(), hs.size() * sizeof(int64_t), "upload runs");
  copy_sync(d.d_dst, hd.data(), hd.size() * sizeof(int64_t), "upload runs");
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
// The copy engines instead of SMs (future work: "evaluate
// the use of the GPU DMA engine for non-contiguous data (e.g.
// cudaMemcpy2D)"): the row geometry as pitched 3-D copies, a third
// dimension folded in when its stride is a whole number of pitches, one call
// per remaining outer index. No SM is used, so the copy can run beside an
// application's kernels; its rate is set by the copy engines.
constexpr int64_t kDmaMaxCalls = 4096;

void dma_copy(const RowDims &r, const uint8_t *src, uint8_t *dst, bool pack, cudaStream_t s, sp_launch_info &li) {
  const size_t w = static_cast<size_t>(r.c0);
  if (r.cnt.empty()) { // one contiguous row
    cuda_check(cudaMemcpyAsync(dst, src, w, cudaMemcpyDefault, s), "cudaMemcpyAsync(dma)");
    li.launches = 1;
    return;
  }
  const int64_t h = r.cnt[0], pitch = r.str[0];
  if (pitch < r.c0) fail(SP_ERR_UNSUPPORTED, "DMA path: rows overlap (pitch below the row length)");
  const bool three = r.cnt.size() >= 2 && r.str[1] % pitch == 0 && r.str[1] / pitch >= h;
  const size_t inner = three ? 2 : 1;
  const int64_t depth = three ? r.cnt[1] : 1;
  int64_t outer = 1;
  for (size_t k = inner; k < r.cnt.size(); ++k) outer *= r.cnt[k];
  if (outer > kDmaMaxCalls) fail(SP_ERR_UNSUPPORTED, "DMA path: more than 4096 pitched copies");
  const int64_t block = static_cast<int64_t>(w) * h * depth; // packed bytes per call
  std::vector<int64_t> idx(r.cnt.size(), 0);
  for (int64_t o = 0; o < outer; ++o) {
    int64_t soff = 0;
    for (size_t k = inner; k < r.cnt.size(); ++k) soff += idx[k] * r.str[k];
    const uint8_t *strided = (pack ? src : dst) + soff;
    uint8_t *packed = (pack ? dst : const_cast<uint8_t *>(src)) + o * block;
    cudaMemcpy3DParms p{};
    const cudaPitchedPtr sp = make_cudaPitchedPtr(const_cast<uint8_t *>(strided), static_cast<size_t>(pitch), w,
                                                  three ? static_cast<size_t>(r.str[1] / pitch) : static_cast<size_t>(h));
    const cudaPitchedPtr pp = make_cudaPitchedPtr(packed, w, w, static_cast<size_t>(h));
    p.srcPtr = pack ? sp : pp;
    p.dstPtr = pack ? pp : sp;
    p.extent = make_cudaExtent(w, static_cast<size_t>(h), static_cast<size_t>(depth));
    p.kind = cudaMemcpyDefault;
    cuda_check(cudaMemcpy3DAsync(&p, s), "cudaMemcpy3DAsync(dma)");
    for (size_t k = inner; k < r.cnt.size(); ++k) { // odometer over the outer dims
      if (++idx[k] < r.cnt[k]) break;
      idx[k] = 0;
    }
  }
  li.launches = static_cast<int>(outer);
}

void launch(const Committed &ct, int64_t count, const uint8_t *strided_in, uint8_t *strided_out,
            const uint8_t *packed_in, uint8_t *packed_out, bool pack, cudaStream_t s,
            const sp_pack_options &opt, sp_launch_info &li) {
  const uint8_t *in = pack ? strided_in : packed_in;
  uint8_t *out = pack ? packed_out : strided_out;
  const uint64_t strided_addr = reinterpret_cast<uint64_t>(pack ? strided_in : strided_out);
  const uint64_t packed_addr = reinterpret_cast<uint64_t>(pack ? packed_out : packed_in);

  if (opt.kernel == SP_KERNEL_DMA) {
    if (ct.form != SP_FORM_STRIDED) fail(SP_ERR_UNSUPPORTED, "DMA path: the type has no strided form");
    dma_copy(row_dims(ct, count), pack ? strided_in + ct.sb.start : packed_in,
             pack ? packed_out : strided_out + ct.sb.start, pack, s, li);
    li.kernel = SP_KERNEL_DMA;
    li.word = 0;
    li.grid = li.block = 0;
    return;
  }
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
    // the word divides every run offset and length, the extent, the object
    // size and both buffer addresses
    int w = pow2_align(dr.align_or | static_cast<uint64_t>(ct.extent) | static_cast<uint64_t>(ct.size) |
                       strided_addr | packed_addr);
    if (opt.force_word) {
      if (opt.force_word > w || (opt.force_word & (opt.force_word - 1)))
        fail(SP_ERR_INVALID_ARGUMENT, "force_word is not legal for these buffers");
      w = opt.force_word;
    }
    // misaligned runs (word < 8) of 32 B and more on average: 16-B blocks of
    // the written side assembled by funnel shifts (profiles/r02_kernel_choices.md)
    const int64_t mean_bytes = ct.size / std::max<int64_t>(dr.n, 1);
    if (w < 8 && mean_bytes >= (pack ? kRunsShiftMinPack : kRunsShiftMinUnpack) && !opt.force_word &&
        opt.kernel != SP_KERNEL_BLOCKLIST) {
      // lanes per piece: the largest power of two G with 2G <= the mean
      // 16-B blocks per piece (each lane moves two chunks of G blocks per
      // step), at most 16
      int lg = 0;
      while (lg < 4 && (int64_t{4} << lg) <= mean_bytes / 16) ++lg;
      const uint64_t items = static_cast<uint64_t>(dr.n * count) << lg;
      unsigned grid = 1;
      if (pack) {
        grid = resident_grid<k_runs_shift<true>>(items);
        k_runs_shift<true><<<grid, 256, 0, s>>>(in, out, dr.d_src, dr.d_dst, dr.n, count, ct.extent, ct.size, lg);
      } else {
        grid = resident_grid<k_runs_shift<false>>(items);
        k_runs_shift<false><<<grid, 256, 0, s>>>(in, out, dr.d_src, dr.d_dst, dr.n, count, ct.extent, ct.size, lg);
      }
      cuda_check(cudaGetLastError(), "k_runs_shift launch");
      li.kernel = SP_KERNEL_BLOCKLIST;
      li.word = 16;
      li.launches = 1;
      li.grid = grid;
      li.block = 256;
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return;
    }
    // lanes per piece: the largest power of two <= the mean piece length
    // in words, at most 16
    const int64_t mean_words = ct.size / w / std::max<int64_t>(dr.n, 1);
    int lg = 0;
    while (lg < 4 && (int64_t{2} << lg) <= mean_words) ++lg;
    // one resident wave: the grid is capped at what fits (48 registers a
    // thread leave room for 5 CTAs of 256 per SM, not the 8 grid_for assumes)
    const uint64_t items = static_cast<uint64_t>(dr.n * count) << lg;
    unsigned grid = 1;
#define SPB_RUNS(WW)                                                                                               \
  if (pack) {                                                                                                      \
    grid = resident_grid<k_runs<WW, true>>(items);                                                                 \
    k_runs<WW, true><<<grid, 256, 0, s>>>(in, out, dr.d_src, dr.d_dst, dr.n, count, ct.extent, ct.size, lg);      \
  } else {                                                                                                         \
    grid = resident_grid<k_runs<WW, false>>(items);                                                                \
    k_runs<WW, false><<<grid, 256, 0, s>>>(in, out, dr.d_src, dr.d_dst, dr.n, count, ct.extent, ct.size, lg);     \
  }
    switch (w) {
    case 16: SPB_RUNS(16) break;
    case 8: SPB_RUNS(8) break;
    case 4: SPB_RUNS(4) break;
    case 2: SPB_RUNS(2) break;
    default: SPB_RUNS(1) break;
    }
#undef SPB_RUNS
    cuda_check(cudaGetLastError(), "k_runs launch");
    li.kernel = SP_KERNEL_BLOCKLIST;
    li.word = w;
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
  // (they read, never write, whole aligned 16-B blocks around the bytes a
  // layout touches: up to 15 B beyond the span inside the same block, which
  // cannot leave an allocation's 256-B-granular footprint; the engine's own
  // staging buffers are padded so the sanitizer's exact bounds hold too)
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
    cuda_check(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&cnt64), KMAX * sizeof(uint64_t), engine_pool(), s), "cudaMallocAsync");
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


template <int W> unsigned launch_runs_multi(const RunTable &t, int lg, cudaStream_t s) {
  const unsigned grid = resident_grid<k_runs_multi<W>>(static_cast<uint64_t>(t.total) << lg);
  k_runs_multi<W><<<grid, 256, 0, s>>>(t, lg);
  return grid;
}
} // namespace



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
  // (the copy-engine path reads and writes pinned memory itself)
  const bool dma_packed = rp.kind == MemKind::Pinned && packed_len >= kDmaStageMin && a.opt.kernel != SP_KERNEL_DMA;
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
    packed_dev = scratch_p; // the H2D of an unpack is issued below (whole, or chunked)
  }
  if (rs.kind == MemKind::Pageable) {
    staged = must_sync = true;
    // + kStagePad: the shift kernels read whole aligned 16-B blocks around
    // the bytes a layout touches, which may run past an exact-size end
    cuda_check(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&scratch_s), static_cast<size_t>(strided_len) + kStagePad, engine_pool(), s),
               "cudaMallocAsync(stage)");
    // pack reads the span; unpack must preserve bytes outside the layout
    cuda_check(cudaMemcpyAsync(scratch_s, strided_user, static_cast<size_t>(strided_len), cudaMemcpyHostToDevice, s),
               "stage strided H2D");
    strided_dev = scratch_s;
  }
  if (rp.kind == MemKind::Pageable) {
    staged = must_sync = true;
    cuda_check(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&scratch_p), static_cast<size_t>(packed_len) + kStagePad, engine_pool(), s),
               "cudaMallocAsync(stage)");
    if (!a.pack)
      cuda_check(cudaMemcpyAsync(scratch_p, static_cast<const uint8_t *>(a.src) + a.position,
                                 static_cast<size_t>(packed_len), cudaMemcpyHostToDevice, s),
                 "stage packed H2D");
    packed_dev = scratch_p;
  }
  // a large pinned message of several objects: pipeline the DMA against
  // the kernels in chunks of whole objects on a copy lane beside `s`
  const int64_t per_chunk = std::max<int64_t>(1, dma_chunk() / std::max<int64_t>(ct.size, 1));
  const bool pipelined = dma_packed && rs.kind != MemKind::Pageable && a.count >= 2 && per_chunk < a.count;
  if (pipelined) {
    DmaLane &lane = dma_lane(s);
    const uint8_t *host_in = static_cast<const uint8_t *>(a.src) + a.position;
    uint8_t *host_out = static_cast<uint8_t *>(a.dst) + a.position;
    // the lane's first copy waits for everything earlier on `s` (the stage
    // buffer may still be read or written by the previous call)
    cudaEvent_t e0 = lane.take();
    cuda_check(cudaEventRecord(e0, s), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(lane.cs, e0, 0), "cudaStreamWaitEvent");
    int launches = 0;
    for (int64_t o = 0; o < a.count; o += per_chunk) {
      const int64_t c = std::min(per_chunk, a.count - o);
      const size_t off = static_cast<size_t>(o * ct.size), n = static_cast<size_t>(c * ct.size);
      uint8_t *sd = strided_dev + o * ct.extent;
      cudaEvent_t e = lane.take();
      if (a.pack) {
        launch(ct, c, sd, nullptr, nullptr, packed_dev + off, true, s, a.opt, li);
        cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(lane.cs, e, 0), "cudaStreamWaitEvent");
        cuda_check(cudaMemcpyAsync(host_out + off, packed_dev + off, n, cudaMemcpyDeviceToHost, lane.cs),
                   "dma packed D2H");
      } else {
        cuda_check(cudaMemcpyAsync(packed_dev + off, host_in + off, n, cudaMemcpyHostToDevice, lane.cs),
                   "dma packed H2D");
        cuda_check(cudaEventRecord(e, lane.cs), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(s, e, 0), "cudaStreamWaitEvent");
        launch(ct, c, nullptr, sd, packed_dev + off, nullptr, false, s, a.opt, li);
      }
      ++launches;
    }
    if (a.pack) { // the call completes on `s` when the last D2H has landed
      cudaEvent_t e = lane.take();
      cuda_check(cudaEventRecord(e, lane.cs), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(s, e, 0), "cudaStreamWaitEvent");
    }
    li.launches = launches;
    li.staged = true;
    set_last_launch(li);
    return a.position + packed_len;
  }
  if (dma_packed && !a.pack)
    cuda_check(cudaMemcpyAsync(scratch_p, static_cast<const uint8_t *>(a.src) + a.position,
                               static_cast<size_t>(packed_len), cudaMemcpyHostToDevice, s),
               "dma packed H2D");
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

// Several run-table moves, one launch per up to kRunEdges jobs: the
// irregular (block-list) edges of a neighbour collective, each packed
// straight into its receiver's dense run, or a dense run scattered through
// the receiver's published run table. Buffers must be device, pinned or
// peer-mapped memory; counts of 0 are skipped.
const DeviceRuns &device_run_table(const Committed &ct) {
  if (ct.form == SP_FORM_STRIDED) fail(SP_ERR_INTERNAL, "run table of a strided form");
  return device_runs(ct, ct.runs);
}

void runs_multi(const std::vector<RunJob> &jobs, void *stream) {
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<RunEdge> edges;
  uint64_t align = 0;
  int64_t bytes = 0, items = 0;
  for (const RunJob &j : jobs) {
    RunEdge e{};
    uint64_t table_align = j.align;
    if (j.ct) {
      if (j.ct->form == SP_FORM_STRIDED) fail(SP_ERR_INTERNAL, "runs_multi: strided form");
      const DeviceRuns &dr = device_runs(*j.ct, j.ct->runs);
      e.psrc = dr.d_src;
      e.pdst = dr.d_dst;
      e.npieces = dr.n;
      e.extent = j.ct->extent;
      e.size = j.ct->size;
      table_align = dr.align_or;
    } else {
      e.psrc = j.psrc;
      e.pdst = j.pdst;
      e.npieces = j.npieces;
      e.extent = j.extent;
      e.size = j.size;
    }
    if (j.count <= 0 || e.size == 0) continue;
    const Resolved rs = resolve(j.src), rd = resolve(j.dst);
    if (rs.kind == MemKind::Pageable || rd.kind == MemKind::Pageable)
      fail(SP_ERR_INVALID_ARGUMENT, "neighbour exchange: buffers must be device, pinned or peer-mapped memory");
    e.nobj = j.count;
    e.in = rs.dptr;
    e.out = rd.dptr;
    e.unpack = j.unpack ? 1 : 0;
    align |= table_align | static_cast<uint64_t>(e.extent) | static_cast<uint64_t>(e.size) |
             reinterpret_cast<uint64_t>(e.in) | reinterpret_cast<uint64_t>(e.out);
    bytes += e.size * e.nobj;
    items += e.npieces * e.nobj;
    edges.push_back(e);
  }
  if (edges.empty()) return;
  require_device();
  const int w = pow2_align(align);
  const int64_t mean_words = bytes / w / std::max<int64_t>(items, 1);
  int lg = 0;
  while (lg < 4 && (int64_t{2} << lg) <= mean_words) ++lg;
  // misaligned runs: the shift variant, at the stricter threshold when any
  // edge scatters (k_runs_shift's measured crossovers)
  const bool any_unpack = std::any_of(edges.begin(), edges.end(), [](const RunEdge &e) { return e.unpack != 0; });
  const int64_t mean_bytes = bytes / std::max<int64_t>(items, 1);
  const bool shift = w < 8 && mean_bytes >= (any_unpack ? kRunsShiftMinUnpack : kRunsShiftMinPack);
  if (shift) {
    lg = 0;
    while (lg < 4 && (int64_t{4} << lg) <= mean_bytes / 16) ++lg;
  }
  for (size_t at = 0; at < edges.size(); at += kRunEdges) {
    RunTable t{};
    t.n = static_cast<int>(std::min<size_t>(kRunEdges, edges.size() - at));
    int64_t acc = 0;
    for (int i = 0; i < t.n; ++i) {
      t.e[i] = edges[at + static_cast<size_t>(i)];
      t.e[i].item0 = acc;
      acc += t.e[i].npieces * t.e[i].nobj;
    }
    t.total = acc;
    if (shift) {
      const unsigned grid = resident_grid<k_runs_multi_shift>(static_cast<uint64_t>(t.total) << lg);
      k_runs_multi_shift<<<grid, 256, 0, s>>>(t, lg);
    } else {
      switch (w) {
      case 16: launch_runs_multi<16>(t, lg, s); break;
      case 8: launch_runs_multi<8>(t, lg, s); break;
      case 4: launch_runs_multi<4>(t, lg, s); break;
      case 2: launch_runs_multi<2>(t, lg, s); break;
      default: launch_runs_multi<1>(t, lg, s); break;
      }
    }
    cuda_check(cudaGetLastError(), "k_runs_multi launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
}

} // namespace spb

extern "C" sp_status sp_last_launch(sp_launch_info *out) {
  if (!out) return SP_ERR_INVALID_ARGUMENT;
  *out = spb::t_last;
  return SP_OK;
}

extern "C" int64_t sp_kernel_launch_count(void) { return spb::g_launches.load(); }
