// batch.cu -- many-job launches (pack, unpack, typed copy), single-job
// ranged launches (pipelined message chunks, sp_copy) and the in-kernel
// completion protocol of the distributed halo and neighbour collectives.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "core.hpp"
#include "kernels.cuh"

namespace spb {

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
// Work distribution: every job is cut into chunks of kBatchChunk words (the
// last one partial), and the chunks of all jobs form one index space that
// the CTAs of a single resident wave walk grid-stride. A thread moves U
// words of its chunk with all U loads issued before the first store. The
// chunk's job is found by binary search on the jobs' first-chunk indices:
// up to kParamJobs jobs with <= 3 row dims travel in kernel-parameter space
// (k_batchp, constant-cache reads), larger batches stage the chunk's job in
// shared memory (k_batch). Measured alternatives (balanced contiguous
// ranges, dynamic chunk tickets, launch-order interleaving, job orderings,
// U = 2 / 8, 8 CTAs/SM with spills) are in profiles/r01_halo_batch.md.
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

// Optional completion protocol (distributed halo). Before any word moves,
// the `pre` flags are published and each `wait` flag (local memory, written
// by peers over NVLink) must reach wait_value, in one of two places:
//  * in the kernel (every rank on its own GPU): block 0 release-stores the
//    pre flags, every block spins on an acquire load of the wait flags;
//  * in the stream (ranks share a GPU -- MPS, time slicing): stream memory
//    operations ahead of the launch (stream_flag_ops) publish and then hold
//    the stream in its front end, on no SM, so a rank's spinning full-wave
//    grid can never starve the peer kernel it waits for; the blocks' acquire
//    loads then no longer spin.
// After its last word, EVERY block adds its share
// of 2^32 to each `signal` counter (peer memory) with a release reduction --
// the shares of a launch sum to exactly 2^32 whatever the grid, so a
// receiver waits for calls << 32 without knowing the sender's grid, and no
// block waits for another to finish before signalling.
constexpr int kMaxSig = kMaxSignalPeers;
struct BatchSig {
  const unsigned long long *wait[kMaxSig];
  unsigned long long *signal[kMaxSig];
  unsigned long long wait_value;
  int n_wait, n_signal;
  int sys_scope;  // some destination lives on another GPU: system-scope fences
  // in-kernel mode only: published by block 0 BEFORE any block waits
  unsigned long long *pre[kMaxSig];
  unsigned long long pre_value;
  int n_pre;
  // waited for by block 0 after it signalled (completion of the peers'
  // writes into this rank's memory folded into the same launch)
  const unsigned long long *post[kMaxSig];
  unsigned long long post_value;
  int n_post;
  // per-target post values (neighbour collectives count calls per peer
  // pair); used instead of post_value when per_target is set
  unsigned long long post_vals[kMaxSig];
  int per_target;
  // bounded waits: a spin that outlives timeout_ns sets *err and gives up
  // (the host reports SP_ERR_TIMEOUT after its next synchronisation)
  unsigned long long timeout_ns;
  int *err;
  // device iteration numbering (BatchSignal::iter): values (it + add) << shift
  const unsigned long long *iter;
  long long pre_add, wait_add, post_add;
  int pre_shift, wait_shift, post_shift;
  unsigned long long *iter_store; // block 0 records iter_value here
  unsigned long long iter_value;
};

// a protocol value: the host's, or derived from the device iteration number
__device__ __forceinline__ unsigned long long sig_value(const BatchSig &sig, unsigned long long host, long long add,
                                                        int shift) {
  if (!sig.iter) return host;
  const unsigned long long it = *reinterpret_cast<const volatile unsigned long long *>(sig.iter);
  return (it + static_cast<unsigned long long>(add)) << shift;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// release reduction: the CTA's stores (ordered before this thread by the
// preceding bar.sync) become visible to whoever acquires the counter
__device__ __forceinline__ void red_release_add(unsigned long long *p, unsigned long long v, int sys) {
  if (sys) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  } else {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  }
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// spin until *p >= v (acquire, system scope); a peer that never publishes
// -- it died, or never entered the call -- ends the spin after
// sig.timeout_ns with *sig.err set instead of hanging this GPU
__device__ __forceinline__ void wait_flag(const unsigned long long *p, unsigned long long v, const BatchSig &sig,
                                          unsigned sleep_ns) {
  if (ld_acquire_sys(p) >= v) return;
  const unsigned long long t0 = global_ns();
  while (ld_acquire_sys(p) < v) {
    __nanosleep(sleep_ns);
    if (sig.timeout_ns && global_ns() - t0 > sig.timeout_ns) {
      if (sig.err) atomicExch(sig.err, 1);
      return;
    }
  }
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
  if (sig.iter_store && blockIdx.x == 0 && threadIdx.x == 0) *sig.iter_store = sig.iter_value;
  if (sig.n_pre && blockIdx.x == 0 && threadIdx.x < static_cast<unsigned>(sig.n_pre))
    st_release_sys(sig.pre[threadIdx.x], sig_value(sig, sig.pre_value, sig.pre_add, sig.pre_shift));
  // stream mode: satisfied before the launch, one acquire load each;
  // in-kernel mode (every rank on its own GPU): spins until the peers publish
  if (sig.n_wait) {
    if (threadIdx.x < static_cast<unsigned>(sig.n_wait))
      wait_flag(sig.wait[threadIdx.x], sig_value(sig, sig.wait_value, sig.wait_add, sig.wait_shift), sig, 64);
    __syncthreads();
  }
}

// Per-CTA completion: bar.sync orders every thread's stores before the
// signalling threads, whose release reductions are cumulative over them (GPU
// scope when every destination is on this device, system scope when some
// were written over NVLink into a peer GPU). Block b adds
// floor((b+1)2^32/G) - floor(b 2^32/G), so one launch adds exactly 2^32 to
// each counter. Block 0 then waits for the post counters: the launch ends
// only when the peers' writes into this rank have landed. No last-block
// election, no serialised completion atomic, no system fence chain.
__device__ __forceinline__ void batch_epilogue(const BatchSig &sig) {
  if (sig.n_signal || sig.n_post) {
    __syncthreads();
    if (threadIdx.x < static_cast<unsigned>(sig.n_signal)) {
      const unsigned long long g = gridDim.x, b = blockIdx.x;
      const unsigned long long share = ((b + 1) << 32) / g - (b << 32) / g;
      red_release_add(sig.signal[threadIdx.x], share, sig.sys_scope);
    }
    // every peer signals before it waits, so block 0 of two ranks cannot
    // wait on each other in a cycle; the grid is one resident wave, so the
    // other blocks run to completion meanwhile
    if (blockIdx.x == 0 && threadIdx.x < static_cast<unsigned>(sig.n_post))
      wait_flag(sig.post[threadIdx.x],
                sig.per_target ? sig.post_vals[threadIdx.x]
                               : sig_value(sig, sig.post_value, sig.post_add, sig.post_shift),
                sig, 32);
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
    copy_sync(g.d_jobs, jobs.data(), jobs.size() * sizeof(BatchJob), "upload batch");
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
  // one resident wave of the kernel actually launched (the parameter-table
  // and the smem-staged variants are occupancy-queried separately)
  static thread_local int occ_dev = -1, occ_t = 0, occ_s = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (occ_dev != dev) {
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_batch<W, MODE>, 256, 0), "occupancy");
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, k_batchp<W, MODE>, 256, 0), "occupancy");
    occ_s = std::max(occ_s, 1);
    occ_t = std::max(occ_t, 1);
    occ_dev = dev;
  }
  const int occ = g.table ? occ_t : occ_s;
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

struct FlagStore {
  unsigned long long *p[kMaxSig];
  unsigned long long v;
  int n;
};

// release-stores v to each flag (system scope): the pre flags of a launch
// whose peers are on other GPUs
__global__ void k_flag_store(const FlagStore f) {
  if (threadIdx.x < static_cast<unsigned>(f.n)) st_release_sys(f.p[threadIdx.x], f.v);
}

// one warp: publish the pre flags, then wait for the wait flags -- the
// prologue of a device-numbered launch when ranks share a GPU (stream memory
// operations carry fixed values, and a full-wave grid spinning here could
// starve the peer kernel it waits for; one warp cannot)
__global__ void k_flag_pre_wait(const BatchSig sig) {
  if (threadIdx.x < static_cast<unsigned>(sig.n_pre))
    st_release_sys(sig.pre[threadIdx.x], sig_value(sig, sig.pre_value, sig.pre_add, sig.pre_shift));
  if (threadIdx.x < static_cast<unsigned>(sig.n_wait))
    wait_flag(sig.wait[threadIdx.x], sig_value(sig, sig.wait_value, sig.wait_add, sig.wait_shift), sig, 256);
}

// Stream memory operations (one cuStreamBatchMemOp): write `value` to each
// `writes` flag (ordered after all earlier work on the stream, with the
// write's memory barrier), then block the stream until each `waits` flag
// reaches wait_value (cyclic >=). The wait is held by the stream's front end:
// no SM is occupied while a peer has still to run.
void stream_flag_ops(cudaStream_t s, const std::vector<uint64_t *> &writes, uint64_t value,
                     const std::vector<const uint64_t *> &waits, uint64_t wait_value) {
  if (writes.empty() && waits.empty()) return;
  using BatchMemOp = CUresult (*)(CUstream, unsigned, CUstreamBatchMemOpParams *, unsigned);
  static BatchMemOp fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuStreamBatchMemOp", &f, cudaEnableDefault, &q);
    return reinterpret_cast<BatchMemOp>(f);
  }();
  if (!fn) fail(SP_ERR_CUDA, "cuStreamBatchMemOp is not available");
  if (writes.size() + waits.size() >= 256) fail(SP_ERR_UNSUPPORTED, "stream flag ops: too many peers");
  std::vector<CUstreamBatchMemOpParams> ops(writes.size() + waits.size());
  std::memset(ops.data(), 0, ops.size() * sizeof(CUstreamBatchMemOpParams));
  size_t k = 0;
  for (uint64_t *w : writes) {
    ops[k].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
    ops[k].writeValue.address = reinterpret_cast<CUdeviceptr>(w);
    ops[k].writeValue.value64 = value;
    ops[k].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
    ++k;
  }
  for (const uint64_t *w : waits) {
    ops[k].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
    ops[k].waitValue.address = reinterpret_cast<CUdeviceptr>(w);
    ops[k].waitValue.value64 = wait_value;
    ops[k].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
    ++k;
  }
  const CUresult r = fn(reinterpret_cast<CUstream>(s), static_cast<unsigned>(ops.size()), ops.data(), 0);
  if (r != CUDA_SUCCESS) fail(SP_ERR_CUDA, "cuStreamBatchMemOp failed (" + std::to_string(static_cast<int>(r)) + ")");
}

__global__ void k_iter_tick(unsigned long long *c) { *c += 1; }

void batch_launch(const Batch &b, void *stream, const BatchSignal *bs) {
  sp_launch_info li{};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (size_t gi = 0; gi < b.groups.size(); ++gi) {
    const BatchGroup &g = b.groups[gi];
    BatchSig sig{};
    if (bs) {
      sig.timeout_ns = bs->timeout_ns;
      sig.err = bs->err;
      sig.iter = reinterpret_cast<const unsigned long long *>(bs->iter);
      sig.pre_add = bs->pre_add;
      sig.wait_add = bs->wait_add;
      sig.post_add = bs->post_add;
      sig.pre_shift = bs->pre_shift;
      sig.wait_shift = bs->wait_shift;
      sig.post_shift = bs->post_shift;
      if (gi == 0) {
        sig.iter_store = reinterpret_cast<unsigned long long *>(bs->iter_store);
        sig.iter_value = bs->iter_value;
      }
    }
    if (bs) { // pre-signal and wait in the first kernel, signal from the last
      if (bs->wait.size() > static_cast<size_t>(kMaxSig) || bs->signal.size() > static_cast<size_t>(kMaxSig) ||
          bs->pre.size() > static_cast<size_t>(kMaxSig))
        fail(SP_ERR_UNSUPPORTED, "batch signalling: more than 32 peers");
      if (gi == 0 && bs->stream_waits && bs->iter) {
        // device-numbered iterations with ranks sharing a GPU: a one-warp
        // kernel publishes and waits ahead of the batch
        BatchSig w = sig;
        w.n_pre = static_cast<int>(bs->pre.size());
        for (int i = 0; i < w.n_pre; ++i) w.pre[i] = reinterpret_cast<unsigned long long *>(bs->pre[i]);
        w.pre_value = bs->pre_value;
        w.n_wait = static_cast<int>(bs->wait.size());
        for (int i = 0; i < w.n_wait; ++i) w.wait[i] = reinterpret_cast<const unsigned long long *>(bs->wait[i]);
        w.wait_value = bs->wait_value;
        w.iter_store = nullptr;
        if (w.n_pre || w.n_wait) {
          k_flag_pre_wait<<<1, 32, 0, s>>>(w);
          cuda_check(cudaGetLastError(), "k_flag_pre_wait launch");
          g_launches.fetch_add(1, std::memory_order_relaxed);
        }
      } else if (gi == 0 && !bs->stream_waits) { // every rank on its own GPU: all in the kernel
        if (bs->pre.size() > static_cast<size_t>(kMaxSig)) fail(SP_ERR_UNSUPPORTED, "batch signalling: more than 32 peers");
        sig.n_pre = static_cast<int>(bs->pre.size());
        for (int i = 0; i < sig.n_pre; ++i) sig.pre[i] = reinterpret_cast<unsigned long long *>(bs->pre[i]);
        sig.pre_value = bs->pre_value;
      } else if (gi == 0) {
        if (bs->sys_scope && !bs->pre.empty()) {
          // pre flags in another GPU's memory: stored from an SM (a
          // system-scope release over NVLink), not by a stream memory op
          if (bs->pre.size() > static_cast<size_t>(kMaxSig)) fail(SP_ERR_UNSUPPORTED, "batch signalling: more than 32 peers");
          FlagStore fs{};
          fs.n = static_cast<int>(bs->pre.size());
          for (int i = 0; i < fs.n; ++i) fs.p[i] = reinterpret_cast<unsigned long long *>(bs->pre[i]);
          fs.v = bs->pre_value;
          k_flag_store<<<1, 32, 0, s>>>(fs);
          cuda_check(cudaGetLastError(), "k_flag_store launch");
          g_launches.fetch_add(1, std::memory_order_relaxed);
          stream_flag_ops(s, {}, 0, bs->wait, bs->wait_value);
        } else {
          stream_flag_ops(s, bs->pre, bs->pre_value, bs->wait, bs->wait_value);
        }
      }
      if (gi == 0 && !(bs->stream_waits && bs->iter)) { // (else waited for by k_flag_pre_wait)
        sig.n_wait = static_cast<int>(bs->wait.size());
        for (int i = 0; i < sig.n_wait; ++i) sig.wait[i] = reinterpret_cast<const unsigned long long *>(bs->wait[i]);
        sig.wait_value = bs->wait_value;
      }
      if (gi + 1 == b.groups.size()) {
        sig.n_signal = static_cast<int>(bs->signal.size());
        for (int i = 0; i < sig.n_signal; ++i) sig.signal[i] = reinterpret_cast<unsigned long long *>(bs->signal[i]);
        sig.sys_scope = bs->sys_scope ? 1 : 0;
        if (bs->post.size() > static_cast<size_t>(kMaxSig)) fail(SP_ERR_UNSUPPORTED, "batch signalling: more than 32 peers");
        sig.n_post = static_cast<int>(bs->post.size());
        for (int i = 0; i < sig.n_post; ++i) sig.post[i] = reinterpret_cast<const unsigned long long *>(bs->post[i]);
        sig.post_value = bs->post_value;
        if (!bs->post_values.empty()) {
          if (bs->post_values.size() != bs->post.size())
            fail(SP_ERR_INTERNAL, "batch signalling: per-target values do not match the targets");
          sig.per_target = 1;
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

// one warp: add a whole launch's 2^32 to each signal counter, then wait for
// each post counter; the completion protocol of a neighbour call that moves
// no bytes
__global__ void k_flag_signal_wait(const BatchSig sig) {
  if (threadIdx.x < static_cast<unsigned>(sig.n_signal)) red_release_add(sig.signal[threadIdx.x], 1ull << 32, 1);
  if (threadIdx.x < static_cast<unsigned>(sig.n_post))
    wait_flag(sig.post[threadIdx.x], sig.per_target ? sig.post_vals[threadIdx.x] : sig.post_value, sig, 32);
}

void flags_signal_wait(const BatchSignal &bs, void *stream) {
  if (bs.signal.size() > static_cast<size_t>(kMaxSig) || bs.post.size() > static_cast<size_t>(kMaxSig))
    fail(SP_ERR_UNSUPPORTED, "flag signalling: more than 32 peers");
  if (bs.signal.empty() && bs.post.empty()) return;
  BatchSig sig{};
  sig.timeout_ns = bs.timeout_ns;
  sig.err = bs.err;
  sig.n_signal = static_cast<int>(bs.signal.size());
  sig.n_post = static_cast<int>(bs.post.size());
  for (int i = 0; i < sig.n_signal; ++i) sig.signal[i] = reinterpret_cast<unsigned long long *>(bs.signal[i]);
  for (int i = 0; i < sig.n_post; ++i) sig.post[i] = reinterpret_cast<const unsigned long long *>(bs.post[i]);
  sig.post_value = bs.post_value;
  if (!bs.post_values.empty()) {
    sig.per_target = 1;
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

void iter_tick(uint64_t *counter, void *stream) {
  k_iter_tick<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<unsigned long long *>(counter));
  cuda_check(cudaGetLastError(), "k_iter_tick launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void batch_destroy(Batch *b) { delete b; }

int64_t batch_bytes(const Batch &b) { return b.bytes; }

} // namespace spb
