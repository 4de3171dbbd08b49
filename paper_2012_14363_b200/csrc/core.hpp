// core.hpp -- host-side datatype engine (internal).
//
// The B200 engine keeps the reference's semantics (canonical StridedBlock,
// reference PackPlan, pack byte order, error precedence) but not its
// structure: definitions carry size/extent/span computed once at
// construction (O(1) per level), the IR chain is a flat vector rewritten in
// place, and overlap is decided exactly from the StridedBlock lattice instead
// of enumerating and sorting every byte run (commit.hpp:57 in the reference
// is O(size log size); here commit is O(tree) + a bounded search).
#pragma once

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime_api.h>

#include "stridepack_b200.h"

namespace spb {

// ---------------------------------------------------------------- errors
struct Error {
  sp_status code;
  std::string msg;
};
[[noreturn]] void fail(sp_status code, std::string msg);
// message returned by sp_last_error() on this thread
void set_last_error(const std::string &msg);

// ---------------------------------------------------------------- types
// Named..Subarray are the reference's constructors. Indexed (MPI indexed,
// hindexed and their _block forms, byte displacements), Struct and Resized
// go beyond it (MPI-3.1 sections 4.1.2-4.1.7; the paper's future work,
// PAPER.md:1164): regular ones canonicalise like the rest, irregular ones
// commit to the block-list form.
enum class Kind : uint8_t { Named, Contiguous, Vector, Hvector, Subarray, Indexed, Struct, Resized };

// One definition level (type_def.hpp:52-123). Immutable once built.
struct TypeDef {
  Kind kind = Kind::Named;
  int named = 0;            // SP_BYTE..SP_DOUBLE
  int64_t count = 0;        // contiguous/vector/hvector count
  int64_t blocklength = 0;  // vector/hvector
  int64_t stride = 0;       // vector: inner extents; hvector: bytes
  std::vector<int64_t> sizes, subsizes, offsets; // subarray, dim 0 innermost
  std::vector<int64_t> blocklens, displs;        // indexed/struct: per block, displs in bytes
  std::shared_ptr<const TypeDef> inner;           // every kind but Named and Struct
  std::vector<std::shared_ptr<const TypeDef>> members; // struct: type of each block
  // derived once (type_def.hpp:198-250 + block_list span); lb is MPI's
  // lower bound (0 for the reference's constructors, which never move it)
  int64_t size = 0, extent = 0, span = 0, lb = 0;
  int depth = 1;
};
using DefPtr = std::shared_ptr<const TypeDef>;

DefPtr make_named(int kind);
DefPtr make_contiguous(int64_t count, DefPtr inner);
DefPtr make_vector(int64_t count, int64_t bl, int64_t stride, DefPtr inner);
DefPtr make_hvector(int64_t count, int64_t bl, int64_t stride_b, DefPtr inner);
DefPtr make_subarray(int64_t ndims, const int64_t *sizes,
                     const int64_t *subsizes, const int64_t *offsets,
                     DefPtr inner, int order);
// MPI_Type_create_hindexed (displacements in bytes; MPI_Type_indexed and
// the _block forms scale/replicate before calling)
DefPtr make_indexed(int64_t count, const int64_t *blocklens, const int64_t *displs_bytes, DefPtr inner);
// MPI_Type_create_struct
DefPtr make_struct(int64_t count, const int64_t *blocklens, const int64_t *displs_bytes,
                   const std::vector<DefPtr> &members);
// MPI_Type_create_resized
DefPtr make_resized(DefPtr inner, int64_t lb, int64_t extent);

// ---------------------------------------------------------------- canon
// Canonical strided form (strided_block.hpp:17-46): counts[0] bytes at
// stride 1, counts[i>0] repetitions at strides[i] (non-decreasing).
struct StridedBlock {
  int64_t start = 0;
  std::vector<int64_t> counts, strides;
  int ndims() const { return static_cast<int>(counts.size()); }
};

// The reference's descriptive plan (plan.hpp:27-44), kept for parity.
struct RefPlan {
  int64_t word = 1;
  int64_t block[3] = {1, 1, 1};
  int64_t grid[3] = {1, 1, 1};
  int strategy = SP_STRATEGY_GRIDZ;
};

struct Run {
  int64_t off, len;
};

// Device copy of the definition-order run table for the block-list kernel.
// The run table on the device, as pieces: runs in definition order, each
// split into pieces of at most kPieceMax bytes so no single long run can
// serialise a kernel.
constexpr int64_t kPieceMax = int64_t{64} << 10;
struct DeviceRuns {
  int device = -1;
  int64_t *d_src = nullptr;   // piece source offsets (within one object)
  int64_t *d_dst = nullptr;   // packed offsets: exclusive prefix sum, n + 1 entries
  int64_t n = 0;              // pieces
  uint64_t align_or = 0;      // OR of every run offset and length (word choice)
};

struct Committed {
  int form = SP_FORM_EMPTY;
  int64_t size = 0, extent = 0, span = 0;
  bool overlapping = false;
  StridedBlock sb;        // valid when form == STRIDED
  RefPlan plan;           // valid when form == STRIDED
  int64_t simplify_rounds = -1;
  int64_t n_def_runs = 0; // reference fallback_runs.size() (Unsupported)
  std::vector<Run> runs;  // definition-order runs, adjacent runs coalesced
                          // (Unsupported form only; multiplicity preserved)
  mutable std::mutex dev_mu;
  mutable DeviceRuns dev; // lazily uploaded block list
  ~Committed();
};
using CommitPtr = std::shared_ptr<const Committed>;

// translate + simplify + lower + plan + exact overlap (commit.hpp:51-79)
CommitPtr commit_def(const TypeDef &def);

// the definition's normalized run list (block_list.hpp:44-61 over :67-121)
std::vector<Run> flatten_def(const TypeDef &def, bool &overlap);

// type-file front end (typefile.hpp:17-260); name = the committed name
DefPtr parse_type_file(const std::string &text, std::string &name);

// exposed for tests via the C-ABI: exact injectivity of a strided block
bool strided_overlaps(const StridedBlock &sb);

// ---------------------------------------------------------------- registry
struct Entry {
  DefPtr def;
  CommitPtr committed; // null until sp_type_commit
};

class Registry {
public:
  sp_type add(DefPtr def);
  Entry get(sp_type h) const;  // copy of the entry, fails on bad handle
  CommitPtr committed(sp_type h) const; // the commit record, fails when absent
  CommitPtr commit(sp_type h);
  void remove(sp_type h);
  // bumped by every remove(): callers that cache handle -> record lookups
  // across calls revalidate when it moves (handles are never reused)
  uint64_t generation() const { return gen_.load(std::memory_order_acquire); }

private:
  mutable std::shared_mutex mu_;
  std::unordered_map<sp_type, Entry> map_;
  sp_type next_ = 1;
  std::atomic<uint64_t> gen_{0};
};
Registry &registry();

// ---------------------------------------------------------------- execution
struct PackArgs {
  const Committed *ct;
  const void *src;
  uint64_t src_bytes;
  void *dst;
  uint64_t dst_bytes;
  int64_t count;    // incount / outcount
  int64_t position; // byte offset into the packed buffer
  void *stream;
  sp_pack_options opt;
  bool pack;        // true: gather (pack), false: scatter (unpack)
};
// validated launch (pack.cu); returns new position
int64_t execute(const PackArgs &a);

// several block-list moves in one launch (pack.cu): each job packs `count`
// objects of a block-list form from src to the packed bytes at dst, or
// (unpack) scatters packed src through the form into dst. The form is `ct`
// (its cached device run table) or, when ct is null, an explicit device
// run table (e.g. a peer's, mapped through CUDA IPC).
struct RunJob {
  const Committed *ct;
  const void *src;
  int64_t count;
  void *dst;
  bool unpack = false;
  const int64_t *psrc = nullptr, *pdst = nullptr;
  int64_t npieces = 0, size = 0, extent = 0;
  uint64_t align = 0;
};
void runs_multi(const std::vector<RunJob> &jobs, void *stream);
// the device run table of a block-list form (uploaded once, cached)
const DeviceRuns &device_run_table(const Committed &ct);

void set_last_launch(const sp_launch_info &li);
void cuda_check(int err, const char *what);  // cudaError_t as int
void require_device();
// the engine's stream-ordered memory pool on the current device (scratch and
// staging buffers; memory stays mapped between uses)
cudaMemPool_t engine_pool();
// Copy `n` bytes (any direction, pageable or device source) and return only
// when they have landed in `dst`. A plain cudaMemcpy is not enough: from
// pageable host memory it may return before the DMA completes, device to
// device it does not wait at all, and in both cases it runs on the legacy
// stream, which orders nothing on the engine's non-blocking streams or in
// other processes reading the buffer through CUDA IPC.
void copy_sync(void *dst, const void *src, size_t n, const char *what);

// persistent multi-job launches (pack.cu)
struct BatchSpec {
  const Committed *ct;
  const void *src;
  uint64_t src_bytes;
  int64_t count;
  void *dst;
  uint64_t dst_bytes;
  int64_t position;
};
struct Batch;
Batch *batch_create(const std::vector<BatchSpec> &specs, bool unpack);
// typed copies: byte k of (sct, scount) at src lands on byte k of
// (dct, dcount) at dst; scount*sct.size must equal dcount*dct.size
struct CopySpec {
  const Committed *sct;
  const void *src;
  uint64_t src_bytes;
  int64_t scount;
  const Committed *dct;
  void *dst;
  uint64_t dst_bytes;
  int64_t dcount;
};
Batch *copy_batch_create(const std::vector<CopySpec> &specs);
// single-job launches over the packed-byte range [lo, hi) of one message
// (chunks of a pipelined message; lo and interior hi multiples of 16):
// no descriptor upload, the job travels as a kernel parameter
bool range_capable(const Committed &ct, int64_t count, const void *strided, const void *packed);
void range_execute(const BatchSpec &spec, bool unpack, uint64_t lo, uint64_t hi, void *stream);
void copy_execute(const CopySpec &spec, uint64_t lo, uint64_t hi, void *stream);
void batch_execute(const Batch &b, void *stream);
void batch_destroy(Batch *b);
// in-kernel completion protocol for distributed exchanges (pack.cu)
struct BatchSignal {
  std::vector<const uint64_t *> wait; // local flags, each must reach wait_value
  uint64_t wait_value = 0;
  std::vector<uint64_t *> signal;     // (peer) counters: every launch adds 2^32 in total
  bool sys_scope = true;              // a destination is on another GPU
  std::vector<uint64_t *> pre;        // (peer) flags set to pre_value BEFORE the wait
  uint64_t pre_value = 0;
  std::vector<const uint64_t *> post; // local counters block 0 waits for after signalling
  uint64_t post_value = 0;
  std::vector<uint64_t> post_values;  // per-target post values (else the scalar)
  bool stream_waits = true; // pre/wait through stream memory ops (else block 0 / every block in-kernel)
  int *err = nullptr;      // set to 1 by an in-kernel wait that gave up (mapped host memory)
  uint64_t timeout_ns = 0; // in-kernel wait limit, 0 = unbounded
  // Device-side iteration numbers (a launch replayed from a CUDA graph): when
  // `iter` is set the kernels read it = *iter (advanced by iter_tick ahead of
  // the launch) and use value = (it + add) << shift for pre / wait / post
  // instead of the values above. In-kernel waits only.
  const uint64_t *iter = nullptr;
  int64_t pre_add = 0, wait_add = 0, post_add = 0;
  int pre_shift = 0, wait_shift = 0, post_shift = 0;
  // host-numbered launches record their iteration here (block 0), so a
  // later switch to device numbering continues from it
  uint64_t *iter_store = nullptr;
  uint64_t iter_value = 0;
};
constexpr int kMaxSignalPeers = 32; // flags a signalled launch carries (batch.cu kMaxSig)
// one-warp kernel: adds 2^32 to each signal counter, then waits for the post counters
void flags_signal_wait(const BatchSignal &sig, void *stream);
void batch_execute_signaled(const Batch &b, void *stream, const BatchSignal &sig);
// one-thread kernel: *counter += 1 (the device iteration number of a
// graph-replayable exchange)
void iter_tick(uint64_t *counter, void *stream);
int64_t batch_bytes(const Batch &b);

} // namespace spb
