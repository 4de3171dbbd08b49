/*
 * stridepack_b200.h -- C-ABI of the B200-native derived-datatype engine
 * (libstridepack_b200.so). Plain pointers and sizes only; no CUDA or torch
 * types cross this boundary (streams are passed as `void *` and interpreted
 * as cudaStream_t, NULL = the legacy default stream).
 *
 * Each entry point replaces one entry of the reference engine's C++ API
 * ("stridepack", /root/reference/proj/include/stridepack/); the cited
 * file:line is the interface it stands in for. The reference reports errors
 * as C++ exceptions (errors.hpp:8-47); here every call returns an sp_status
 * whose values map 1:1 onto those exception types, and never throws.
 *
 * Threading: type construction, commit and queries are thread-safe
 * (commit.hpp:81-99). sp_pack/sp_unpack may run concurrently on distinct
 * destination buffers. Kernels are enqueued on the caller's
 * stream on the CURRENT CUDA device; calls on device or pinned host memory
 * return without synchronising. Pageable host buffers are staged through the
 * device and synchronise the stream before returning.
 */
#ifndef STRIDEPACK_B200_H
#define STRIDEPACK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: errors.hpp:8-47 ---------------------------------- */
typedef int sp_status;
enum {
  SP_OK = 0,
  SP_ERR_INVALID_ARGUMENT = 1,   /* InvalidArgument   errors.hpp:13 */
  SP_ERR_UNSUPPORTED_ORDER = 2,  /* UnsupportedOrder  errors.hpp:18 */
  SP_ERR_INVALID_LAYOUT = 3,     /* InvalidLayout     errors.hpp:23 */
  SP_ERR_BUFFER_TOO_SMALL = 4,   /* BufferTooSmall    errors.hpp:27 */
  SP_ERR_OVERLAPPING_LAYOUT = 5, /* OverlappingLayout errors.hpp:32 */
  SP_ERR_UNSUPPORTED = 6,        /* Unsupported       errors.hpp:37 */
  SP_ERR_EMPTY_PROFILE = 7,      /* EmptyProfile      errors.hpp:41 */
  SP_ERR_PARSE = 8,              /* ParseError        errors.hpp:45 */
  SP_ERR_INTERNAL = 9,
  SP_ERR_INVALID_HANDLE = 11,
  SP_ERR_CUDA = 12,              /* a CUDA runtime call failed */
  SP_ERR_NO_DEVICE = 13,         /* no usable CUDA device: the GPU path is
                                    the only execution path, there is no
                                    host fallback */
  SP_ERR_TIMEOUT = 14            /* runtime: a peer rank exited, or did not
                                    answer within TEMPI_TIMEOUT seconds
                                    (host waits and in-kernel flag waits) */
};

/* version of this C-ABI: bumped when a declaration changes incompatibly
 * (SP_ABI_VERSION at compile time, sp_abi_version() at run time) */
#define SP_ABI_VERSION 2
int sp_abi_version(void);

const char *sp_status_string(sp_status s);
/* message of the last failing call on this thread ("" if none) */
const char *sp_last_error(void);

/* ---- datatype construction: type_def.hpp:125-195 -------------------- */
typedef uint64_t sp_type; /* opaque handle; 0 is never valid */

enum { SP_BYTE = 0, SP_INT = 1, SP_FLOAT = 2, SP_DOUBLE = 3 }; /* NamedKind type_def.hpp:15 */
enum { SP_ORDER_C = 0, SP_ORDER_FORTRAN = 1 };                 /* ArrayOrder type_def.hpp:47 */

/* make_named                 type_def.hpp:125 */
sp_status sp_type_named(int kind, sp_type *out);
/* make_contiguous            type_def.hpp:129 */
sp_status sp_type_contiguous(int64_t count, sp_type inner, sp_type *out);
/* make_vector  (stride in inner extents)   type_def.hpp:137 */
sp_status sp_type_vector(int64_t count, int64_t blocklength, int64_t stride,
                         sp_type inner, sp_type *out);
/* make_hvector (stride in bytes)           type_def.hpp:149 */
sp_status sp_type_hvector(int64_t count, int64_t blocklength,
                          int64_t stride_bytes, sp_type inner, sp_type *out);
/* make_subarray: dim 0 innermost, C order only (type_def.hpp:161-195) */
sp_status sp_type_subarray(int64_t ndims, const int64_t *sizes,
                           const int64_t *subsizes, const int64_t *offsets,
                           sp_type inner, int order, sp_type *out);
/* ---- beyond the reference: MPI-3.1 4.1.2-4.1.7 (the paper's future work,
 * PAPER.md:1164; the reference has no indexed/struct/resized types).
 * Displacements must be nonnegative. A type whose blocks are one
 * arithmetic progression of equal blocks of one member type canonicalises
 * to a StridedBlock like the constructors above; any other commits to the
 * block-list form (SP_FORM_UNSUPPORTED, executed by the device run-table
 * kernel in MPI typemap order; unpack allowed unless bytes repeat).
 * Struct extents get no alignment padding: resize to set one. */
/* MPI_Type_indexed (displacements in inner extents) */
sp_status sp_type_indexed(int64_t count, const int64_t *blocklens,
                          const int64_t *displs, sp_type inner, sp_type *out);
/* MPI_Type_create_hindexed (displacements in bytes) */
sp_status sp_type_hindexed(int64_t count, const int64_t *blocklens,
                           const int64_t *displs_bytes, sp_type inner,
                           sp_type *out);
/* MPI_Type_create_indexed_block / _hindexed_block */
sp_status sp_type_indexed_block(int64_t count, int64_t blocklen,
                                const int64_t *displs, sp_type inner,
                                sp_type *out);
sp_status sp_type_hindexed_block(int64_t count, int64_t blocklen,
                                 const int64_t *displs_bytes, sp_type inner,
                                 sp_type *out);
/* MPI_Type_create_struct */
sp_status sp_type_struct(int64_t count, const int64_t *blocklens,
                         const int64_t *displs_bytes, const sp_type *types,
                         sp_type *out);
/* MPI_Type_create_resized: same bytes, new lower bound and extent */
sp_status sp_type_resized(sp_type inner, int64_t lb, int64_t extent,
                          sp_type *out);
/* MPI_Type_get_extent's lb (0 for every reference constructor) */
sp_status sp_type_lb(sp_type t, int64_t *lb);
/* releases the handle; definitions that wrap it keep their own reference */
sp_status sp_type_free(sp_type t);
/* type_size                  type_def.hpp:198 */
sp_status sp_type_size(sp_type t, int64_t *size);
/* type_extent                type_def.hpp:221 */
sp_status sp_type_extent(sp_type t, int64_t *extent);
/* flatten_oracle (block_list.hpp:123-126; CLI `flatten`, cli.hpp:98-108):
 * the definition's byte runs, sorted, abutting/overlapping runs merged
 * (normalize_blocks, block_list.hpp:44-61). *n = run count; the arrays are
 * filled when cap >= *n; *overlap = 1 if some byte is described twice. */
sp_status sp_type_flatten(sp_type t, int64_t *offsets, int64_t *lengths,
                          int64_t cap, int64_t *n, int *overlap);
/* parse_type_file (typefile.hpp:131-258): parses a type-description text
 * and returns a NEW uncommitted handle for the committed statement's type;
 * `name` (if cap > 0) receives its name. Diagnostics are SP_ERR_PARSE with
 * "line N: ..." messages (sp_last_error). */
sp_status sp_typefile_parse(const char *text, sp_type *out, char *name,
                            int64_t name_cap);

/* ---- commit: commit.hpp:51 (commit_type) / :87 (TypeRegistry::commit) -
 * Canonicalises the definition (translate -> fold/elide/flatten/sort to a
 * fixpoint -> StridedBlock -> plan), decides overlap exactly, and records
 * the execution plan. Idempotent. O(definition tree), not O(size). */
sp_status sp_type_commit(sp_type t);

enum { SP_FORM_STRIDED = 0, SP_FORM_EMPTY = 1, SP_FORM_UNSUPPORTED = 2 }; /* commit.hpp:21 */
enum { SP_STRATEGY_GRIDZ = 0, SP_STRATEGY_ITERATE = 1 };                   /* plan.hpp:13 */

/* CommittedType (commit.hpp:30-43) + PackPlan (plan.hpp:27-44) */
typedef struct {
  int64_t form;
  int64_t size;        /* described bytes per object */
  int64_t extent;      /* placement span for consecutive objects */
  int64_t span;        /* one past the last described byte */
  int64_t overlapping; /* some byte described twice */
  int64_t ndims;       /* StridedBlock dims (0 unless form == STRIDED) */
  int64_t start;       /* StridedBlock start */
  int64_t word;        /* PackPlan.word (reference select_word_size) */
  int64_t block[3], grid[3], strategy; /* PackPlan block/grid/count strategy */
  int64_t n_fallback_runs; /* definition-order runs (Unsupported form) */
  int64_t simplify_rounds; /* fixpoint rounds (canon.hpp:117), -1 if n/a */
} sp_type_info;

/* Fills info and, when cap >= ndims, the StridedBlock counts/strides
 * (strided_block.hpp:17-46). Requires a committed type. */
sp_status sp_type_query(sp_type t, sp_type_info *info, int64_t *counts,
                        int64_t *strides, int64_t cap);

/* ---- pack / unpack: pack.hpp:99 / pack.hpp:143 ---------------------- *
 * pack: gathers `incount` objects laid out at src + j*extent into
 * dst + *position in canonical order (object-major, dimension 1 fastest,
 * exactly the reference executor's byte order) and advances *position by
 * incount*size. Error precedence follows pack.hpp:102-126:
 * INVALID_ARGUMENT (incount < 1, position < 0), BUFFER_TOO_SMALL (dst),
 * EMPTY no-op, BUFFER_TOO_SMALL (src), UNSUPPORTED (fallback disabled).
 * src_bytes/dst_bytes are the caller's buffer sizes (UINT64_MAX = unknown).
 * unpack follows pack.hpp:146-159: INVALID_ARGUMENT, OVERLAPPING_LAYOUT,
 * BUFFER_TOO_SMALL (src), EMPTY no-op, BUFFER_TOO_SMALL (dst). Bytes of dst
 * outside the layout are never written. */
sp_status sp_pack(const void *src, uint64_t src_bytes, sp_type t,
                  int64_t incount, void *dst, uint64_t dst_bytes,
                  int64_t *position, void *stream);
sp_status sp_unpack(const void *src, uint64_t src_bytes, int64_t *position,
                    sp_type t, int64_t outcount, void *dst, uint64_t dst_bytes,
                    void *stream);

/* Options mirror PackOptions (pack.hpp:15-18) plus test/bench knobs. */
enum {
  SP_KERNEL_AUTO = 0,
  SP_KERNEL_WORDS = 1,    /* generic N-D word kernel */
  SP_KERNEL_SMALLROW = 2, /* rows of 1/2/4/8 B gathered into 16 B stores */
  SP_KERNEL_BLOCKLIST = 3,/* device block-list (definition-order runs) */
  SP_KERNEL_TMA = 4,      /* tensor-map box staged through shared memory */
  SP_KERNEL_WORDS64 = 5,  /* generic kernel with 64-bit indexing (chosen
                             automatically beyond 2^32 words or rows) */
  SP_KERNEL_BATCH = 6,    /* many jobs in one launch (sp_batch_*) */
  SP_KERNEL_SHIFT = 7,    /* misaligned rows >= 16 B: aligned 16-B packed
                             chunks assembled by funnel shifts */
  SP_KERNEL_DMA = 8       /* no kernel: the copy engines move the rows as
                             pitched 3-D copies (cudaMemcpy3DAsync; at most
                             4096 calls, strided forms only) -- the paper's
                             "GPU DMA engine for non-contiguous data" */
};
typedef struct {
  int allow_fallback; /* PackOptions.allow_fallback (default 1) */
  int kernel;         /* SP_KERNEL_* (0 = auto) */
  int force_word;     /* 0 = auto, else 1/2/4/8/16 (must be legal) */
} sp_pack_options;
sp_status sp_pack_ex(const void *src, uint64_t src_bytes, sp_type t,
                     int64_t incount, void *dst, uint64_t dst_bytes,
                     int64_t *position, void *stream,
                     const sp_pack_options *opt);
sp_status sp_unpack_ex(const void *src, uint64_t src_bytes, int64_t *position,
                       sp_type t, int64_t outcount, void *dst,
                       uint64_t dst_bytes, void *stream,
                       const sp_pack_options *opt);

/* What the last pack or unpack call on this thread launched. */
typedef struct {
  int64_t kernel;      /* SP_KERNEL_* actually used, 0 = no launch (empty) */
  int64_t word;        /* word size of the launch */
  int64_t launches;    /* kernels enqueued by that call */
  int64_t grid, block; /* launch shape of the main kernel */
  int64_t staged;      /* 1 if pageable host memory was staged */
} sp_launch_info;
sp_status sp_last_launch(sp_launch_info *out);
/* total kernels this library enqueued in this process */
int64_t sp_kernel_launch_count(void);

/* ---- batches: many pack (or unpack) jobs in ONE kernel launch -------- *
 * Replaces a loop of pack() calls over one buffer (halo.hpp:227-235: 26
 * region packs into one send buffer) with a persistent plan. Each job has
 * the arguments of sp_pack (unpack == 0) or sp_unpack (unpack == 1) and is
 * validated at creation in the same precedence; the plan binds the
 * pointers, which must be device memory, pinned host memory or peer-GPU
 * memory mapped through CUDA IPC (pack-to-peer). Empty types are skipped;
 * forms without a strided canon are rejected (SP_ERR_UNSUPPORTED). */
typedef struct {
  const void *src;
  uint64_t src_bytes;
  sp_type type;
  int64_t count;
  void *dst;
  uint64_t dst_bytes;
  int64_t position; /* offset into the packed buffer (dst for pack, src for unpack) */
} sp_batch_job;
typedef struct sp_batch_s *sp_batch;
sp_status sp_batch_create(const sp_batch_job *jobs, int64_t n, int unpack,
                          sp_batch *out);
sp_status sp_batch_execute(sp_batch b, void *stream);
/* Typed copies in ONE launch (no packed intermediate): byte k of `count`
 * objects of `src_type` at src (pack order) is stored at byte k of
 * `dst_count` objects of `dst_type` at dst (unpack order) -- the pack of
 * pack.hpp:99 fused with the unpack of pack.hpp:143 that MPI_Sendrecv with
 * two datatypes, a self-send, or MPI_Neighbor_alltoallw would run. Both
 * sides must describe the same byte count (SP_ERR_INVALID_ARGUMENT), the
 * destination must not overlap itself (SP_ERR_OVERLAPPING_LAYOUT), the
 * buffers must cover (count-1)*extent+span (SP_ERR_BUFFER_TOO_SMALL), and
 * both types need a strided form (SP_ERR_UNSUPPORTED). dst may be peer-GPU
 * memory mapped through CUDA IPC (copy-to-peer over NVLink). */
typedef struct {
  const void *src;
  uint64_t src_bytes;
  sp_type src_type;
  int64_t src_count;
  void *dst;
  uint64_t dst_bytes;
  sp_type dst_type;
  int64_t dst_count;
} sp_copy_job;
/* one typed copy, one launch, no descriptor upload (the job travels as a
 * kernel parameter): MPI_Sendrecv of two datatypes within one process, or
 * a send to self. Buffers: device, pinned or peer-mapped memory. A
 * block-list (irregular) layout on one side needs one dense run on the
 * other (it runs as a run-table pack or unpack); two irregular sides are
 * SP_ERR_UNSUPPORTED. */
sp_status sp_copy(const sp_copy_job *job, void *stream);
sp_status sp_copy_batch_create(const sp_copy_job *jobs, int64_t n,
                               sp_batch *out);
/* payload bytes one execution moves */
sp_status sp_batch_bytes(sp_batch b, int64_t *bytes);
sp_status sp_batch_free(sp_batch b);

/* ---- send-method model: perf_model.hpp / profile_io.hpp ------------- *
 * A MachineProfile (perf_model.hpp:36-45) holds four transfer curves
 * (bytes -> seconds) and four pack surfaces ((object, block) -> seconds).
 * The model (paper Eqs. 1-3) is
 *   device  = gpu_pack + gpu_gpu + gpu_unpack
 *   oneshot = host_pack + cpu_cpu + host_unpack
 *   staged  = gpu_pack + d2h + cpu_cpu + h2d + gpu_unpack
 * with log-log interpolation clamped at the sampled range. */
typedef struct sp_profile_s *sp_profile;
typedef struct sp_model_cache_s *sp_model_cache;
enum { SP_CURVE_CPU_CPU = 0, SP_CURVE_GPU_GPU = 1, SP_CURVE_D2H = 2, SP_CURVE_H2D = 3 };
enum { SP_SURF_GPU_PACK = 0, SP_SURF_GPU_UNPACK = 1, SP_SURF_HOST_PACK = 2, SP_SURF_HOST_UNPACK = 3,
       /* B200 extension (optional in the profile text, written only when
        * measured): one typed-copy launch from the probe layout to the same
        * layout on this GPU / on a peer GPU over NVLink -- the DIRECT method */
       SP_SURF_GPU_DIRECT = 4, SP_SURF_GPU_DIRECT_PEER = 5 };
enum { SP_METHOD_ONESHOT = 0, SP_METHOD_DEVICE = 1, SP_METHOD_STAGED = 2, /* MethodChoice perf_model.hpp:46 */
       SP_METHOD_DIRECT = 3 /* runtime only (sp_rt_*): the device path with the
                               pack, NVLink transfer and unpack fused into one
                               typed-copy kernel into the receiver's buffer */ };

sp_status sp_profile_create(sp_profile *out);
/* load_profile           profile_io.hpp:88 (text) / :166 (file) */
sp_status sp_profile_parse(const char *text, sp_profile *out);
sp_status sp_profile_load(const char *path, sp_profile *out);
/* save_profile           profile_io.hpp:174; *len = text length; buf may be
 * NULL to query the size (cap must exceed *len) */
sp_status sp_profile_save(sp_profile p, const char *header, char *buf,
                          int64_t cap, int64_t *len);
sp_status sp_profile_free(sp_profile p);
sp_status sp_profile_set_curve(sp_profile p, int curve, const double *size,
                               const double *time, int64_t n);
/* time is row-major [nobj][nblk] */
sp_status sp_profile_set_surface(sp_profile p, int surf, const double *object,
                                 int64_t nobj, const double *block,
                                 int64_t nblk, const double *time);
/* interp_1d              perf_model.hpp:113 */
sp_status sp_interp_1d(sp_profile p, int curve, double size, double *t);
/* interp_2d              perf_model.hpp:125 */
sp_status sp_interp_2d(sp_profile p, int surf, double object, double block,
                       double *t);
/* t_device/t_oneshot/t_staged  perf_model.hpp:139-159 (NULL outputs ok) */
sp_status sp_model_times(sp_profile p, int64_t object_size, int64_t block_size,
                         double *t_device, double *t_oneshot, double *t_staged);
/* choose_method          perf_model.hpp:163 */
sp_status sp_choose_method(sp_profile p, int64_t object_size,
                           int64_t block_size, int *method);
/* B200 extension of choose_method: Eqs. 1-3 plus Eq. 4 (DIRECT = the
 * gpu_direct surface when dst_kind = 1, a device buffer on this GPU, or the
 * gpu_direct_peer surface when dst_kind = 2, a device buffer on a peer GPU;
 * never for dst_kind = 0, host memory, or an unmeasured surface). Ties
 * prefer DIRECT, then the reference's order. times (NULL ok) = device,
 * one-shot, staged, direct (+inf when DIRECT is not a candidate). */
sp_status sp_choose_method_b200(sp_profile p, int64_t object_size,
                                int64_t block_size, int dst_kind, int *method,
                                double times[4]);
/* ModelCache             perf_model.hpp:184-229 (the profile must outlive
 * nothing: the cache keeps its own reference) */
sp_status sp_model_cache_create(sp_profile p, sp_model_cache *out);
sp_status sp_model_cache_choose(sp_model_cache c, int64_t object_size,
                                int64_t block_size, int *method);
sp_status sp_model_cache_free(sp_model_cache c);

/* ---- 3D halo exchange: halo.hpp ------------------------------------- *
 * HaloConfig (halo.hpp:25-30): periodic rank grid, interior cells per rank
 * per axis, stencil radius, payload bytes per cell. */
typedef struct {
  int64_t ranks[3];
  int64_t interior[3];
  int64_t radius;
  int64_t element_bytes;
} sp_halo_config;

/* build_halo_types (halo.hpp:98-130): the 26 (send, recv) byte-normalised
 * subarray types over the padded allocation, committed, in direction order
 * z, y, x in {-1,0,1}. dir[k*3 + a] is the direction on axis a (x,y,z);
 * cells[k] the grid points per region. Handles are owned by the caller. */
sp_status sp_halo_types(const sp_halo_config *cfg, sp_type send[26],
                        sp_type recv[26], int dir[78], int64_t cells[26]);
/* rank index of the neighbour of `rank` in direction dir (periodic) */
sp_status sp_halo_neighbor(const sp_halo_config *cfg, int64_t rank,
                           const int dir[3], int64_t *neighbor);
/* fill_cell pattern (halo.hpp:152-164) into rank's padded allocation
 * (device memory): interior from the global pattern, ghosts 0xee */
sp_status sp_halo_fill(const sp_halo_config *cfg, int64_t rank, void *alloc,
                       void *stream);
/* exact check of every padded cell against the wrapped global pattern
 * (halo.hpp:264-285); synchronises `stream`; *mismatched = bad cells */
sp_status sp_halo_verify(const sp_halo_config *cfg, int64_t rank,
                         const void *alloc, void *stream, int64_t *mismatched);

enum { SP_HALO_FUSED = 0, /* pack-to-peer: one batch stores every segment
                             into the receiver's buffer */
       SP_HALO_COPY = 1,  /* pack, per-segment copies, unpack (the
                             reference's three phases) */
       SP_HALO_FUSED_ASYNC = 2, /* distributed plans only: pack-to-peer with
                             in-kernel completion flags (acquire/release on
                             IPC-mapped peer memory); the iteration is
                             ordered on the GPU, no host barrier between
                             pack and unpack */
       SP_HALO_DIRECT = 3 /* ghost writes: one typed-copy launch moves every
                             send region straight into the receiving rank's
                             ghost cells (no packed segment, no unpack); in
                             distributed plans ordered by in-kernel flags */ };
/* ExchangeReport (halo.hpp:132-138) + measured device times */
typedef struct {
  double pack_seconds, alltoallv_seconds, unpack_seconds; /* modeled */
  int64_t verified, bytes_moved, mismatched_cells;
  double measured_pack_seconds, measured_exchange_seconds,
      measured_unpack_seconds; /* CUDA-event averages over iters */
} sp_halo_report;
/* run_exchange (halo.hpp:172): every rank of the grid on the CURRENT
 * device; profile may be NULL (no modeled times). */
sp_status sp_halo_run(const sp_halo_config *cfg, sp_profile profile,
                      int method, int iters, sp_halo_report *out);

/* ---- node-local runtime (the "system MPI" this image lacks) ---------- *
 * One process per GPU. A POSIX shared-memory segment named after `job`
 * carries bootstrap, barriers and control mailboxes; CUDA IPC maps peer
 * device memory (kernels store into a peer's HBM over NVLink); each rank
 * owns a device receive window and a shared pinned host region.
 * device < 0 initialises the control plane only (no CUDA calls). */
sp_status sp_rt_init(int rank, int size, const char *job, int device,
                     int64_t window_bytes, int64_t host_bytes);
sp_status sp_rt_finalize(void);
sp_status sp_rt_rank(int *rank);
sp_status sp_rt_size(int *size);
sp_status sp_rt_barrier(void);
/* small control payloads (<= 16 bytes) between ranks, matched by tag */
sp_status sp_rt_host_send(int dst, int tag, const void *data, int64_t bytes);
sp_status sp_rt_host_recv(int src, int tag, void *data, int64_t cap,
                          int64_t *bytes);
/* collective: peers[r] = rank r's `local` device pointer mapped here */
sp_status sp_rt_exchange_ptr(void *local, void **peers);
/* the runtime's stream (cudaStream_t) on which sends, batches and halo
 * plans are enqueued; work the caller orders before them goes here */
sp_status sp_rt_stream(void **stream);
/* the send-method model used by sp_rt_send when method < 0 */
sp_status sp_rt_set_profile(sp_profile p);
sp_status sp_rt_choose(sp_type t, int64_t count, int *method);
/* MPI_Send / MPI_Recv of `count` objects of a committed type between two
 * ranks: rendezvous, then DEVICE (pack kernel stores into the receiver's
 * HBM window through IPC, the receiver unpacks), ONESHOT (pack kernel
 * stores into the receiver's pinned host region) or STAGED (device pack,
 * D2H, H2D, unpack); DIRECT = the device path where the receiver, when its
 * buffer is device memory, publishes buffer + canonical geometry and the
 * sender runs one typed-copy kernel into it (falls back to DEVICE
 * otherwise). method < 0 = model-selected (Eqs. 1-3) with DIRECT offered to
 * the receiver, the model's choice being the fallback when the receive
 * buffer is not device memory. Messages above two chunks (sp_rt_set_chunk,
 * default 4 MiB) are
 * pipelined chunk by chunk. source/tag < 0 match any. status = {source,
 * tag, bytes, method used}. Blocking; the buffers must be device-accessible
 * (or pinned / pageable host memory, staged by the engine). */
sp_status sp_rt_send(const void *buf, uint64_t buf_bytes, int64_t count,
                     sp_type t, int dest, int tag, int method,
                     int *used_method);
sp_status sp_rt_recv(void *buf, uint64_t buf_bytes, int64_t count, sp_type t,
                     int source, int tag, int64_t status[4]);
/* MPI_Isend / MPI_Irecv / MPI_Test / MPI_Wait: the same protocol as
 * non-blocking requests. Every runtime call (and sp_rt_barrier) progresses
 * all pending requests. sp_rt_test sets *done and, once done, fills status
 * and frees the request; sp_rt_wait blocks until done. The error of a
 * failed request (e.g. truncation) is returned by test/wait. */
typedef uint64_t sp_request;
sp_status sp_rt_isend(const void *buf, uint64_t buf_bytes, int64_t count,
                      sp_type t, int dest, int tag, int method,
                      sp_request *req);
sp_status sp_rt_irecv(void *buf, uint64_t buf_bytes, int64_t count, sp_type t,
                      int source, int tag, sp_request *req);
sp_status sp_rt_test(sp_request req, int *done, int64_t status[4]);
sp_status sp_rt_wait(sp_request req, int64_t status[4]);
/* packed bytes per pipelined chunk (multiple of 16; TEMPI_CHUNK env) */
sp_status sp_rt_set_chunk(int64_t bytes);

/* MPI_Neighbor_alltoallv over a distributed graph (collective over every
 * runtime rank): block i (sendcounts[i] objects of sendtype at
 * sdispls[i]*extent) goes to dests[i]; block j from sources[j] lands at
 * rdispls[j]*extent(recvtype). ONE batch launch per rank packs every block
 * with sendtype straight into the receiving rank's buffer through CUDA IPC.
 * With a dense-bytes recvtype (MPI_PACKED/MPI_BYTE-like) the blocks are
 * packed into the receivers' buffers; with a strided recvtype each block is
 * a typed copy straight to its strided place (the alltoallw path). The k-th
 * edge to a rank matches that rank's k-th edge from this one. No host barrier: a
 * rank announces each call to its in-neighbours through shared memory,
 * waits only for its out-neighbours' announcements, and the data kernel
 * publishes per-pair READY counters to the receivers and waits (last CTA)
 * for its senders', so the call returns when its own blocks have landed. */
sp_status sp_rt_neighbor_alltoallv(const void *sendbuf,
                                   const int64_t *sendcounts,
                                   const int64_t *sdispls, int64_t outdegree,
                                   const int *dests, sp_type sendtype,
                                   void *recvbuf, const int64_t *recvcounts,
                                   const int64_t *rdispls, int64_t indegree,
                                   const int *sources, sp_type recvtype);
/* MPI_Neighbor_alltoallw (collective): per-edge datatypes on both sides and
 * BYTE displacements. Each rank publishes, per in-edge, its receive buffer
 * and the canonical geometry of recvtypes[j]; block i (sendcounts[i]
 * objects of sendtypes[i] at sendbuf + sdispls[i]) is then stored by ONE
 * typed-copy launch per rank straight to its strided place in the
 * receiver's buffer (recvbuf + rdispls[j], recvtypes[j]) -- no packed
 * intermediate, no unpack. Send and receive of an edge must describe the
 * same byte count; receive types need a strided non-overlapping form. */
sp_status sp_rt_neighbor_alltoallw(const void *sendbuf,
                                   const int64_t *sendcounts,
                                   const int64_t *sdispls,
                                   const sp_type *sendtypes, int64_t outdegree,
                                   const int *dests, void *recvbuf,
                                   const int64_t *recvcounts,
                                   const int64_t *rdispls,
                                   const sp_type *recvtypes, int64_t indegree,
                                   const int *sources);

/* persistent neighbour alltoallw (MPI-4.0 MPI_Neighbor_alltoallw_init;
 * collective): the typed-copy batch is built once against the receivers'
 * layouts, each start is ONE launch carrying the halo plans' device
 * protocol (no host entry protocol), and starts capture into CUDA graphs.
 * Strided types only (SP_ERR_UNSUPPORTED otherwise, on every rank). The
 * buffers stay bound to the plan. start enqueues on sp_rt_stream; test /
 * wait complete a start (this rank's sends done, its receives landed). */
typedef struct sp_nbr_plan_s *sp_nbr_plan;
sp_status sp_rt_neighbor_alltoallw_init(const void *sendbuf, const int64_t *sendcounts, const int64_t *sdispls,
                                        const sp_type *sendtypes, int64_t outdegree, const int *dests,
                                        void *recvbuf, const int64_t *recvcounts, const int64_t *rdispls,
                                        const sp_type *recvtypes, int64_t indegree, const int *sources,
                                        sp_nbr_plan *out);
sp_status sp_nbr_plan_start(sp_nbr_plan p);
sp_status sp_nbr_plan_test(sp_nbr_plan p, int *done);
sp_status sp_nbr_plan_wait(sp_nbr_plan p);
sp_status sp_nbr_plan_free(sp_nbr_plan p);

/* distributed halo exchange: one rank per process (grid size == runtime
 * size); `alloc` is this rank's padded allocation on its device. */
typedef struct sp_halo_plan_s *sp_halo_plan;
sp_status sp_halo_plan_create(const sp_halo_config *cfg, void *alloc,
                              int method, sp_halo_plan *out);
/* collective; times = {pack, exchange, unpack, iteration} seconds (the call
 * then waits for the iteration). With times == NULL the device-ordered
 * methods (DIRECT, FUSED_ASYNC) only enqueue on the runtime stream
 * (sp_rt_stream): iterations pipeline on the GPU and work the caller
 * enqueues on that stream sees complete ghost shells. */
sp_status sp_halo_plan_exchange(sp_halo_plan p, double times[4]);
sp_status sp_halo_plan_free(sp_halo_plan p);

#ifdef __cplusplus
}
#endif
#endif /* STRIDEPACK_B200_H */
