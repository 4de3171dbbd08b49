// interpose.cpp -- libtempi_interpose.so: TEMPI as a PMPI interposer over a
// system MPI.
//
// Link order `-ltempi_interpose -lmpi`, or LD_PRELOAD=libtempi_interpose.so
// under an unmodified MPI program. This library defines only the MPI_* entry
// points TEMPI accelerates; every other MPI_* symbol resolves to the system
// MPI as usual, and inside the intercepted calls the system MPI is reached
// through dlsym(RTLD_NEXT, "PMPI_*") -- the profiling interface, so the
// system library needs no change and never calls back into this one.
//
// What is accelerated (everything else is forwarded untouched):
//  * datatypes: every constructor is forwarded first (the system MPI owns
//    the handle), then mirrored as an engine type through the C-ABI
//    (include/stridepack_b200.h) and canonicalised at MPI_Type_commit
//    (commit.hpp:51). A constructor the engine rejects (e.g. a negative
//    displacement) leaves the handle un-mirrored: the system MPI handles it;
//  * MPI_Pack / MPI_Unpack with a device or pinned buffer on either side:
//    the sm_100a pack/unpack kernels (pack.hpp:99, :143);
//  * MPI_Send / Isend / Recv / Irecv / Sendrecv of a non-contiguous mirrored
//    type in device memory: the message travels as MPI_BYTE of its packed
//    bytes (the MPI type signature of a homogeneous system, so a peer without
//    the interposer receives it with the original type), through a device,
//    one-shot (pinned) or staged buffer picked per message by the
//    performance model (perf_model.hpp:139-179; Eqs. 1-3, the reference's
//    three methods -- DIRECT needs the engine's own transport and is not a
//    candidate here);
//  * MPI_Neighbor_alltoallv / alltoallw and MPI_Alltoallv / Alltoallw with
//    mirrored types on device buffers: all segments of a side packed
//    (unpacked) by ONE batched launch around a single MPI_BYTE exchange of
//    the system MPI.
// TEMPI_CUDA_AWARE=0 declares a system MPI that cannot read device memory:
// device-resident packed messages are then staged through pinned memory.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "mpi.h"
#include "stridepack_b200.h"

namespace {

// the next definition of a PMPI_* symbol after this library (the system MPI)
template <class F> F next_sym(const char *name) {
  void *p = dlsym(RTLD_NEXT, name);
  if (!p) {
    std::fprintf(stderr, "tempi-interpose: the system MPI does not export %s\n", name);
    std::abort();
  }
  return reinterpret_cast<F>(p);
}
#define REAL(fn) (*([] { static const auto f = next_sym<decltype(&MPI_##fn)>("PMPI_" #fn); return f; }()))
// a PMPI_* an older system MPI may lack (MPI-4 calls): null when absent
#define REAL_OPT(fn)                                                                                             \
  ([] {                                                                                                          \
    static const auto f = reinterpret_cast<decltype(&MPI_##fn)>(dlsym(RTLD_NEXT, "PMPI_" #fn));                 \
    return f;                                                                                                    \
  }())

enum class Mem { Device, Pinned, Pageable };

Mem mem_kind(const void *p) {
  cudaPointerAttributes a{};
  if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return Mem::Pageable;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return Mem::Device;
  return a.type == cudaMemoryTypeHost ? Mem::Pinned : Mem::Pageable;
}

struct Mirror {
  sp_type h = 0;
  bool committed = false;
  int64_t size = 0, extent = 0, span = 0, block = 0;
  bool contiguous = false; // one dense run per object and objects abut
};

// a scratch buffer reused across calls (grow-only, one per kind and role)
struct Scratch {
  void *p = nullptr;
  size_t cap = 0;
  bool pinned = false;
  void *get(size_t n) {
    if (n <= cap) return p;
    release();
    cap = std::max<size_t>(n, 1 << 20);
    if ((pinned ? cudaMallocHost(&p, cap) : cudaMalloc(&p, cap)) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      cap = 0;
    }
    return p;
  }
  void release() {
    if (p) pinned ? cudaFreeHost(p) : cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// per-request message buffers, recycled: a non-blocking message takes one
// at Isend/Irecv and returns it at completion (cudaMalloc / cudaMallocHost
// on every request would cost more than the pack itself)
class Pool {
 public:
  explicit Pool(bool pinned) : pinned_(pinned) {}
  void *take(size_t n) {
    n = std::max<size_t>(n, 1);
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto it = free_.lower_bound(n);
      if (it != free_.end() && it->first <= 2 * n) { // no more than 2x waste
        void *p = it->second;
        const size_t have = it->first;
        cached_ -= have;
        free_.erase(it);
        size_[p] = have;
        return p;
      }
    }
    void *p = nullptr;
    if ((pinned_ ? cudaMallocHost(&p, n) : cudaMalloc(&p, n)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    std::lock_guard<std::mutex> lk(mu_);
    size_[p] = n;
    return p;
  }
  void give(void *p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu_);
    const size_t n = size_[p];
    size_.erase(p);
    free_.emplace(n, p);
    cached_ += n;
    while (cached_ > kCap && !free_.empty()) { // drop the largest first
      auto last = std::prev(free_.end());
      cached_ -= last->first;
      pinned_ ? cudaFreeHost(last->second) : cudaFree(last->second);
      free_.erase(last);
    }
  }
  void clear() {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto &kv : free_) pinned_ ? cudaFreeHost(kv.second) : cudaFree(kv.second);
    free_.clear();
    cached_ = 0;
  }

 private:
  static constexpr size_t kCap = size_t{1} << 30; // idle bytes kept per pool
  const bool pinned_;
  std::mutex mu_;
  std::multimap<size_t, void *> free_;
  std::unordered_map<void *, size_t> size_;
  size_t cached_ = 0;
};

// the packed copy of one non-blocking message, alive until its request completes
struct Pending {
  bool recv = false;
  void *dev = nullptr, *host = nullptr; // owned scratch
  void *user = nullptr;
  int64_t count = 0;
  sp_type type = 0;
  int64_t size = 0;
  int method = 0;
};

struct Stats {
  std::atomic<int64_t> commits{0}, packs{0}, unpacks{0}, sends[3], recvs[3], exchanges{0}, forwarded{0};
  Stats() {
    for (auto &s : sends) s = 0;
    for (auto &r : recvs) r = 0;
  }
};

struct BatchKey {
  std::vector<uint64_t> k;
  bool operator<(const BatchKey &o) const { return k < o.k; }
};

// one segment of a neighbour exchange side: `count` objects of `type`
// between the caller's buffer and a packed buffer at `position`
struct Segment {
  const void *src;
  sp_type type;
  int64_t count;
  void *dst;
  int64_t position;
};

struct State {
  std::mutex mu;         // tables
  std::mutex scratch_mu; // the reusable scratch buffers (one blocking call at a time)
  std::unordered_map<MPI_Datatype, Mirror> types;
  std::unordered_map<MPI_Comm, std::pair<int, int>> degree; // comm -> (indegree, outdegree)
  std::unordered_map<MPI_Request, Pending> pending;
  // persistent requests of accelerated types (MPI_Send_init / MPI_Recv_init):
  // their packed message buffers live until MPI_Request_free
  std::unordered_map<MPI_Request, Pending> persist;
  // persistent neighbour collectives (MPI-4): packed segments on both
  // sides, packed at MPI_Start and unpacked at completion
  struct Coll {
    std::vector<Segment> pack, unpack;
    void *sp = nullptr, *rp = nullptr;
    bool pinned = false, started = false;
  };
  std::unordered_map<MPI_Request, Coll> colls;
  // mirrors still named by a pending receive, and the ones among them whose
  // MPI type was freed (MPI lets a pending operation outlive its datatype):
  // released when the last such receive completes
  std::unordered_map<sp_type, int> in_flight;
  std::unordered_set<sp_type> retired;
  std::map<BatchKey, sp_batch> batches;
  std::unordered_map<int, cudaStream_t> streams; // one per device the application uses
  sp_profile profile = nullptr;
  sp_model_cache model = nullptr;
  int forced = -1;
  bool cuda_aware = true, gpu = false, stats_on = false;
  Scratch dev_s, dev_r, host_s{nullptr, 0, true}, host_r{nullptr, 0, true};
  Pool dev_pool{false}, host_pool{true};
  Stats st;
};

State &S() {
  static State s;
  return s;
}

int to_mpi(sp_status st) {
  switch (st) {
  case SP_OK: return MPI_SUCCESS;
  case SP_ERR_BUFFER_TOO_SMALL: return MPI_ERR_TRUNCATE;
  case SP_ERR_INVALID_LAYOUT:
  case SP_ERR_OVERLAPPING_LAYOUT:
  case SP_ERR_INVALID_HANDLE: return MPI_ERR_TYPE;
  case SP_ERR_INVALID_ARGUMENT:
  case SP_ERR_UNSUPPORTED_ORDER: return MPI_ERR_ARG;
  case SP_ERR_UNSUPPORTED: return MPI_ERR_UNSUPPORTED_OPERATION;
  default: return MPI_ERR_INTERN;
  }
}

#define TRY(expr)                                                                                                \
  do {                                                                                                           \
    const sp_status _st = (expr);                                                                                \
    if (_st != SP_OK) {                                                                                          \
      if (std::getenv("TEMPI_VERBOSE")) std::fprintf(stderr, "tempi-interpose: %s: %s\n", #expr, sp_last_error()); \
      return to_mpi(_st);                                                                                        \
    }                                                                                                            \
  } while (0)

// the interposer's stream on the application's CURRENT device (an
// application may select its GPU after MPI_Init). A blocking stream: the
// kernels of an MPI call run after everything the application issued
// before it on the legacy default stream (a cudaMemset of the receive
// buffer, say), as users of a CUDA-aware MPI expect.
cudaStream_t cur_stream() {
  int d = 0;
  cudaGetDevice(&d);
  std::lock_guard<std::mutex> lk(S().mu);
  cudaStream_t &st = S().streams[d];
  if (!st) cudaStreamCreate(&st);
  return st;
}

int stream_sync() { return cudaStreamSynchronize(cur_stream()) == cudaSuccess ? MPI_SUCCESS : MPI_ERR_INTERN; }

bool mirror_of(MPI_Datatype t, sp_type *h) {
  std::lock_guard<std::mutex> lk(S().mu);
  auto it = S().types.find(t);
  if (it == S().types.end()) return false;
  *h = it->second.h;
  return true;
}

// the message buffers of a non-blocking request's method
bool take_buffers(Pending &p, size_t bytes) {
  if (p.method != SP_METHOD_ONESHOT && !(p.dev = S().dev_pool.take(bytes))) return false;
  if (p.method != SP_METHOD_DEVICE && !(p.host = S().host_pool.take(bytes))) {
    S().dev_pool.give(p.dev);
    p.dev = nullptr;
    return false;
  }
  return true;
}

void give_buffers(Pending &p) {
  S().dev_pool.give(p.dev);
  S().host_pool.give(p.host);
  p.dev = p.host = nullptr;
}

// a committed mirror, or nothing
bool committed(MPI_Datatype t, Mirror *m) {
  std::lock_guard<std::mutex> lk(S().mu);
  auto it = S().types.find(t);
  if (it == S().types.end() || !it->second.committed) return false;
  *m = it->second;
  return true;
}

void record(MPI_Datatype t, sp_type h) {
  std::lock_guard<std::mutex> lk(S().mu);
  auto it = S().types.find(t);
  if (it != S().types.end() && it->second.h) sp_type_free(it->second.h);
  S().types[t] = Mirror{h};
}

// mirror a freshly built system handle when every input has a mirror
template <class Build> int mirror(int rc, MPI_Datatype *out, Build build) {
  if (rc != MPI_SUCCESS) return rc;
  sp_type h = 0;
  if (build(&h) == SP_OK) record(*out, h);
  return rc;
}

// the performance model (Eqs. 1-3) for one message of `count` objects
int choose(const Mirror &m, int64_t count) {
  int method = S().forced;
  if (method == SP_METHOD_DIRECT) method = SP_METHOD_DEVICE; // no fused peer copy over a system MPI
  if (method < 0) {
    method = SP_METHOD_DEVICE;
    if (S().model) sp_model_cache_choose(S().model, m.size * count, m.block, &method);
  }
  if (method == SP_METHOD_DEVICE && !S().cuda_aware) method = SP_METHOD_STAGED;
  return method;
}

// accelerated point-to-point: a committed non-contiguous mirror over device memory
bool accel(MPI_Datatype t, const void *buf, int count, Mirror *m) {
  return S().gpu && count > 0 && committed(t, m) && !m->contiguous && m->size > 0 && mem_kind(buf) == Mem::Device;
}

// pack `count` objects at buf into a message buffer for `method`; *msg is
// the buffer the system MPI sends from
int pack_message(const Mirror &m, const void *buf, int count, int method, void *dev, void *host, void **msg) {
  const int64_t bytes = m.size * count;
  int64_t pos = 0;
  if (method == SP_METHOD_ONESHOT) { // the kernel writes the pinned buffer (zero-copy or chunked DMA)
    TRY(sp_pack(buf, UINT64_MAX, m.h, count, host, bytes, &pos, cur_stream()));
    *msg = host;
  } else {
    TRY(sp_pack(buf, UINT64_MAX, m.h, count, dev, bytes, &pos, cur_stream()));
    *msg = dev;
    if (method == SP_METHOD_STAGED) {
      if (cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, cur_stream()) != cudaSuccess) return MPI_ERR_INTERN;
      *msg = host;
    }
  }
  S().st.packs++;
  S().st.sends[method]++;
  return stream_sync();
}

// unpack a received message of `bytes` into whole objects at buf
int unpack_message(const Mirror &m, void *buf, int64_t bytes, int method, void *dev, void *host) {
  const int64_t n = bytes / m.size;
  if (n == 0) return MPI_SUCCESS;
  int64_t pos = 0;
  if (method == SP_METHOD_ONESHOT) {
    TRY(sp_unpack(host, bytes, &pos, m.h, n, buf, UINT64_MAX, cur_stream()));
  } else {
    if (method == SP_METHOD_STAGED &&
        cudaMemcpyAsync(dev, host, n * m.size, cudaMemcpyHostToDevice, cur_stream()) != cudaSuccess)
      return MPI_ERR_INTERN;
    TRY(sp_unpack(dev, bytes, &pos, m.h, n, buf, UINT64_MAX, cur_stream()));
  }
  S().st.unpacks++;
  S().st.recvs[method]++;
  return stream_sync();
}

// the transfer method of a receive, in the status field this image's mpi.h
// has for it; a vendor MPI_Status has no such field
void report_method(MPI_Status *st, int method) {
#ifdef TEMPI_B200_MPI_H
  st->method = method;
#else
  (void)st;
  (void)method;
#endif
}

// bytes a completed receive of MPI_BYTE delivered, asked of the system MPI
int64_t received(const MPI_Status *st) {
  int n = 0;
  return REAL(Get_count)(st, MPI_BYTE, &n) == MPI_SUCCESS && n != MPI_UNDEFINED ? n : 0;
}

// the buffer a receive of `method` lands in
void *recv_target(int method, void *dev, void *host) { return method == SP_METHOD_DEVICE ? dev : host; }

std::string default_profile_path() {
  Dl_info info{};
  if (dladdr(reinterpret_cast<void *>(&default_profile_path), &info) && info.dli_fname) {
    std::string p(info.dli_fname);
    const auto slash = p.rfind('/');
    if (slash != std::string::npos) return p.substr(0, slash) + "/../profiles/b200.profile";
  }
  return "";
}

int env_int(const char *k, int dflt) {
  const char *v = std::getenv(k);
  return v ? std::atoi(v) : dflt;
}

void setup() {
  State &s = S();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
    cudaGetLastError();
    ndev = 0;
  }
  s.gpu = ndev > 0;
  s.stats_on = std::getenv("TEMPI_INTERPOSE_STATS") != nullptr;
  s.cuda_aware = env_int("TEMPI_CUDA_AWARE", 1) != 0;
  if (const char *m = std::getenv("TEMPI_METHOD")) s.forced = std::atoi(m);
  const std::pair<MPI_Datatype, int> named[] = {{MPI_BYTE, SP_BYTE},   {MPI_CHAR, SP_BYTE},   {MPI_UNSIGNED_CHAR, SP_BYTE},
                                                {MPI_PACKED, SP_BYTE}, {MPI_INT, SP_INT},     {MPI_FLOAT, SP_FLOAT},
                                                {MPI_DOUBLE, SP_DOUBLE}};
  for (auto [t, k] : named) {
    sp_type h = 0;
    if (sp_type_named(k, &h) == SP_OK && sp_type_commit(h) == SP_OK) {
      s.types[t] = Mirror{h, true, 0, 0, 0, 0, true};
      sp_type_size(h, &s.types[t].size);
      s.types[t].extent = s.types[t].span = s.types[t].size;
    }
  }
  if (!s.gpu) return;
  // like the engine's own runtime: local rank r starts on GPU r % ndev
  // (TEMPI_DEVICE overrides); an application that selects another GPU later
  // is followed (cur_stream)
  const int local = env_int("TEMPI_LOCAL_RANK", env_int("LOCAL_RANK", env_int("OMPI_COMM_WORLD_LOCAL_RANK", -1)));
  const int dev = env_int("TEMPI_DEVICE", local >= 0 ? local % ndev : -1);
  if (dev >= 0) cudaSetDevice(dev);
  const std::string prof = std::getenv("TEMPI_PROFILE") ? std::getenv("TEMPI_PROFILE") : default_profile_path();
  if (!prof.empty() && sp_profile_load(prof.c_str(), &s.profile) == SP_OK)
    sp_model_cache_create(s.profile, &s.model);
}

// the pack (or unpack) of every accelerated segment of one exchange side in
// one launch; plans are cached on the call's full argument list
int run_segments(const std::vector<Segment> &segs, bool unpack) {
  if (segs.empty()) return MPI_SUCCESS;
  BatchKey key;
  key.k.push_back(unpack);
  for (const auto &g : segs) {
    key.k.insert(key.k.end(), {reinterpret_cast<uint64_t>(g.src), g.type, static_cast<uint64_t>(g.count),
                               reinterpret_cast<uint64_t>(g.dst), static_cast<uint64_t>(g.position)});
  }
  sp_batch b = nullptr;
  {
    std::lock_guard<std::mutex> lk(S().mu);
    auto it = S().batches.find(key);
    if (it != S().batches.end()) b = it->second;
  }
  if (!b) {
    std::vector<sp_batch_job> jobs;
    for (const auto &g : segs)
      if (g.count > 0) jobs.push_back({g.src, UINT64_MAX, g.type, g.count, g.dst, UINT64_MAX, g.position});
    if (sp_batch_create(jobs.data(), static_cast<int64_t>(jobs.size()), unpack, &b) == SP_OK) {
      std::lock_guard<std::mutex> lk(S().mu);
      if (S().batches.size() > 256) { // a bounded cache: drop everything
        for (auto &kv : S().batches) sp_batch_free(kv.second);
        S().batches.clear();
      }
      S().batches[key] = b;
    } else {
      b = nullptr;
    }
  }
  if (b) {
    TRY(sp_batch_execute(b, cur_stream()));
  } else { // a form without a strided canon (block-list runs): one call per segment
    for (const auto &g : segs) {
      if (g.count <= 0) continue;
      int64_t pos = g.position;
      if (unpack) {
        TRY(sp_unpack(g.src, UINT64_MAX, &pos, g.type, g.count, g.dst, UINT64_MAX, cur_stream()));
      } else {
        TRY(sp_pack(g.src, UINT64_MAX, g.type, g.count, g.dst, UINT64_MAX, &pos, cur_stream()));
      }
    }
  }
  (unpack ? S().st.unpacks : S().st.packs) += static_cast<int64_t>(segs.size());
  return MPI_SUCCESS;
}

// one side of a neighbour exchange: accelerated when the buffer is device
// memory and every segment's type is a committed mirror
struct Side {
  bool accel = false;
  std::vector<Mirror> m;
  std::vector<int> bytes, offs; // packed segment sizes / offsets
  int64_t total = 0;
};

Side plan_side(const void *buf, int n, const int counts[], const MPI_Datatype types[], MPI_Datatype one) {
  Side s;
  if (!S().gpu || n == 0 || mem_kind(buf) != Mem::Device) return s;
  bool any_strided = false;
  for (int i = 0; i < n; ++i) {
    Mirror m;
    if (!committed(types ? types[i] : one, &m)) return s;
    any_strided |= !m.contiguous;
    s.m.push_back(m);
    const int64_t b = m.size * counts[i];
    if (s.total + b > INT32_MAX) return s;
    s.offs.push_back(static_cast<int>(s.total));
    s.bytes.push_back(static_cast<int>(b));
    s.total += b;
  }
  s.accel = any_strided;
  return s;
}

} // namespace

extern "C" {

// ============================================================ runtime
int MPI_Init(int *argc, char ***argv) {
  const int rc = REAL(Init)(argc, argv);
  if (rc == MPI_SUCCESS) setup();
  return rc;
}

int MPI_Init_thread(int *argc, char ***argv, int required, int *provided) {
  const int rc = REAL(Init_thread)(argc, argv, required, provided);
  if (rc == MPI_SUCCESS) setup();
  return rc;
}

int MPI_Finalize(void) {
  State &s = S();
  if (s.stats_on) {
    int rank = 0;
    REAL(Comm_rank)(MPI_COMM_WORLD, &rank);
    char line[512];
    const int n = std::snprintf(
        line, sizeof line,
        "tempi-interpose rank %d: commits %lld packs %lld unpacks %lld sends(oneshot/device/staged) "
        "%lld/%lld/%lld recvs %lld/%lld/%lld exchanges %lld forwarded %lld kernels %lld\n",
        rank, (long long)s.st.commits, (long long)s.st.packs, (long long)s.st.unpacks, (long long)s.st.sends[0],
        (long long)s.st.sends[1], (long long)s.st.sends[2], (long long)s.st.recvs[0], (long long)s.st.recvs[1],
        (long long)s.st.recvs[2], (long long)s.st.exchanges, (long long)s.st.forwarded,
        (long long)sp_kernel_launch_count());
    // one write(2) below PIPE_BUF: lines of concurrent ranks never interleave
    if (n > 0) (void)!write(2, line, static_cast<size_t>(std::min<int>(n, sizeof line - 1)));
  }
  for (auto &kv : s.batches) sp_batch_free(kv.second);
  s.batches.clear();
  for (Scratch *b : {&s.dev_s, &s.dev_r, &s.host_s, &s.host_r}) b->release();
  s.dev_pool.clear();
  s.host_pool.clear();
  if (s.model) sp_model_cache_free(s.model);
  if (s.profile) sp_profile_free(s.profile);
  for (auto &kv : s.streams) cudaStreamDestroy(kv.second);
  s.streams.clear();
  s.model = nullptr;
  s.profile = nullptr;
  return REAL(Finalize)();
}

// ============================================================ datatypes
int MPI_Type_contiguous(int count, MPI_Datatype old, MPI_Datatype *out) {
  return mirror(REAL(Type_contiguous)(count, old, out), out, [&](sp_type *h) -> sp_status {
    sp_type in;
    return mirror_of(old, &in) ? sp_type_contiguous(count, in, h) : SP_ERR_INVALID_HANDLE;
  });
}

int MPI_Type_vector(int count, int bl, int stride, MPI_Datatype old, MPI_Datatype *out) {
  return mirror(REAL(Type_vector)(count, bl, stride, old, out), out, [&](sp_type *h) -> sp_status {
    sp_type in;
    return mirror_of(old, &in) ? sp_type_vector(count, bl, stride, in, h) : SP_ERR_INVALID_HANDLE;
  });
}

int MPI_Type_create_hvector(int count, int bl, MPI_Aint stride, MPI_Datatype old, MPI_Datatype *out) {
  return mirror(REAL(Type_create_hvector)(count, bl, stride, old, out), out, [&](sp_type *h) -> sp_status {
    sp_type in;
    return mirror_of(old, &in) ? sp_type_hvector(count, bl, stride, in, h) : SP_ERR_INVALID_HANDLE;
  });
}

// MPI_ORDER_C lists the slowest dimension first; the engine (like the
// reference, type_def.hpp:75) keeps dimension 0 innermost
int MPI_Type_create_subarray(int nd, const int sizes[], const int subs[], const int starts[], int order,
                             MPI_Datatype old, MPI_Datatype *out) {
  return mirror(REAL(Type_create_subarray)(nd, sizes, subs, starts, order, old, out), out, [&](sp_type *h) -> sp_status {
    sp_type in;
    if (!mirror_of(old, &in) || nd < 1) return SP_ERR_INVALID_HANDLE;
    std::vector<int64_t> sz(nd), sub(nd), off(nd);
    for (int i = 0; i < nd; ++i) {
      const int j = order == MPI_ORDER_C ? nd - 1 - i : i;
      sz[i] = sizes[j];
      sub[i] = subs[j];
      off[i] = starts[j];
    }
    return sp_type_subarray(nd, sz.data(), sub.data(), off.data(), in, SP_ORDER_C, h);
  });
}

int MPI_Type_indexed(int count, const int bl[], const int disp[], MPI_Datatype old, MPI_Datatype *out) {
  return mirror(REAL(Type_indexed)(count, bl, disp, old, out), out, [&](sp_type *h) -> sp_status {
    sp_type in;
    if (!mirror_of(old, &in)) return SP_ERR_INVALID_HANDLE;
    std::vector<int64_t> b(bl, bl + count), d(disp, disp + count);
    return sp_type_indexed(count, b.data(), d.data(), in, h);
  });
}

int MPI_Type_create_hindexed(int count, const int bl[], const MPI_Aint disp[], MPI_Datatype old, MPI_Datatype *out) {
  return mirror(REAL(Type_create_hindexed)(count, bl, disp, old, out), out, [&](sp_type *h) -> sp_status {
    sp_type in;
    if (!mirror_of(old, &in)) return SP_ERR_INVALID_HANDLE;
    std::vector<int64_t> b(bl, bl + count), d(disp, disp + count);
    return sp_type_hindexed(count, b.data(), d.data(), in, h);
  });
}

int MPI_Type_create_indexed_block(int count, int bl, const int disp[], MPI_Datatype old, MPI_Datatype *out) {
  return mirror(REAL(Type_create_indexed_block)(count, bl, disp, old, out), out, [&](sp_type *h) -> sp_status {
    sp_type in;
    if (!mirror_of(old, &in)) return SP_ERR_INVALID_HANDLE;
    std::vector<int64_t> d(disp, disp + count);
    return sp_type_indexed_block(count, bl, d.data(), in, h);
  });
}

int MPI_Type_create_hindexed_block(int count, int bl, const MPI_Aint disp[], MPI_Datatype old, MPI_Datatype *out) {
  return mirror(REAL(Type_create_hindexed_block)(count, bl, disp, old, out), out, [&](sp_type *h) -> sp_status {
    sp_type in;
    if (!mirror_of(old, &in)) return SP_ERR_INVALID_HANDLE;
    std::vector<int64_t> d(disp, disp + count);
    return sp_type_hindexed_block(count, bl, d.data(), in, h);
  });
}

int MPI_Type_create_struct(int count, const int bl[], const MPI_Aint disp[], const MPI_Datatype types[],
                           MPI_Datatype *out) {
  return mirror(REAL(Type_create_struct)(count, bl, disp, types, out), out, [&](sp_type *h) -> sp_status {
    std::vector<sp_type> ts(count);
    for (int i = 0; i < count; ++i)
      if (!mirror_of(types[i], &ts[i])) return SP_ERR_INVALID_HANDLE;
    std::vector<int64_t> b(bl, bl + count), d(disp, disp + count);
    return sp_type_struct(count, b.data(), d.data(), ts.data(), h);
  });
}

int MPI_Type_create_resized(MPI_Datatype old, MPI_Aint lb, MPI_Aint extent, MPI_Datatype *out) {
  return mirror(REAL(Type_create_resized)(old, lb, extent, out), out, [&](sp_type *h) -> sp_status {
    sp_type in;
    return mirror_of(old, &in) ? sp_type_resized(in, lb, extent, h) : SP_ERR_INVALID_HANDLE;
  });
}

// commit.hpp:51: canonicalise once, here, so every later call is a lookup
int MPI_Type_commit(MPI_Datatype *dt) {
  const int rc = REAL(Type_commit)(dt);
  if (rc != MPI_SUCCESS || !dt) return rc;
  std::lock_guard<std::mutex> lk(S().mu);
  auto it = S().types.find(*dt);
  if (it == S().types.end() || it->second.committed) return rc;
  Mirror &m = it->second;
  sp_type_info info{};
  int64_t counts[8] = {0}, strides[8] = {0};
  if (sp_type_commit(m.h) != SP_OK || sp_type_query(m.h, &info, counts, strides, 8) != SP_OK) {
    sp_type_free(m.h);
    S().types.erase(it); // the system MPI keeps handling this type
    return rc;
  }
  m.committed = true;
  S().st.commits++;
  m.size = info.size;
  m.extent = info.extent;
  m.span = info.span;
  m.block = info.form == SP_FORM_STRIDED && info.ndims > 0 ? counts[0] : m.size;
  m.contiguous = info.form == SP_FORM_STRIDED && info.ndims == 1 && info.start == 0 && m.extent == m.size;
  return rc;
}

int MPI_Type_free(MPI_Datatype *dt) {
  if (dt) {
    std::lock_guard<std::mutex> lk(S().mu);
    auto it = S().types.find(*dt);
    if (it != S().types.end()) {
      const sp_type h = it->second.h;
      if (S().in_flight.count(h)) {
        S().retired.insert(h); // a pending receive still unpacks with it
      } else {
        sp_type_free(h);
      }
      S().types.erase(it);
    }
  }
  return REAL(Type_free)(dt);
}

// ============================================================ packing
int MPI_Pack(const void *in, int incount, MPI_Datatype dt, void *out, int outsize, int *position, MPI_Comm comm) {
  Mirror m;
  if (!S().gpu || incount <= 0 || !position || !committed(dt, &m) ||
      (mem_kind(in) == Mem::Pageable && mem_kind(out) == Mem::Pageable)) {
    S().st.forwarded++;
    return REAL(Pack)(in, incount, dt, out, outsize, position, comm);
  }
  if (outsize < 0) return MPI_ERR_ARG;
  int64_t pos = *position;
  TRY(sp_pack(in, UINT64_MAX, m.h, incount, out, static_cast<uint64_t>(outsize), &pos, cur_stream()));
  const int rc = stream_sync();
  S().st.packs++;
  *position = static_cast<int>(pos);
  return rc;
}

int MPI_Unpack(const void *in, int insize, int *position, void *out, int outcount, MPI_Datatype dt, MPI_Comm comm) {
  Mirror m;
  if (!S().gpu || outcount <= 0 || !position || !committed(dt, &m) ||
      (mem_kind(in) == Mem::Pageable && mem_kind(out) == Mem::Pageable)) {
    S().st.forwarded++;
    return REAL(Unpack)(in, insize, position, out, outcount, dt, comm);
  }
  if (insize < 0) return MPI_ERR_ARG;
  int64_t pos = *position;
  TRY(sp_unpack(in, static_cast<uint64_t>(insize), &pos, m.h, outcount, out, UINT64_MAX, cur_stream()));
  const int rc = stream_sync();
  S().st.unpacks++;
  *position = static_cast<int>(pos);
  return rc;
}

// ============================================================ point to point
int MPI_Send(const void *buf, int count, MPI_Datatype dt, int dest, int tag, MPI_Comm comm) {
  Mirror m;
  if (!accel(dt, buf, count, &m) || m.size * count > INT32_MAX) {
    S().st.forwarded++;
    return REAL(Send)(buf, count, dt, dest, tag, comm);
  }
  const int method = choose(m, count);
  const size_t bytes = static_cast<size_t>(m.size * count);
  std::lock_guard<std::mutex> lk(S().scratch_mu);
  void *dev = method != SP_METHOD_ONESHOT ? S().dev_s.get(bytes) : nullptr;
  void *host = method != SP_METHOD_DEVICE ? S().host_s.get(bytes) : nullptr;
  if ((method != SP_METHOD_ONESHOT && !dev) || (method != SP_METHOD_DEVICE && !host)) return MPI_ERR_NO_MEM;
  void *msg = nullptr;
  int rc = pack_message(m, buf, count, method, dev, host, &msg);
  if (rc != MPI_SUCCESS) return rc;
  return REAL(Send)(msg, static_cast<int>(bytes), MPI_BYTE, dest, tag, comm);
}

int MPI_Recv(void *buf, int count, MPI_Datatype dt, int source, int tag, MPI_Comm comm, MPI_Status *status) {
  Mirror m;
  if (!accel(dt, buf, count, &m) || m.size * count > INT32_MAX) {
    S().st.forwarded++;
    return REAL(Recv)(buf, count, dt, source, tag, comm, status);
  }
  const int method = choose(m, count);
  const size_t bytes = static_cast<size_t>(m.size * count);
  std::lock_guard<std::mutex> lk(S().scratch_mu);
  void *dev = method != SP_METHOD_ONESHOT ? S().dev_r.get(bytes) : nullptr;
  void *host = method != SP_METHOD_DEVICE ? S().host_r.get(bytes) : nullptr;
  if ((method != SP_METHOD_ONESHOT && !dev) || (method != SP_METHOD_DEVICE && !host)) return MPI_ERR_NO_MEM;
  MPI_Status st{};
  int rc = REAL(Recv)(recv_target(method, dev, host), static_cast<int>(bytes), MPI_BYTE, source, tag, comm, &st);
  if (rc == MPI_SUCCESS) rc = unpack_message(m, buf, received(&st), method, dev, host);
  report_method(&st, method);
  if (status) *status = st;
  return rc;
}

int MPI_Isend(const void *buf, int count, MPI_Datatype dt, int dest, int tag, MPI_Comm comm, MPI_Request *req) {
  Mirror m;
  if (!req) return MPI_ERR_ARG;
  if (!accel(dt, buf, count, &m) || m.size * count > INT32_MAX) {
    S().st.forwarded++;
    return REAL(Isend)(buf, count, dt, dest, tag, comm, req);
  }
  Pending p;
  p.method = choose(m, count);
  const size_t bytes = static_cast<size_t>(m.size * count);
  if (!take_buffers(p, bytes)) return MPI_ERR_NO_MEM;
  void *msg = nullptr;
  int rc = pack_message(m, buf, count, p.method, p.dev, p.host, &msg);
  if (rc == MPI_SUCCESS) rc = REAL(Isend)(msg, static_cast<int>(bytes), MPI_BYTE, dest, tag, comm, req);
  if (rc != MPI_SUCCESS) {
    give_buffers(p);
    return rc;
  }
  std::lock_guard<std::mutex> lk(S().mu);
  S().pending[*req] = p;
  return MPI_SUCCESS;
}

int MPI_Irecv(void *buf, int count, MPI_Datatype dt, int source, int tag, MPI_Comm comm, MPI_Request *req) {
  Mirror m;
  if (!req) return MPI_ERR_ARG;
  if (!accel(dt, buf, count, &m) || m.size * count > INT32_MAX) {
    S().st.forwarded++;
    return REAL(Irecv)(buf, count, dt, source, tag, comm, req);
  }
  Pending p;
  p.recv = true;
  p.user = buf;
  p.count = count;
  p.type = m.h;
  p.size = m.size;
  p.method = choose(m, count);
  const size_t bytes = static_cast<size_t>(m.size * count);
  if (!take_buffers(p, bytes)) return MPI_ERR_NO_MEM;
  const int rc = REAL(Irecv)(recv_target(p.method, p.dev, p.host), static_cast<int>(bytes), MPI_BYTE, source, tag,
                             comm, req);
  if (rc != MPI_SUCCESS) {
    give_buffers(p);
    return rc;
  }
  std::lock_guard<std::mutex> lk(S().mu);
  S().pending[*req] = p;
  ++S().in_flight[p.type];
  return MPI_SUCCESS;
}

} // extern "C"

namespace {

// a request the system MPI just completed: unpack a receive, free its scratch
int finish(MPI_Request key, MPI_Status *status, int rc) {
  { // a persistent neighbour collective: unpack what its start received
    std::vector<Segment> unpack;
    bool ours = false;
    {
      std::lock_guard<std::mutex> lk(S().mu);
      auto c = S().colls.find(key);
      if (c != S().colls.end()) {
        ours = true;
        if (c->second.started) unpack = c->second.unpack; // (a wait on an inactive request moves nothing)
        c->second.started = false;
      }
    }
    if (ours) {
      if (rc == MPI_SUCCESS && !unpack.empty()) {
        rc = run_segments(unpack, true);
        if (rc == MPI_SUCCESS) rc = stream_sync();
      }
      return rc;
    }
  }
  Pending p;
  bool persistent = false;
  {
    std::lock_guard<std::mutex> lk(S().mu);
    auto it = S().pending.find(key);
    if (it == S().pending.end()) {
      auto q = S().persist.find(key);
      if (q == S().persist.end()) return rc;
      p = q->second; // a persistent request: unpack a receive, keep the buffers
      persistent = true;
    } else {
      p = it->second;
      S().pending.erase(it);
    }
  }
  if (persistent) {
    if (p.recv && rc == MPI_SUCCESS && status) {
      Mirror m;
      m.h = p.type;
      m.size = p.size;
      rc = unpack_message(m, p.user, received(status), p.method, p.dev, p.host);
      report_method(status, p.method);
    }
    return rc;
  }
  struct Release { // the receive's mirror, once nothing pending names it
    sp_type h;
    ~Release() {
      if (!h) return;
      std::lock_guard<std::mutex> lk(S().mu);
      auto f = S().in_flight.find(h);
      if (f != S().in_flight.end() && --f->second == 0) {
        S().in_flight.erase(f);
        if (S().retired.erase(h)) sp_type_free(h);
      }
    }
  } release{p.recv ? p.type : 0};
  if (p.recv && rc == MPI_SUCCESS && status) {
    Mirror m;
    m.h = p.type;
    m.size = p.size;
    rc = unpack_message(m, p.user, received(status), p.method, p.dev, p.host);
    report_method(status, p.method);
  }
  give_buffers(p);
  return rc;
}

} // namespace

extern "C" {

int MPI_Wait(MPI_Request *req, MPI_Status *status) {
  if (!req) return MPI_ERR_ARG;
  const MPI_Request key = *req;
  MPI_Status st{};
  const int rc = REAL(Wait)(req, &st);
  const int out = finish(key, &st, rc);
  if (status) *status = st;
  return out;
}

int MPI_Test(MPI_Request *req, int *flag, MPI_Status *status) {
  if (!req || !flag) return MPI_ERR_ARG;
  const MPI_Request key = *req;
  MPI_Status st{};
  const int rc = REAL(Test)(req, flag, &st);
  if (!*flag) return rc;
  const int out = finish(key, &st, rc);
  if (status) *status = st;
  return out;
}

int MPI_Waitall(int n, MPI_Request reqs[], MPI_Status statuses[]) {
  if (n < 0 || (n && !reqs)) return MPI_ERR_ARG;
  int first = MPI_SUCCESS;
  for (int i = 0; i < n; ++i) {
    const int rc = MPI_Wait(&reqs[i], statuses ? &statuses[i] : nullptr);
    if (rc != MPI_SUCCESS && first == MPI_SUCCESS) first = rc;
  }
  return first;
}

// the set forms of MPI-3.1 3.7.5: the system MPI completes, the interposer
// then unpacks the receives among the completed requests (their handles
// are saved first: completion resets them to MPI_REQUEST_NULL)
int MPI_Waitany(int n, MPI_Request reqs[], int *index, MPI_Status *status) {
  if (n < 0 || (n && !reqs) || !index) return MPI_ERR_ARG;
  const std::vector<MPI_Request> keys(reqs, reqs + n);
  MPI_Status st{};
  const int rc = REAL(Waitany)(n, reqs, index, &st);
  int out = rc;
  if (*index != MPI_UNDEFINED && *index >= 0 && *index < n) out = finish(keys[*index], &st, rc);
  if (status) *status = st;
  return out;
}

int MPI_Testany(int n, MPI_Request reqs[], int *index, int *flag, MPI_Status *status) {
  if (n < 0 || (n && !reqs) || !index || !flag) return MPI_ERR_ARG;
  const std::vector<MPI_Request> keys(reqs, reqs + n);
  MPI_Status st{};
  const int rc = REAL(Testany)(n, reqs, index, flag, &st);
  int out = rc;
  if (*flag && *index != MPI_UNDEFINED && *index >= 0 && *index < n) out = finish(keys[*index], &st, rc);
  if (status) *status = st;
  return out;
}

int MPI_Waitsome(int n, MPI_Request reqs[], int *outcount, int indices[], MPI_Status statuses[]) {
  if (n < 0 || (n && !reqs) || !outcount) return MPI_ERR_ARG;
  const std::vector<MPI_Request> keys(reqs, reqs + n);
  std::vector<MPI_Status> st(std::max(n, 1));
  const int rc = REAL(Waitsome)(n, reqs, outcount, indices, st.data());
  int out = rc;
  if (*outcount != MPI_UNDEFINED)
    for (int i = 0; i < *outcount; ++i) {
      const int r = finish(keys[indices[i]], &st[i], rc);
      if (r != MPI_SUCCESS && out == MPI_SUCCESS) out = r;
      if (statuses) statuses[i] = st[i];
    }
  return out;
}

int MPI_Testall(int n, MPI_Request reqs[], int *flag, MPI_Status statuses[]) {
  if (n < 0 || (n && !reqs) || !flag) return MPI_ERR_ARG;
  const std::vector<MPI_Request> keys(reqs, reqs + n);
  std::vector<MPI_Status> st(std::max(n, 1));
  const int rc = REAL(Testall)(n, reqs, flag, st.data());
  int out = rc;
  if (*flag)
    for (int i = 0; i < n; ++i) {
      const int r = finish(keys[i], &st[i], rc);
      if (r != MPI_SUCCESS && out == MPI_SUCCESS) out = r;
      if (statuses) statuses[i] = st[i];
    }
  return out;
}

// an interposed request must still unpack (a receive) or keep its packed
// buffer until the system MPI is done with it (a send): it is completed here
int MPI_Request_free(MPI_Request *req) {
  if (!req) return MPI_ERR_ARG;
  {
    bool coll = false;
    {
      std::lock_guard<std::mutex> lk(S().mu);
      coll = S().colls.count(*req) != 0;
    }
    if (coll) { // complete a start still in flight, then release its packed buffers
      const MPI_Request key = *req;
      const int rc = MPI_Wait(req, MPI_STATUS_IGNORE);
      *req = key;
      const int rf = REAL(Request_free)(req);
      State::Coll c;
      {
        std::lock_guard<std::mutex> lk(S().mu);
        c = S().colls[key];
        S().colls.erase(key);
      }
      for (void *b : {c.sp, c.rp})
        if (b) c.pinned ? cudaFreeHost(b) : cudaFree(b);
      return rc != MPI_SUCCESS ? rc : rf;
    }
  }
  bool ours = false, persistent = false;
  {
    std::lock_guard<std::mutex> lk(S().mu);
    ours = S().pending.count(*req) != 0;
    persistent = S().persist.count(*req) != 0;
  }
  if (persistent) { // complete an operation still in flight, then release the buffers
    const MPI_Request key = *req;
    int rc = MPI_Wait(req, MPI_STATUS_IGNORE);
    const int rf = REAL(Request_free)(req);
    Pending p;
    {
      std::lock_guard<std::mutex> lk(S().mu);
      p = S().persist[key];
      S().persist.erase(key);
      if (p.recv) {
        auto f = S().in_flight.find(p.type);
        if (f != S().in_flight.end() && --f->second == 0) {
          S().in_flight.erase(f);
          if (S().retired.erase(p.type)) sp_type_free(p.type);
        }
      }
    }
    give_buffers(p);
    return rc != MPI_SUCCESS ? rc : rf;
  }
  if (!ours) return REAL(Request_free)(req);
  return MPI_Wait(req, MPI_STATUS_IGNORE);
}

// ---- persistent requests (MPI-3.1 3.9): the system MPI's persistent
// request moves the packed MPI_BYTE message; MPI_Start packs first
int MPI_Send_init(const void *buf, int count, MPI_Datatype dt, int dest, int tag, MPI_Comm comm, MPI_Request *req) {
  Mirror m;
  if (!req) return MPI_ERR_ARG;
  if (!accel(dt, buf, count, &m) || m.size * count > INT32_MAX) {
    S().st.forwarded++;
    return REAL(Send_init)(buf, count, dt, dest, tag, comm, req);
  }
  Pending p;
  p.user = const_cast<void *>(buf);
  p.count = count;
  p.type = m.h;
  p.size = m.size;
  p.method = choose(m, count);
  const size_t bytes = static_cast<size_t>(m.size * count);
  if (!take_buffers(p, bytes)) return MPI_ERR_NO_MEM;
  // the buffer the system MPI sends from: pinned for one-shot / staged
  void *msg = p.method == SP_METHOD_DEVICE ? p.dev : p.host;
  const int rc = REAL(Send_init)(msg, static_cast<int>(bytes), MPI_BYTE, dest, tag, comm, req);
  if (rc != MPI_SUCCESS) {
    give_buffers(p);
    return rc;
  }
  std::lock_guard<std::mutex> lk(S().mu);
  S().persist[*req] = p;
  return MPI_SUCCESS;
}

int MPI_Recv_init(void *buf, int count, MPI_Datatype dt, int source, int tag, MPI_Comm comm, MPI_Request *req) {
  Mirror m;
  if (!req) return MPI_ERR_ARG;
  if (!accel(dt, buf, count, &m) || m.size * count > INT32_MAX) {
    S().st.forwarded++;
    return REAL(Recv_init)(buf, count, dt, source, tag, comm, req);
  }
  Pending p;
  p.recv = true;
  p.user = buf;
  p.count = count;
  p.type = m.h;
  p.size = m.size;
  p.method = choose(m, count);
  const size_t bytes = static_cast<size_t>(m.size * count);
  if (!take_buffers(p, bytes)) return MPI_ERR_NO_MEM;
  const int rc = REAL(Recv_init)(recv_target(p.method, p.dev, p.host), static_cast<int>(bytes), MPI_BYTE, source,
                                 tag, comm, req);
  if (rc != MPI_SUCCESS) {
    give_buffers(p);
    return rc;
  }
  std::lock_guard<std::mutex> lk(S().mu);
  S().persist[*req] = p;
  ++S().in_flight[p.type];
  return MPI_SUCCESS;
}

int MPI_Start(MPI_Request *req) {
  if (!req) return MPI_ERR_ARG;
  Pending p;
  bool ours = false;
  {
    std::lock_guard<std::mutex> lk(S().mu);
    auto it = S().persist.find(*req);
    if (it != S().persist.end()) {
      ours = true;
      p = it->second;
    }
  }
  std::vector<Segment> pack;
  bool coll = false;
  {
    std::lock_guard<std::mutex> lk(S().mu);
    auto c = S().colls.find(*req);
    if (c != S().colls.end()) {
      coll = true;
      pack = c->second.pack;
      c->second.started = true;
    }
  }
  if (coll && !pack.empty()) { // the send side's segments into its packed buffer
    int rc = run_segments(pack, false);
    if (rc == MPI_SUCCESS) rc = stream_sync();
    if (rc != MPI_SUCCESS) return rc;
  }
  if (ours && !p.recv) { // pack this round's data into the registered message buffer
    Mirror m;
    m.h = p.type;
    m.size = p.size;
    void *msg = nullptr;
    const int rc = pack_message(m, p.user, static_cast<int>(p.count), p.method, p.dev, p.host, &msg);
    if (rc != MPI_SUCCESS) return rc;
  }
  return REAL(Start)(req);
}

int MPI_Startall(int n, MPI_Request reqs[]) {
  if (n < 0 || (n && !reqs)) return MPI_ERR_ARG;
  for (int i = 0; i < n; ++i) {
    const int rc = MPI_Start(&reqs[i]);
    if (rc != MPI_SUCCESS) return rc;
  }
  return MPI_SUCCESS;
}

// through the intercepted non-blocking calls, so both halves are accelerated
int MPI_Sendrecv(const void *sbuf, int scount, MPI_Datatype stype, int dest, int stag, void *rbuf, int rcount,
                 MPI_Datatype rtype, int source, int rtag, MPI_Comm comm, MPI_Status *status) {
  MPI_Request r[2] = {MPI_REQUEST_NULL, MPI_REQUEST_NULL};
  int rc = MPI_Irecv(rbuf, rcount, rtype, source, rtag, comm, &r[0]);
  if (rc != MPI_SUCCESS) return rc;
  rc = MPI_Isend(sbuf, scount, stype, dest, stag, comm, &r[1]);
  if (rc != MPI_SUCCESS) {
    MPI_Wait(&r[0], MPI_STATUS_IGNORE);
    return rc;
  }
  const int rc1 = MPI_Wait(&r[1], MPI_STATUS_IGNORE);
  const int rc0 = MPI_Wait(&r[0], status);
  return rc0 != MPI_SUCCESS ? rc0 : rc1;
}

// ============================================================ topologies (degrees recorded for the exchanges)
int MPI_Dist_graph_create_adjacent(MPI_Comm old, int indeg, const int sources[], const int sw[], int outdeg,
                                   const int dests[], const int dw[], MPI_Info info, int reorder, MPI_Comm *out) {
  const int rc = REAL(Dist_graph_create_adjacent)(old, indeg, sources, sw, outdeg, dests, dw, info, reorder, out);
  if (rc == MPI_SUCCESS && out) {
    std::lock_guard<std::mutex> lk(S().mu);
    S().degree[*out] = {indeg, outdeg};
  }
  return rc;
}

int MPI_Cart_create(MPI_Comm old, int nd, const int dims[], const int periods[], int reorder, MPI_Comm *out) {
  const int rc = REAL(Cart_create)(old, nd, dims, periods, reorder, out);
  if (rc == MPI_SUCCESS && out) {
    std::lock_guard<std::mutex> lk(S().mu);
    S().degree[*out] = {2 * nd, 2 * nd};
  }
  return rc;
}

int MPI_Comm_free(MPI_Comm *comm) {
  if (comm) {
    std::lock_guard<std::mutex> lk(S().mu);
    S().degree.erase(*comm);
  }
  return REAL(Comm_free)(comm);
}

} // extern "C"

namespace {

bool degrees(MPI_Comm comm, int *in, int *out) {
  std::lock_guard<std::mutex> lk(S().mu);
  auto it = S().degree.find(comm);
  if (it == S().degree.end()) return false;
  *in = it->second.first;
  *out = it->second.second;
  return true;
}

// a neighbour exchange (all = false) or an all-to-all over the whole
// communicator (all = true) with packed MPI_BYTE sides where accelerated
int exchange(const void *sbuf, const int scounts[], const int64_t *sdisp_b, const MPI_Datatype *stypes,
             MPI_Datatype stype, void *rbuf, const int rcounts[], const int64_t *rdisp_b,
             const MPI_Datatype *rtypes, MPI_Datatype rtype, int indeg, int outdeg, MPI_Comm comm, bool all,
             bool *done) {
  *done = false;
  Side s = plan_side(sbuf, outdeg, scounts, stypes, stype);
  Side r = plan_side(rbuf, indeg, rcounts, rtypes, rtype);
  if (!s.accel && !r.accel) return MPI_SUCCESS;
  *done = true;
  State &st = S();
  st.st.exchanges++;
  std::lock_guard<std::mutex> lk(st.scratch_mu);
  // packed segments stay on the device for a CUDA-aware system MPI, else
  // they are written to (read from) pinned memory by the same launch
  Scratch &sb = st.cuda_aware ? st.dev_s : st.host_s, &rb = st.cuda_aware ? st.dev_r : st.host_r;
  void *sp = s.accel ? sb.get(static_cast<size_t>(s.total)) : nullptr;
  void *rp = r.accel ? rb.get(static_cast<size_t>(r.total)) : nullptr;
  if ((s.accel && s.total && !sp) || (r.accel && r.total && !rp)) return MPI_ERR_NO_MEM;
  if (s.accel) {
    std::vector<Segment> segs;
    for (int i = 0; i < outdeg; ++i)
      segs.push_back({static_cast<const uint8_t *>(sbuf) + sdisp_b[i], s.m[i].h, scounts[i], sp, s.offs[i]});
    int rc = run_segments(segs, false);
    if (rc == MPI_SUCCESS) rc = stream_sync();
    if (rc != MPI_SUCCESS) return rc;
  }
  // the system MPI's exchange over the packed bytes (alltoallw: each side
  // either its packed MPI_BYTE segments or the caller's own arguments)
  std::vector<int> scb, rcb;
  std::vector<MPI_Aint> sdb, rdb;
  std::vector<MPI_Datatype> stb, rtb;
  for (int i = 0; i < outdeg; ++i) {
    scb.push_back(s.accel ? s.bytes[i] : scounts[i]);
    sdb.push_back(s.accel ? s.offs[i] : sdisp_b[i]);
    stb.push_back(s.accel ? MPI_BYTE : stypes ? stypes[i] : stype);
  }
  for (int j = 0; j < indeg; ++j) {
    rcb.push_back(r.accel ? r.bytes[j] : rcounts[j]);
    rdb.push_back(r.accel ? r.offs[j] : rdisp_b[j]);
    rtb.push_back(r.accel ? MPI_BYTE : rtypes ? rtypes[j] : rtype);
  }
  int rc = MPI_SUCCESS;
  if (all) { // MPI_Alltoallw: int byte displacements
    const std::vector<int> sdi(sdb.begin(), sdb.end()), rdi(rdb.begin(), rdb.end());
    rc = REAL(Alltoallw)(s.accel ? sp : sbuf, scb.data(), sdi.data(), stb.data(), r.accel ? rp : rbuf, rcb.data(),
                         rdi.data(), rtb.data(), comm);
  } else {
    rc = REAL(Neighbor_alltoallw)(s.accel ? sp : sbuf, scb.data(), sdb.data(), stb.data(), r.accel ? rp : rbuf,
                                  rcb.data(), rdb.data(), rtb.data(), comm);
  }
  if (rc != MPI_SUCCESS || !r.accel) return rc;
  std::vector<Segment> segs;
  for (int j = 0; j < indeg; ++j)
    segs.push_back({rp, r.m[j].h, rcounts[j], static_cast<uint8_t *>(rbuf) + rdisp_b[j], r.offs[j]});
  rc = run_segments(segs, true);
  if (rc == MPI_SUCCESS) rc = stream_sync();
  return rc;
}

} // namespace

extern "C" {

int MPI_Neighbor_alltoallv(const void *sbuf, const int scounts[], const int sdispls[], MPI_Datatype stype, void *rbuf,
                           const int rcounts[], const int rdispls[], MPI_Datatype rtype, MPI_Comm comm) {
  int indeg = 0, outdeg = 0;
  Mirror sm, rm;
  if (degrees(comm, &indeg, &outdeg) && committed(stype, &sm) && committed(rtype, &rm)) {
    std::vector<int64_t> sd(outdeg), rd(indeg);
    for (int i = 0; i < outdeg; ++i) sd[i] = static_cast<int64_t>(sdispls[i]) * sm.extent;
    for (int j = 0; j < indeg; ++j) rd[j] = static_cast<int64_t>(rdispls[j]) * rm.extent;
    bool done = false;
    const int rc = exchange(sbuf, scounts, sd.data(), nullptr, stype, rbuf, rcounts, rd.data(), nullptr, rtype, indeg,
                            outdeg, comm, false, &done);
    if (done) return rc;
  }
  S().st.forwarded++;
  return REAL(Neighbor_alltoallv)(sbuf, scounts, sdispls, stype, rbuf, rcounts, rdispls, rtype, comm);
}

int MPI_Neighbor_alltoallw(const void *sbuf, const int scounts[], const MPI_Aint sdispls[],
                           const MPI_Datatype stypes[], void *rbuf, const int rcounts[], const MPI_Aint rdispls[],
                           const MPI_Datatype rtypes[], MPI_Comm comm) {
  int indeg = 0, outdeg = 0;
  if (degrees(comm, &indeg, &outdeg)) {
    std::vector<int64_t> sd(sdispls, sdispls + outdeg), rd(rdispls, rdispls + indeg);
    bool done = false;
    const int rc = exchange(sbuf, scounts, sd.data(), stypes, MPI_DATATYPE_NULL, rbuf, rcounts, rd.data(), rtypes,
                            MPI_DATATYPE_NULL, indeg, outdeg, comm, false, &done);
    if (done) return rc;
  }
  S().st.forwarded++;
  return REAL(Neighbor_alltoallw)(sbuf, scounts, sdispls, stypes, rbuf, rcounts, rdispls, rtypes, comm);
}

// MPI-4.0 persistent neighbour collective: the system MPI's persistent
// byte exchange between packed buffers owned by the request; MPI_Start
// packs every accelerated send segment in one launch first, completion
// unpacks every accelerated receive segment in one launch
int MPI_Neighbor_alltoallw_init(const void *sbuf, const int scounts[], const MPI_Aint sdispls[],
                                const MPI_Datatype stypes[], void *rbuf, const int rcounts[],
                                const MPI_Aint rdispls[], const MPI_Datatype rtypes[], MPI_Comm comm, MPI_Info info,
                                MPI_Request *req) {
  int indeg = 0, outdeg = 0;
  if (!req) return MPI_ERR_ARG;
  const auto real_init = REAL_OPT(Neighbor_alltoallw_init);
  if (!real_init) return MPI_ERR_UNSUPPORTED_OPERATION; // an MPI-3 system library
  if (!degrees(comm, &indeg, &outdeg))
    return real_init(sbuf, scounts, sdispls, stypes, rbuf, rcounts, rdispls, rtypes, comm, info, req);
  Side s = plan_side(sbuf, outdeg, scounts, stypes, MPI_DATATYPE_NULL);
  Side r = plan_side(rbuf, indeg, rcounts, rtypes, MPI_DATATYPE_NULL);
  if (!s.accel && !r.accel) {
    S().st.forwarded++;
    return real_init(sbuf, scounts, sdispls, stypes, rbuf, rcounts, rdispls, rtypes, comm, info, req);
  }
  State::Coll c;
  c.pinned = !S().cuda_aware;
  auto alloc = [&](int64_t n) -> void * {
    void *p = nullptr;
    const size_t b = static_cast<size_t>(std::max<int64_t>(n, 1));
    if ((c.pinned ? cudaMallocHost(&p, b) : cudaMalloc(&p, b)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return p;
  };
  if (s.accel && !(c.sp = alloc(s.total))) return MPI_ERR_NO_MEM;
  if (r.accel && !(c.rp = alloc(r.total))) {
    if (c.sp) c.pinned ? cudaFreeHost(c.sp) : cudaFree(c.sp);
    return MPI_ERR_NO_MEM;
  }
  std::vector<int> scb, rcb;
  std::vector<MPI_Aint> sdb, rdb;
  std::vector<MPI_Datatype> stb, rtb;
  for (int i = 0; i < outdeg; ++i) {
    scb.push_back(s.accel ? s.bytes[i] : scounts[i]);
    sdb.push_back(s.accel ? s.offs[i] : sdispls[i]);
    stb.push_back(s.accel ? MPI_BYTE : stypes[i]);
    if (s.accel)
      c.pack.push_back({static_cast<const uint8_t *>(sbuf) + sdispls[i], s.m[i].h, scounts[i], c.sp, s.offs[i]});
  }
  for (int j = 0; j < indeg; ++j) {
    rcb.push_back(r.accel ? r.bytes[j] : rcounts[j]);
    rdb.push_back(r.accel ? r.offs[j] : rdispls[j]);
    rtb.push_back(r.accel ? MPI_BYTE : rtypes[j]);
    if (r.accel)
      c.unpack.push_back({c.rp, r.m[j].h, rcounts[j], static_cast<uint8_t *>(rbuf) + rdispls[j], r.offs[j]});
  }
  const int rc = real_init(s.accel ? c.sp : sbuf, scb.data(), sdb.data(), stb.data(), r.accel ? c.rp : rbuf,
                           rcb.data(), rdb.data(), rtb.data(), comm, info, req);
  if (rc != MPI_SUCCESS) {
    for (void *b : {c.sp, c.rp})
      if (b) c.pinned ? cudaFreeHost(b) : cudaFree(b);
    return rc;
  }
  std::lock_guard<std::mutex> lk(S().mu);
  S().colls[*req] = std::move(c);
  return MPI_SUCCESS;
}

// the v form: one type per side, displacements in extents -- the w form's
// arguments (byte displacements, the type on every edge)
int MPI_Neighbor_alltoallv_init(const void *sbuf, const int scounts[], const int sdispls[], MPI_Datatype stype,
                                void *rbuf, const int rcounts[], const int rdispls[], MPI_Datatype rtype,
                                MPI_Comm comm, MPI_Info info, MPI_Request *req) {
  int indeg = 0, outdeg = 0;
  Mirror sm, rm;
  if (!degrees(comm, &indeg, &outdeg) || !committed(stype, &sm) || !committed(rtype, &rm)) {
    const auto real_v = REAL_OPT(Neighbor_alltoallv_init);
    if (!real_v) return MPI_ERR_UNSUPPORTED_OPERATION;
    S().st.forwarded++;
    return real_v(sbuf, scounts, sdispls, stype, rbuf, rcounts, rdispls, rtype, comm, info, req);
  }
  std::vector<MPI_Aint> sd(outdeg), rd(indeg);
  for (int i = 0; i < outdeg; ++i) sd[i] = static_cast<MPI_Aint>(sdispls[i]) * sm.extent;
  for (int j = 0; j < indeg; ++j) rd[j] = static_cast<MPI_Aint>(rdispls[j]) * rm.extent;
  const std::vector<MPI_Datatype> st(outdeg, stype), rt(indeg, rtype);
  return MPI_Neighbor_alltoallw_init(sbuf, scounts, sd.data(), st.data(), rbuf, rcounts, rd.data(), rt.data(), comm,
                                     info, req);
}

// ============================================================ all-to-all (MPI-3.1 5.8)
int MPI_Alltoallv(const void *sbuf, const int scounts[], const int sdispls[], MPI_Datatype stype, void *rbuf,
                  const int rcounts[], const int rdispls[], MPI_Datatype rtype, MPI_Comm comm) {
  int n = 0;
  Mirror sm, rm;
  if (REAL(Comm_size)(comm, &n) == MPI_SUCCESS && committed(stype, &sm) && committed(rtype, &rm)) {
    std::vector<int64_t> sd(n), rd(n);
    for (int i = 0; i < n; ++i) {
      sd[i] = static_cast<int64_t>(sdispls[i]) * sm.extent;
      rd[i] = static_cast<int64_t>(rdispls[i]) * rm.extent;
    }
    bool done = false;
    const int rc = exchange(sbuf, scounts, sd.data(), nullptr, stype, rbuf, rcounts, rd.data(), nullptr, rtype, n, n,
                            comm, true, &done);
    if (done) return rc;
  }
  S().st.forwarded++;
  return REAL(Alltoallv)(sbuf, scounts, sdispls, stype, rbuf, rcounts, rdispls, rtype, comm);
}

int MPI_Alltoallw(const void *sbuf, const int scounts[], const int sdispls[], const MPI_Datatype stypes[], void *rbuf,
                  const int rcounts[], const int rdispls[], const MPI_Datatype rtypes[], MPI_Comm comm) {
  int n = 0;
  if (REAL(Comm_size)(comm, &n) == MPI_SUCCESS) {
    std::vector<int64_t> sd(sdispls, sdispls + n), rd(rdispls, rdispls + n);
    bool done = false;
    const int rc = exchange(sbuf, scounts, sd.data(), stypes, MPI_DATATYPE_NULL, rbuf, rcounts, rd.data(), rtypes,
                            MPI_DATATYPE_NULL, n, n, comm, true, &done);
    if (done) return rc;
  }
  S().st.forwarded++;
  return REAL(Alltoallw)(sbuf, scounts, sdispls, stypes, rbuf, rcounts, rdispls, rtypes, comm);
}

// ============================================================ TEMPI controls
int TEMPI_Set_method(int method) {
  if (method < -1 || method > 3) return MPI_ERR_ARG;
  S().forced = method;
  return MPI_SUCCESS;
}

int TEMPI_Load_profile(const char *path) {
  sp_profile p = nullptr;
  TRY(sp_profile_load(path, &p));
  sp_model_cache c = nullptr;
  TRY(sp_model_cache_create(p, &c));
  if (S().model) sp_model_cache_free(S().model);
  if (S().profile) sp_profile_free(S().profile);
  S().profile = p;
  S().model = c;
  return MPI_SUCCESS;
}

} // extern "C"
