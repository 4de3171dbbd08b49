// rt.cpp -- single-node multi-process runtime under the MPI surface.
//
// TEMPI sits on a system MPI; this image has none, so
// the engine carries its own node-local transport: one process per GPU,
// a POSIX shared-memory segment for bootstrap, barriers and control
// mailboxes, CUDA IPC for device memory (kernels store straight into a
// peer's HBM over NVLink), and shared pinned host regions for the one-shot
// and staged methods. Nothing here needs a device except the data paths,
// so the control plane is testable on CPU.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <csignal>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "guard.hpp"
#include "model.hpp"
#include "rt.hpp"

namespace spb {

void nbr_reset();

void engine_init(int64_t window_bytes, int64_t host_bytes);
void engine_fini();

namespace {

constexpr uint64_t kMagic = 0x5350423230305254ull; // "SPB200RT"
constexpr int kMaxRanks = 64;
constexpr int kRing = 32;
constexpr int kMaxEdges = 256;

struct Msg {
  uint32_t kind;
  int32_t src;
  int32_t tag;
  int32_t method;
  int64_t bytes;
  int64_t offset;
  int64_t aux;
};

struct Mailbox { // single producer (src) / single consumer (dst)
  std::atomic<uint64_t> head; // next slot the consumer reads
  std::atomic<uint64_t> tail; // next slot the producer writes
  Msg ring[kRing];
};

// a receiver's published destination for a DIRECT message: its buffer (IPC
// handle + offset, raw pointer for self-sends) and its type's canonical
// StridedBlock, from which the sender rebuilds the destination geometry
constexpr int kDescs = 32;
constexpr int kDescDims = 12;
constexpr int kMaxWEdges = 64;
struct Desc {
  int32_t ndims;
  int32_t runs; // 1: a block-list layout, described by its device run table below
  int64_t start, size, extent, span, count;
  int64_t counts[kDescDims], strides[kDescDims];
  cudaIpcMemHandle_t h;
  int64_t off;
  uint64_t raw;
  uint64_t hr[2], sr[2], dr[2]; // the exporter's allocation (base, bytes) behind h, hs, hd
  // runs == 1: the receiver's run table (piece source offsets, packed
  // prefix) for peers through CUDA IPC, and raw for the receiver itself
  cudaIpcMemHandle_t hs, hd;
  int64_t os, od, npieces;
  uint64_t align, raw_s, raw_d;
};

struct Slot {
  std::atomic<uint32_t> ready;
  int32_t pid;
  int32_t device;
  int32_t pad;
  uint8_t uuid[16];           // the GPU's UUID (ordinals differ between processes)
  cudaIpcMemHandle_t window;  // device receive window (DEVICE method)
  int64_t window_bytes;
  int64_t host_bytes;         // shared pinned host region (ONESHOT/STAGED)
  cudaIpcMemHandle_t xh;      // publication area of sp_rt_exchange_ptr
  int64_t xoff;
  uint64_t xr[2];             // the allocation behind xh in the publisher's address space (base, bytes)
  int64_t xbytes;
  int32_t nedges;             // neighbour-exchange in-edges: (src, offset, bytes)
  int32_t pad2;
  int64_t edges[kMaxEdges][3];
  Desc desc[kDescs];          // DIRECT destinations granted by this rank
  Desc wdesc[kMaxWEdges];     // MPI_Neighbor_alltoallw in-edge destinations
  // neighbour collectives: pair_entered[s] = how many calls with s as a
  // source this rank has entered (its layout for that call is published)
  std::atomic<uint64_t> pair_entered[kMaxRanks];
  std::atomic<uint64_t> layout_ver; // bumped whenever the published neighbour layout changes
};

struct Shm {
  uint64_t magic;
  int32_t size;
  int32_t pad;
  std::atomic<uint32_t> arrived;
  std::atomic<uint32_t> generation;
  Slot slots[kMaxRanks];
  Mailbox box[kMaxRanks][kMaxRanks]; // box[dst][src]
};

enum : uint32_t { kRTS = 1, kCTS = 2, kFIN = 3 };

void pause_briefly(unsigned &spins) {
  if (++spins < 256) return;
  if (spins < 4096) {
    sched_yield();
  } else {
    timespec ts{0, 2000};
    nanosleep(&ts, nullptr);
  }
}

// TEMPI_TIMEOUT (seconds, default 300; 0 = wait forever): how long any
// host wait for a peer and any in-kernel wait for a peer's flag may last
double timeout_s() {
  static const double t = [] {
    const char *e = std::getenv("TEMPI_TIMEOUT");
    return e && *e ? std::atof(e) : 300.0;
  }();
  return t;
}

struct Runtime;
Runtime *g_rt = nullptr;
void check_peers_alive(int peer, const char *what);

// A host wait on other ranks: backs off like pause_briefly, and every few
// milliseconds checks that the awaited rank(s) still exist and that the
// wait has not outlived TEMPI_TIMEOUT -- a dead or stuck peer becomes
// SP_ERR_TIMEOUT (MPI_ERR_OTHER) instead of a hang.
struct Waiter {
  unsigned spins = 0;
  int peer; // the rank waited for, -1: any rank
  const char *what;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit Waiter(const char *w, int p = -1) : peer(p), what(w) {}
  void pause() {
    pause_briefly(spins);
    if (spins < 4096 || (spins & 127)) return;
    if (g_rt) check_peers_alive(peer, what);
    const double lim = timeout_s();
    if (lim > 0 && std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > lim)
      fail(SP_ERR_TIMEOUT, std::string(what) + ": no progress within TEMPI_TIMEOUT=" + std::to_string(lim) + " s" +
                               (peer >= 0 ? " waiting for rank " + std::to_string(peer) : std::string()));
  }
};

struct Runtime {
  int rank = -1, size = 0, device = -1;
  std::string name;
  Shm *shm = nullptr;
  size_t shm_bytes = 0;
  // device window and pinned host region owned by this rank
  uint8_t *window = nullptr;
  int64_t window_bytes = 0;
  uint8_t *host = nullptr;
  int64_t host_bytes = 0;
  // peers' resources, opened lazily
  std::vector<uint8_t *> peer_window;
  std::vector<uint8_t *> peer_host;
  // peers' allocations mapped through CUDA IPC, by handle bytes; `pins`
  // counts long-lived users (halo plans), unpinned entries are a cache
  struct IpcMap {
    uint8_t *p = nullptr;
    int peer = -1;
    int pins = 0;
    uint64_t used = 0; // ipc_clock at the last open_ipc that returned it
    uint64_t base = 0, bytes = 0; // the allocation in the peer's address space (0: unknown)
  };
  std::map<std::string, IpcMap> ipc_cache;
  uint64_t ipc_clock = 0, ipc_call_mark = 0; // mappings used since the mark belong to the call in progress
  std::map<const uint8_t *, std::string> exchanged; // rt_exchange_ptr result -> its mapping
  std::deque<Msg> unexpected;
  cudaStream_t stream = nullptr;  // sends, batches, halo plans
  cudaStream_t rstream = nullptr; // receives (unpack of arriving chunks)
  // neighbour collectives: per-source READY counters written by the
  // senders' kernels (IPC-mapped), calls per peer pair, a block counter
  uint64_t *nbr_flags = nullptr;
  std::vector<uint8_t *> peer_nbr_flags;
  std::vector<uint64_t> pair_sent, pair_recv;
  bool nbr_remote = false;
  bool shared_device = false; // another rank of the job runs on this rank's GPU
  // set (to 1) by an in-kernel flag wait that gave up after TEMPI_TIMEOUT;
  // mapped pinned memory, read by the host after each synchronisation
  int *err_host = nullptr, *err_dev = nullptr;
  std::string nbr_layout; // bytes of the last published neighbour layout
  std::unique_ptr<sp_model_cache_s, sp_status (*)(sp_model_cache_s *)> cache{nullptr, sp_model_cache_free};
  // the model's profile: the runtime holds its own reference (the caller's
  // sp_profile handle may be freed right after sp_rt_set_profile)
  std::shared_ptr<const Profile> profile;
  std::map<std::tuple<int64_t, int64_t, int>, bool> direct_cache; // model_prefers_direct answers
  std::mutex mu; // the runtime serialises its own calls (MPI_THREAD_SERIALIZED)
};

Runtime &rt() {
  if (!g_rt) fail(SP_ERR_INVALID_ARGUMENT, "runtime not initialised (sp_rt_init)");
  return *g_rt;
}

void check_peers_alive(int peer, const char *what) {
  Runtime &R = *g_rt;
  for (int r = peer < 0 ? 0 : peer; r < (peer < 0 ? R.size : peer + 1); ++r) {
    if (r == R.rank) continue;
    const int32_t pid = R.shm->slots[r].pid;
    if (pid <= 0) continue;
    bool gone = kill(pid, 0) != 0 && errno == ESRCH;
    if (!gone) { // an exited process nobody has reaped yet is a zombie
      char path[64], buf[256];
      std::snprintf(path, sizeof(path), "/proc/%d/stat", static_cast<int>(pid));
      if (FILE *f = std::fopen(path, "r")) {
        const size_t n = std::fread(buf, 1, sizeof(buf) - 1, f);
        std::fclose(f);
        buf[n] = 0;
        const char *close_paren = std::strrchr(buf, ')');
        gone = close_paren && close_paren[1] == ' ' && (close_paren[2] == 'Z' || close_paren[2] == 'X');
      }
    }
    if (gone)
      fail(SP_ERR_TIMEOUT, std::string(what) + ": rank " + std::to_string(r) + " (pid " + std::to_string(pid) +
                               ") has exited");
  }
}

std::string host_name(const std::string &base, int r) { return base + "_h" + std::to_string(r); }

void *map_shm(const std::string &nm, size_t bytes, bool create) {
  int fd = -1;
  for (int tries = 0; fd < 0; ++tries) {
    fd = shm_open(nm.c_str(), O_RDWR | (create ? O_CREAT : 0), 0600);
    if (fd < 0 && (create || tries > 200000)) fail(SP_ERR_INTERNAL, "shm_open(" + nm + ") failed");
    if (fd < 0) usleep(50);
  }
  if (create && ftruncate(fd, static_cast<off_t>(bytes)) != 0) {
    close(fd);
    fail(SP_ERR_INTERNAL, "ftruncate(" + nm + ") failed");
  }
  if (!create) { // wait until the creator has sized it
    struct stat st{};
    for (int tries = 0; fstat(fd, &st) == 0 && static_cast<size_t>(st.st_size) < bytes; ++tries) {
      if (tries > 200000) fail(SP_ERR_INTERNAL, "shm segment never sized: " + nm);
      usleep(50);
    }
  }
  void *p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) fail(SP_ERR_INTERNAL, "mmap(" + nm + ") failed");
  return p;
}

void drain();

void post(int dst, const Msg &m) {
  Runtime &R = rt();
  Mailbox &b = R.shm->box[dst][R.rank];
  const uint64_t t = b.tail.load(std::memory_order_relaxed);
  Waiter w("control message (mailbox full)", dst);
  // a full ring: keep draining our own mailboxes so two ranks posting to
  // each other cannot wait on each other
  while (t - b.head.load(std::memory_order_acquire) >= kRing) {
    drain();
    w.pause();
  }
  b.ring[t % kRing] = m;
  b.tail.store(t + 1, std::memory_order_release);
}

// pull everything waiting in my mailboxes into the unexpected queue
void drain() {
  Runtime &R = rt();
  for (int s = 0; s < R.size; ++s) {
    Mailbox &b = R.shm->box[R.rank][s];
    uint64_t h = b.head.load(std::memory_order_relaxed);
    const uint64_t t = b.tail.load(std::memory_order_acquire);
    for (; h < t; ++h) R.unexpected.push_back(b.ring[h % kRing]);
    b.head.store(h, std::memory_order_release);
  }
}

Msg wait_msg(uint32_t kind, int src, int tag) {
  Runtime &R = rt();
  Waiter w("control message", src);
  for (;;) {
    drain();
    for (auto it = R.unexpected.begin(); it != R.unexpected.end(); ++it) {
      if (it->kind == kind && (src < 0 || it->src == src) && (tag < 0 || it->tag == tag)) {
        Msg m = *it;
        R.unexpected.erase(it);
        return m;
      }
    }
    w.pause();
  }
}

// A peer that frees an allocation and makes a new one at the same address
// exports a new handle that the driver refuses to map while this process
// still maps the old one (cudaErrorAlreadyMapped). The old allocation is
// gone on the peer's side, so its mapping here is stale: the unpinned
// mappings of that peer are closed one by one (after the device drained,
// and with every cached neighbour launch that could name them dropped)
// until the new handle opens. Mappings the call in progress already uses
// (since ipc_call_mark) are never closed.
// When the publisher also sent the allocation's range in its own address
// space (`range` = base, bytes), a cached mapping of the same peer whose
// range overlaps it under another handle is known to be stale before the
// open is tried (the peer can only reuse addresses it freed): it is closed
// first, and the driver never sees the conflicting open. The retry loop
// stays for publishers that give no range.
uint8_t *open_ipc(const cudaIpcMemHandle_t &h, int peer, const uint64_t *range = nullptr) {
  Runtime &R = rt();
  const std::string key(reinterpret_cast<const char *>(&h), sizeof(h));
  ++R.ipc_clock;
  auto it = R.ipc_cache.find(key);
  if (it != R.ipc_cache.end()) {
    it->second.used = R.ipc_clock;
    return it->second.p;
  }
  auto evictable = [&](const Runtime::IpcMap &m) {
    return m.peer == peer && m.pins == 0 && m.used <= R.ipc_call_mark;
  };
  auto close_entry = [&](std::map<std::string, Runtime::IpcMap>::iterator e) {
    cudaIpcCloseMemHandle(e->second.p);
    for (auto x = R.exchanged.begin(); x != R.exchanged.end();)
      x = x->second == e->first ? R.exchanged.erase(x) : std::next(x);
    return R.ipc_cache.erase(e);
  };
  const uint64_t base = range ? range[0] : 0, bytes = range ? range[1] : 0;
  auto overlaps = [&](const Runtime::IpcMap &m) {
    if (!m.base) return false;
    if (!m.bytes || !bytes) return m.base == base;
    return base < m.base + m.bytes && m.base < base + bytes;
  };
  if (base) {
    bool drained = false;
    for (auto e = R.ipc_cache.begin(); e != R.ipc_cache.end();) {
      if (!overlaps(e->second) || !evictable(e->second)) {
        ++e;
        continue;
      }
      if (!drained) {
        cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize(stale IPC mappings)");
        nbr_reset();
        drained = true;
      }
      e = close_entry(e);
    }
  }
  void *p = nullptr;
  cudaError_t err = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (err == cudaErrorAlreadyMapped) {
    cudaGetLastError();
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize(stale IPC mappings)");
    nbr_reset();
    for (auto e = R.ipc_cache.begin(); e != R.ipc_cache.end() && err == cudaErrorAlreadyMapped;) {
      if (!evictable(e->second)) {
        ++e;
        continue;
      }
      e = close_entry(e);
      err = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (err == cudaErrorAlreadyMapped) cudaGetLastError();
    }
  }
  cuda_check(err, "cudaIpcOpenMemHandle");
  R.ipc_cache[key] = Runtime::IpcMap{static_cast<uint8_t *>(p), peer, 0, R.ipc_clock, base, bytes};
  return static_cast<uint8_t *>(p);
}

} // namespace

// a halo plan holds the peer mappings rt_exchange_ptr gave it for its
// lifetime (pin = +1 at creation, -1 when the plan is freed)
// hold (delta > 0) or release a mapping by its handle (persistent plans)
void ipc_pin_handle(const cudaIpcMemHandle_t &h, int delta) {
  if (!g_rt) return;
  auto e = g_rt->ipc_cache.find(std::string(reinterpret_cast<const char *>(&h), sizeof(h)));
  if (e != g_rt->ipc_cache.end()) e->second.pins = std::max(0, e->second.pins + delta);
}

// marks the start of a call whose mappings must survive stale-mapping eviction
void ipc_call_begin() {
  if (g_rt) g_rt->ipc_call_mark = g_rt->ipc_clock;
}

void rt_pin_ptrs(const std::vector<uint8_t *> &ptrs, int delta) {
  if (!g_rt) return;
  Runtime &R = rt();
  for (const uint8_t *q : ptrs) {
    auto x = R.exchanged.find(q);
    if (x == R.exchanged.end()) continue;
    auto e = R.ipc_cache.find(x->second);
    if (e != R.ipc_cache.end()) e->second.pins = std::max(0, e->second.pins + delta);
  }
}

namespace {

uint8_t *peer_window(int r) {
  Runtime &R = rt();
  if (r == R.rank) return R.window;
  if (!R.peer_window[r]) {
    R.peer_window[r] = open_ipc(R.shm->slots[r].window, r);
    const std::string key(reinterpret_cast<const char *>(&R.shm->slots[r].window), sizeof(cudaIpcMemHandle_t));
    R.ipc_cache[key].pins = 1 << 20; // the runtime's own windows stay mapped until finalize
  }
  return R.peer_window[r];
}

uint8_t *peer_host(int r) {
  Runtime &R = rt();
  if (r == R.rank) return R.host;
  if (!R.peer_host[r]) {
    const int64_t bytes = R.shm->slots[r].host_bytes;
    auto *p = static_cast<uint8_t *>(map_shm(host_name(R.name, r), static_cast<size_t>(bytes), false));
    cuda_check(cudaHostRegister(p, static_cast<size_t>(bytes), cudaHostRegisterPortable | cudaHostRegisterMapped),
               "cudaHostRegister(peer host region)");
    R.peer_host[r] = p;
  }
  return R.peer_host[r];
}

// `range` (optional) receives the allocation's base and size in this
// process, published beside the handle so importers can tell stale mappings
void ipc_handle_of(const void *ptr, cudaIpcMemHandle_t *h, int64_t *offset, uint64_t *range = nullptr) {
  // handles name whole allocations; carry the offset inside it separately.
  // One driver query gives the allocation's process-unique buffer id, its
  // base and its memory type; the handle itself (cudaIpcGetMemHandle, the
  // expensive part) is cached per buffer id -- ids are never reused, so a
  // freed and re-made allocation at the same address gets a fresh handle.
  // A repeated neighbour call asks for its receive buffer's handle each time.
  using GetAttrs = int (*)(unsigned, int *, void **, uint64_t);
  static GetAttrs get_attrs = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuPointerGetAttributes", &fn, cudaEnableDefault, &q);
    return reinterpret_cast<GetAttrs>(fn);
  }();
  constexpr int kMemoryType = 2, kBufferId = 7, kRangeStart = 11, kRangeSize = 12, kDeviceMemory = 2; // cuda.h enums
  unsigned mtype = 0;
  unsigned long long id = 0;
  uint64_t base = 0;
  size_t span = 0;
  int which[4] = {kMemoryType, kBufferId, kRangeStart, kRangeSize};
  void *vals[4] = {&mtype, &id, &base, &span};
  if (!get_attrs || get_attrs(4, which, vals, reinterpret_cast<uint64_t>(ptr)) != 0)
    fail(SP_ERR_CUDA, "cuPointerGetAttributes failed");
  if (mtype != kDeviceMemory || !base) fail(SP_ERR_INVALID_ARGUMENT, "IPC export needs device memory");
  static std::mutex mu;
  static std::map<unsigned long long, cudaIpcMemHandle_t> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(id);
    if (it == cache.end()) {
      cudaIpcMemHandle_t nh{};
      cuda_check(cudaIpcGetMemHandle(&nh, reinterpret_cast<void *>(base)), "cudaIpcGetMemHandle");
      if (cache.size() >= 4096) cache.clear();
      it = cache.emplace(id, nh).first;
    }
    *h = it->second;
  }
  *offset = static_cast<const uint8_t *>(ptr) - reinterpret_cast<const uint8_t *>(base);
  if (range) {
    range[0] = base;
    range[1] = span;
  }
}

} // namespace

// ------------------------------------------------------------ lifecycle
void rt_init(int rank, int size, const char *name, int device, int64_t window_bytes, int64_t host_bytes) {
  if (g_rt) fail(SP_ERR_INVALID_ARGUMENT, "runtime already initialised");
  if (size < 1 || size > kMaxRanks || rank < 0 || rank >= size) fail(SP_ERR_INVALID_ARGUMENT, "bad rank/size");
  if (!name || !*name) fail(SP_ERR_INVALID_ARGUMENT, "runtime needs a job name");
  auto R = std::make_unique<Runtime>();
  R->rank = rank;
  R->size = size;
  R->device = device;
  R->name = std::string("/spb200_") + name;
  R->shm_bytes = sizeof(Shm);
  R->peer_window.assign(size, nullptr);
  R->peer_host.assign(size, nullptr);
  if (rank == 0) shm_unlink(R->name.c_str()); // a stale segment of an earlier job
  R->shm = static_cast<Shm *>(map_shm(R->name, R->shm_bytes, rank == 0));
  g_rt = R.release();
  Runtime &G = *g_rt;
  if (rank == 0) {
    G.shm->size = size;
    std::atomic_thread_fence(std::memory_order_release);
    reinterpret_cast<std::atomic<uint64_t> *>(&G.shm->magic)->store(kMagic, std::memory_order_release);
  } else {
    Waiter w("runtime bootstrap (rank 0)");
    while (reinterpret_cast<std::atomic<uint64_t> *>(&G.shm->magic)->load(std::memory_order_acquire) != kMagic)
      w.pause();
  }
  Slot &me = G.shm->slots[rank];
  me.pid = static_cast<int32_t>(getpid());
  me.device = device;
  if (device >= 0) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    std::memcpy(me.uuid, prop.uuid.bytes, sizeof(me.uuid));
    // blocking streams: a call that writes or reads a user buffer runs after
    // everything the application issued before it on the legacy default
    // stream (cudaMemset / cudaMemcpy / <<<>>> launches), as users of a
    // CUDA-aware MPI expect; work on the application's own non-blocking
    // streams still needs the application's synchronisation
    cuda_check(cudaStreamCreate(&G.stream), "cudaStreamCreate");
    cuda_check(cudaStreamCreate(&G.rstream), "cudaStreamCreate");
    if (window_bytes > 0) {
      cuda_check(cudaMalloc(&G.window, static_cast<size_t>(window_bytes)), "cudaMalloc(window)");
      cuda_check(cudaIpcGetMemHandle(&me.window, G.window), "cudaIpcGetMemHandle(window)");
      G.window_bytes = window_bytes;
    }
    if (host_bytes > 0) {
      const std::string hn = host_name(G.name, rank);
      shm_unlink(hn.c_str());
      G.host = static_cast<uint8_t *>(map_shm(hn, static_cast<size_t>(host_bytes), true));
      cuda_check(cudaHostRegister(G.host, static_cast<size_t>(host_bytes),
                                  cudaHostRegisterPortable | cudaHostRegisterMapped),
                 "cudaHostRegister(host region)");
      G.host_bytes = host_bytes;
    }
  }
  me.window_bytes = G.window_bytes;
  me.host_bytes = G.host_bytes;
  engine_init(G.window_bytes, G.host_bytes);
  G.pair_sent.assign(size, 0);
  G.pair_recv.assign(size, 0);
  if (device >= 0) {
    cuda_check(cudaMalloc(&G.nbr_flags, kMaxRanks * sizeof(uint64_t)), "cudaMalloc(nbr flags)");
    cuda_check(cudaMemset(G.nbr_flags, 0, kMaxRanks * sizeof(uint64_t)), "cudaMemset(nbr flags)");
    cuda_check(cudaHostAlloc(reinterpret_cast<void **>(&G.err_host), sizeof(int), cudaHostAllocMapped),
               "cudaHostAlloc(device wait error flag)");
    *G.err_host = 0;
    cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void **>(&G.err_dev), G.err_host, 0),
               "cudaHostGetDevicePointer");
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  }
  me.ready.store(1, std::memory_order_release);
  rt_barrier();
  if (device >= 0)
    for (int r = 0; r < size; ++r)
      if (r != rank && G.shm->slots[r].device >= 0 && !std::memcmp(G.shm->slots[r].uuid, me.uuid, sizeof(me.uuid)))
        G.shared_device = true;
  rt_exchange_ptr(G.nbr_flags, G.peer_nbr_flags);
  rt_pin_ptrs(G.peer_nbr_flags, 1 << 20); // the neighbour READY counters stay mapped until finalize
  // system-scope flags whenever any peer runs on another GPU: by UUID (device
  // ordinals are per process under CUDA_VISIBLE_DEVICES), and by where the
  // peer's mapped flags live
  if (device >= 0)
    for (int r = 0; r < size; ++r) {
      if (r != rank && G.shm->slots[r].device >= 0 && std::memcmp(G.shm->slots[r].uuid, me.uuid, sizeof(me.uuid)))
        G.nbr_remote = true;
      cudaPointerAttributes at{};
      if (G.peer_nbr_flags[r] && cudaPointerGetAttributes(&at, G.peer_nbr_flags[r]) == cudaSuccess &&
          at.device != device)
        G.nbr_remote = true;
    }
  cudaGetLastError();
}

void nbr_reset();

void rt_finalize() {
  if (!g_rt) return;
  rt_barrier();
  nbr_reset();
  Runtime &R = *g_rt;
  for (auto &kv : R.ipc_cache) cudaIpcCloseMemHandle(kv.second.p);
  for (int r = 0; r < R.size; ++r)
    if (R.peer_host[r] && r != R.rank) {
      cudaHostUnregister(R.peer_host[r]);
      munmap(R.peer_host[r], static_cast<size_t>(R.shm->slots[r].host_bytes));
    }
  rt_barrier();
  if (R.window) cudaFree(R.window);
  if (R.nbr_flags) cudaFree(R.nbr_flags);
  if (R.err_host) cudaFreeHost(R.err_host);
  if (R.host) {
    cudaHostUnregister(R.host);
    munmap(R.host, static_cast<size_t>(R.host_bytes));
    shm_unlink(host_name(R.name, R.rank).c_str());
  }
  engine_fini();
  if (R.stream) cudaStreamDestroy(R.stream);
  if (R.rstream) cudaStreamDestroy(R.rstream);
  const bool last = R.rank == 0;
  const std::string nm = R.name;
  munmap(R.shm, R.shm_bytes);
  if (last) shm_unlink(nm.c_str());
  delete g_rt;
  g_rt = nullptr;
}

uint64_t rt_device_timeout_ns() {
  const double t = timeout_s();
  return t > 0 ? static_cast<uint64_t>(t * 1e9) : 0;
}

int *rt_device_err() { return rt().err_dev; }

bool rt_peers_remote() { return rt().nbr_remote; }

void rt_check_device_error(const char *what) {
  Runtime &R = rt();
  if (R.err_host && *reinterpret_cast<volatile int *>(R.err_host)) {
    *R.err_host = 0;
    fail(SP_ERR_TIMEOUT, std::string(what) + ": an in-kernel wait for a peer's flag gave up after TEMPI_TIMEOUT=" +
                             std::to_string(timeout_s()) + " s (a peer rank died or never entered the call)");
  }
}

// Stream work that waits on peers' flags (stream memory operations) cannot
// time out on the device: the host polls its completion event like any other
// wait on the peers, so a dead or absent peer becomes SP_ERR_TIMEOUT.
void rt_sync_event(cudaEvent_t e, const char *what) {
  Waiter w(what);
  for (;;) {
    const cudaError_t q = cudaEventQuery(e);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) cuda_check(q, what);
    w.pause();
  }
}

// Where a launch waits for its peers' flags. In the kernel (every block
// spins on an acquire load) is the fastest, and safe when every rank has its
// own GPU: a peer's grid never competes for this GPU's SMs. When ranks share
// a GPU (MPS, or time-sliced processes), one rank's spinning full-wave grid
// can hold every SM the peer's kernel needs, so the waits move into the
// stream's front end (stream memory operations). TEMPI_FLAG_WAIT=stream |
// kernel overrides the choice.
bool rt_flag_waits_in_stream() {
  static const int forced = [] {
    const char *e = std::getenv("TEMPI_FLAG_WAIT");
    if (!e || !*e) return -1;
    if (!std::strcmp(e, "stream")) return 1;
    if (!std::strcmp(e, "kernel")) return 0;
    return -1;
  }();
  return forced >= 0 ? forced == 1 : rt().shared_device;
}

int rt_rank() { return rt().rank; }
int rt_size() { return rt().size; }

// sense-reversing barrier on two shared counters
void rt_barrier() {
  Runtime &R = rt();
  const uint32_t gen = R.shm->generation.load(std::memory_order_acquire);
  if (R.shm->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<uint32_t>(R.size)) {
    R.shm->arrived.store(0, std::memory_order_relaxed);
    R.shm->generation.store(gen + 1, std::memory_order_release);
  } else {
    Waiter w("barrier");
    while (R.shm->generation.load(std::memory_order_acquire) == gen) {
      rt_progress(); // pending non-blocking messages keep moving
      w.pause();
    }
  }
}

void rt_host_send(int dst, int tag, const void *data, int64_t bytes) {
  // small control payloads ride in the message itself (up to 16 bytes)
  if (bytes < 0 || bytes > 16) fail(SP_ERR_INVALID_ARGUMENT, "control payload > 16 bytes");
  Msg m{kFIN + 1, rt().rank, tag, 0, bytes, 0, 0};
  std::memcpy(&m.offset, data, static_cast<size_t>(bytes));
  post(dst, m);
}

int64_t rt_host_recv(int src, int tag, void *data, int64_t cap) {
  const Msg m = wait_msg(kFIN + 1, src, tag);
  std::memcpy(data, &m.offset, static_cast<size_t>(std::min(cap, m.bytes)));
  return m.bytes;
}

// collective: every rank contributes one device pointer; returns all of
// them mapped into this process (own pointer for self)
void rt_exchange_ptr(void *local, std::vector<uint8_t *> &out) {
  Runtime &R = rt();
  ipc_call_begin();
  Slot &me = R.shm->slots[R.rank];
  // the publication area is the one a neighbour collective's receive layout
  // uses: the next collective must publish its layout again
  R.nbr_layout.clear();
  if (local) {
    ipc_handle_of(local, &me.xh, &me.xoff, me.xr);
    me.xbytes = 1;
  } else {
    me.xbytes = 0;
  }
  rt_barrier();
  out.assign(R.size, nullptr);
  for (int r = 0; r < R.size; ++r) {
    if (r == R.rank) {
      out[r] = static_cast<uint8_t *>(local);
    } else if (R.shm->slots[r].xbytes) {
      const Slot &sl = R.shm->slots[r];
      out[r] = open_ipc(sl.xh, r, sl.xr) + sl.xoff;
      R.exchanged[out[r]] = std::string(reinterpret_cast<const char *>(&R.shm->slots[r].xh), sizeof(cudaIpcMemHandle_t));
    }
  }
  rt_barrier();
}

// ------------------------------------------------------------ point to point
// Non-blocking rendezvous with a progress engine (MPI_Isend / MPI_Irecv;
// the blocking calls are isend/irecv + wait). Per message:
//   sender   RTS(method, bytes, direct-capable)          -> receiver
//   receiver CTS(method', offset of its grant)           -> sender
//   sender   CHUNK(k of n, packed bytes [lo, hi)) ...    -> receiver
// Transfer methods (the model picks the first three):
//   DEVICE : pack kernel -> receiver's device window through CUDA IPC
//            (NVLink); the receiver unpacks from its own HBM
//   ONESHOT: pack kernel -> receiver's shared pinned host region (mapped);
//            the receiver's unpack kernel reads host memory directly
//   STAGED : pack kernel -> local device scratch -> D2H into the receiver's
//            host region; the receiver copies H2D, then unpacks
//   DIRECT : the receiver upgrades a DEVICE message whose destination is
//            device memory: it publishes its buffer (IPC) and the canonical
//            geometry of its type, and the sender runs ONE typed-copy kernel
//            that stores every byte at its final strided address in the
//            receiver's HBM -- pack, NVLink transfer and unpack fused, no
//            window, no unpack launch.
// Messages above two chunks (TEMPI_CHUNK / sp_rt_set_chunk, default 4 MiB)
// move in chunks of the packed stream: the sender reports each chunk as its
// event completes, and the receiver unpacks (STAGED: copies in and unpacks)
// chunk k while the sender is still producing chunk k+1, so packing, the
// link and unpacking overlap. Grants are carved out of the receiver's window
// / host region by a first-fit allocator, so several messages can be in
// flight to one rank.
namespace {

constexpr uint32_t kCHUNK = 5;
constexpr int64_t kOfferForced = 4; // RTS offer flag: DIRECT was asked for explicitly
constexpr int64_t kGrantAlign = 256;

struct RangeAlloc {
  std::map<int64_t, int64_t> free_; // offset -> length
  void reset(int64_t cap) {
    free_.clear();
    if (cap > 0) free_[0] = cap;
  }
  int64_t take(int64_t n) {
    n = std::max<int64_t>(kGrantAlign, (n + kGrantAlign - 1) / kGrantAlign * kGrantAlign);
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second < n) continue;
      const int64_t off = it->first, len = it->second;
      free_.erase(it);
      if (len > n) free_[off + n] = len - n;
      return off;
    }
    return -1;
  }
  void give(int64_t off, int64_t n) {
    n = std::max<int64_t>(kGrantAlign, (n + kGrantAlign - 1) / kGrantAlign * kGrantAlign);
    auto it = free_.emplace(off, n).first;
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_.erase(nx);
    }
    if (it != free_.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        free_.erase(it);
      }
    }
  }
};

enum class St { Start, WaitCts, Streaming, WaitRts, Matched, Receiving, Draining, Done };

struct Req {
  uint64_t id = 0;
  bool send = false;
  St st = St::Start;
  const void *sbuf = nullptr;
  void *rbuf = nullptr;
  uint64_t buf_bytes = 0;
  int64_t count = 0;
  CommitPtr ct;
  int peer = -1, tag = 0, method = 0;
  bool allow_direct = false;
  bool forced_direct = false; // the sender asked for DIRECT explicitly (no model veto)
  int64_t bytes = 0;
  // sender
  uint64_t rreq = 0;
  int64_t grant = 0;
  int nchunks = 0, reported = 0;
  std::vector<std::pair<int64_t, int64_t>> chunks;
  std::vector<cudaEvent_t> evs;
  uint8_t *scratch = nullptr;
  // receiver
  int src_want = -1, tag_want = -1;
  uint64_t sreq = 0;
  int region = 0; // 1 window, 2 host region, 3 descriptor
  int got = 0, expect = -1;
  bool ranged = false;
  uint8_t *rbuf_stage = nullptr;
  cudaEvent_t last = nullptr;
  RtStatus status{};
  // completion
  sp_status err = SP_OK;
  std::string msg;
};

struct Engine {
  uint64_t next_id = 1;
  std::deque<std::unique_ptr<Req>> active;      // posting order
  std::map<uint64_t, std::unique_ptr<Req>> done; // completed, not yet waited
  std::vector<cudaEvent_t> pool;
  RangeAlloc win, host;
  uint32_t desc_used = 0; // bitmap of this rank's published descriptors
  int64_t chunk = int64_t{4} << 20;
  bool in_progress = false;
};
Engine *g_eng = nullptr;

Engine &eng() {
  if (!g_eng) fail(SP_ERR_INVALID_ARGUMENT, "runtime not initialised (sp_rt_init)");
  return *g_eng;
}

cudaEvent_t get_event() {
  Engine &E = eng();
  if (!E.pool.empty()) {
    cudaEvent_t e = E.pool.back();
    E.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  return e;
}

void put_event(cudaEvent_t e) {
  if (e) eng().pool.push_back(e);
}

bool event_done(cudaEvent_t e) {
  const cudaError_t q = cudaEventQuery(e);
  if (q == cudaSuccess) return true;
  if (q == cudaErrorNotReady) return false;
  cuda_check(q, "cudaEventQuery");
  return false;
}

// first message of `kind` from `src` addressed to request `id`
bool take(uint32_t kind, int src, uint64_t id, Msg &out) {
  Runtime &R = rt();
  for (auto it = R.unexpected.begin(); it != R.unexpected.end(); ++it)
    if (it->kind == kind && it->src == src && static_cast<uint64_t>(it->aux) == id) {
      out = *it;
      R.unexpected.erase(it);
      return true;
    }
  return false;
}

std::vector<std::pair<int64_t, int64_t>> chunk_plan(int64_t bytes) {
  const int64_t c = eng().chunk;
  std::vector<std::pair<int64_t, int64_t>> out;
  if (bytes <= 2 * c) {
    out.emplace_back(0, bytes);
    return out;
  }
  for (int64_t lo = 0; lo < bytes; lo += c) out.emplace_back(lo, std::min(bytes, lo + c));
  return out;
}

void committed_from(const Desc &d, Committed &c) {
  c.form = SP_FORM_STRIDED;
  c.size = d.size;
  c.extent = d.extent;
  c.span = d.span;
  c.overlapping = false;
  c.sb.start = d.start;
  c.sb.counts.assign(d.counts, d.counts + d.ndims);
  c.sb.strides.assign(d.strides, d.strides + d.ndims);
}

bool describable(const Committed &ct) {
  return ct.form == SP_FORM_STRIDED && !ct.overlapping && ct.sb.ndims() <= kDescDims;
}

// ---- sender
void send_stream(Req &q) {
  Runtime &R = rt();
  ipc_call_begin();
  const cudaStream_t s = R.stream;
  if (q.bytes == 0) {
    q.chunks.assign(1, {0, 0});
  } else if (q.method == SP_METHOD_DIRECT) {
    const Desc &d = R.shm->slots[q.peer].desc[q.grant];
    Committed dst;
    committed_from(d, dst);
    uint8_t *base = q.peer == R.rank ? reinterpret_cast<uint8_t *>(d.raw) : open_ipc(d.h, q.peer, d.hr) + d.off;
    if (q.ct->form != SP_FORM_STRIDED) { // block-list send type: pack into the dense receive run
      PackArgs a{};
      a.ct = q.ct.get();
      a.src = q.sbuf;
      a.src_bytes = q.buf_bytes;
      a.dst = base + d.start;
      a.dst_bytes = static_cast<uint64_t>(q.bytes);
      a.count = q.count;
      a.stream = s;
      a.opt = sp_pack_options{1, SP_KERNEL_AUTO, 0};
      a.pack = true;
      execute(a);
    } else {
      const CopySpec spec{q.ct.get(), q.sbuf, q.buf_bytes, q.count, &dst, base, UINT64_MAX, d.count};
      copy_execute(spec, 0, static_cast<uint64_t>(q.bytes), s);
    }
    q.chunks.assign(1, {0, q.bytes});
  } else {
    uint8_t *dst = nullptr;
    if (q.method == SP_METHOD_DEVICE) {
      dst = peer_window(q.peer) + q.grant;
    } else if (q.method == SP_METHOD_ONESHOT) {
      dst = peer_host(q.peer) + q.grant;
    } else {
      cuda_check(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&q.scratch), static_cast<size_t>(q.bytes), engine_pool(), s),
                 "cudaMallocAsync(staged)");
      dst = q.scratch;
    }
    const bool ranged = range_capable(*q.ct, q.count, q.sbuf, dst);
    q.chunks = ranged ? chunk_plan(q.bytes) : std::vector<std::pair<int64_t, int64_t>>{{0, q.bytes}};
    const BatchSpec spec{q.ct.get(), q.sbuf, q.buf_bytes, q.count, dst, static_cast<uint64_t>(q.bytes), 0};
    for (auto [lo, hi] : q.chunks) {
      if (ranged) {
        range_execute(spec, false, static_cast<uint64_t>(lo), static_cast<uint64_t>(hi), s);
      } else {
        PackArgs a{};
        a.ct = q.ct.get();
        a.src = q.sbuf;
        a.src_bytes = q.buf_bytes;
        a.count = q.count;
        a.dst = dst;
        a.dst_bytes = static_cast<uint64_t>(q.bytes);
        a.stream = s;
        a.opt = sp_pack_options{1, SP_KERNEL_AUTO, 0};
        a.pack = true;
        execute(a);
      }
      if (q.method == SP_METHOD_STAGED)
        cuda_check(cudaMemcpyAsync(peer_host(q.peer) + q.grant + lo, q.scratch + lo, static_cast<size_t>(hi - lo),
                                   cudaMemcpyDeviceToHost, s),
                   "staged D2H");
      cudaEvent_t e = get_event();
      cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
      q.evs.push_back(e);
    }
    if (q.scratch) {
      cuda_check(cudaFreeAsync(q.scratch, s), "cudaFreeAsync(staged)");
      q.scratch = nullptr;
    }
  }
  if (q.evs.empty()) { // nothing was launched (empty message) or DIRECT
    cudaEvent_t e = get_event();
    cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
    q.evs.push_back(e);
  }
  q.nchunks = static_cast<int>(q.chunks.size());
}

bool step_send(Req &q) {
  Runtime &R = rt();
  switch (q.st) {
  case St::Start: {
    // DIRECT travels as an upgrade offer on the fallback method's request:
    // the sender can run the copy kernel when its source is
    // device-accessible, the receiver accepts when its buffer is device
    // memory, and otherwise the fallback (the model's choice, or DEVICE
    // for an explicit DIRECT) moves the message
    // offer 1: a strided send type (typed copy into any describable
    // receive layout); offer 2: a block-list send type (run-table pack,
    // needs a receive layout that is one dense run)
    int offer = 0;
    if (q.bytes > 0 && q.allow_direct) {
      if (q.ct->form == SP_FORM_STRIDED && range_capable(*q.ct, q.count, q.sbuf, q.sbuf)) offer = 1;
      if (q.ct->form == SP_FORM_UNSUPPORTED) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, q.sbuf) == cudaSuccess && at.type == cudaMemoryTypeDevice) offer = 2;
        cudaGetLastError();
      }
    }
    if (offer && q.forced_direct) offer |= kOfferForced;
    post(q.peer, Msg{kRTS, R.rank, q.tag, q.method, q.bytes, offer, static_cast<int64_t>(q.id)});
    q.st = St::WaitCts;
    return true;
  }
  case St::WaitCts: {
    Msg m;
    if (!take(kCTS, q.peer, q.id, m)) return false;
    q.method = m.method;
    q.grant = m.offset;
    q.rreq = static_cast<uint64_t>(m.tag);
    q.bytes = m.bytes; // 0 when the receiver refused the message (truncation)
    send_stream(q);
    q.st = St::Streaming;
    return true;
  }
  case St::Streaming: {
    bool moved = false;
    while (q.reported < static_cast<int>(q.evs.size()) && event_done(q.evs[q.reported])) {
      const int k = q.reported;
      const auto [lo, hi] = k < static_cast<int>(q.chunks.size()) ? q.chunks[k] : std::pair<int64_t, int64_t>{0, 0};
      post(q.peer, Msg{kCHUNK, R.rank, k, q.nchunks, hi, lo, static_cast<int64_t>(q.rreq)});
      ++q.reported;
      moved = true;
    }
    if (q.reported == static_cast<int>(q.evs.size())) {
      for (auto e : q.evs) put_event(e);
      q.evs.clear();
      q.st = St::Done;
    }
    return moved;
  }
  default:
    return false;
  }
}

// ---- receiver
bool step_recv(Req &q) {
  Runtime &R = rt();
  Engine &E = eng();
  const cudaStream_t s = R.rstream;
  switch (q.st) {
  case St::WaitRts: {
    for (auto it = R.unexpected.begin(); it != R.unexpected.end(); ++it) {
      if (it->kind != kRTS || (q.src_want >= 0 && it->src != q.src_want) || (q.tag_want >= 0 && it->tag != q.tag_want))
        continue;
      const Msg m = *it;
      R.unexpected.erase(it);
      q.peer = m.src;
      q.tag = m.tag;
      q.method = m.method;
      q.bytes = m.bytes;
      q.sreq = static_cast<uint64_t>(m.aux);
      q.status = RtStatus{m.src, m.tag, m.method, m.bytes};
      if (m.bytes > q.count * q.ct->size) {
        q.err = SP_ERR_BUFFER_TOO_SMALL;
        q.msg = "recv: message truncated (MPI_ERR_TRUNCATE)";
      } else if (m.bytes > 0 && (q.ct->size == 0 || m.bytes % q.ct->size)) {
        q.err = SP_ERR_INVALID_ARGUMENT;
        q.msg = "recv: message is not whole objects";
      } else if (m.bytes > 0 &&
                 static_cast<uint64_t>((m.bytes / q.ct->size - 1) * q.ct->extent + q.ct->span) > q.buf_bytes) {
        // every method writes the receive buffer through the layout (DIRECT
        // straight from the sender's kernel): check it before any transfer
        q.err = SP_ERR_BUFFER_TOO_SMALL;
        q.msg = "recv: receive buffer smaller than the layout of the message";
      }
      // DIRECT upgrade: the sender can run the copy kernel, the destination
      // is device memory and the type has a publishable canonical form
      const int64_t objs = q.ct->size ? m.bytes / q.ct->size : 0;
      const bool dense = q.ct->form == SP_FORM_STRIDED && q.ct->sb.ndims() == 1 &&
                         (objs <= 1 || q.ct->extent == q.ct->size);
      const int64_t offer = m.offset & 3;
      if (!q.err && ((offer == 1 && describable(*q.ct) && range_capable(*q.ct, objs, q.rbuf, q.rbuf)) ||
                     (offer == 2 && dense && describable(*q.ct)))) {
        cudaPointerAttributes at{};
        const bool dev = cudaPointerGetAttributes(&at, q.rbuf) == cudaSuccess && at.type == cudaMemoryTypeDevice;
        cudaGetLastError();
        // the fused copy stores every destination row as its own write (over
        // NVLink when the sender is on another GPU): the receiver's layout
        // has a say too -- a model-offered DIRECT is accepted only when the
        // model, asked with this side's geometry, also prefers it
        const bool model_ok = (m.offset & kOfferForced) || model_prefers_direct(*q.ct, objs, m.src);
        if (dev && model_ok) q.method = SP_METHOD_DIRECT; // a descriptor slot is taken at the grant
      }
      q.st = St::Matched;
      return true;
    }
    return false;
  }
  case St::Matched: {
    if (q.err) { // release the sender without a transfer; the error surfaces at wait
      post(q.peer, Msg{kCTS, R.rank, static_cast<int32_t>(q.id), SP_METHOD_DEVICE, 0, 0, static_cast<int64_t>(q.sreq)});
      q.bytes = 0;
      q.st = St::Receiving;
      return true;
    }
    int64_t grant = 0;
    if (q.bytes == 0) {
      q.region = 0;
    } else if (q.method == SP_METHOD_DIRECT && E.desc_used == ~0u) {
      // every descriptor slot is held by a DIRECT message still in flight:
      // this one moves by the sender's fallback method instead
      q.method = q.status.method;
      return true; // Matched again with the fallback
    } else if (q.method == SP_METHOD_DIRECT) {
      int slot = 0;
      while (E.desc_used & (1u << slot)) ++slot;
      Desc &d = R.shm->slots[R.rank].desc[slot];
      const Committed &c = *q.ct;
      d.ndims = c.sb.ndims();
      d.start = c.sb.start;
      for (int i = 0; i < d.ndims; ++i) {
        d.counts[i] = c.sb.counts[i];
        d.strides[i] = c.sb.strides[i];
      }
      d.size = c.size;
      d.extent = c.extent;
      d.span = c.span;
      d.count = q.bytes / c.size;
      d.raw = reinterpret_cast<uint64_t>(q.rbuf);
      ipc_handle_of(q.rbuf, &d.h, &d.off, d.hr);
      E.desc_used |= 1u << slot;
      q.region = 3;
      grant = slot;
    } else if (q.method == SP_METHOD_DEVICE) {
      if (q.bytes > R.window_bytes) {
        q.err = SP_ERR_UNSUPPORTED;
        q.msg = "recv: message larger than the receive window and not deliverable directly";
        return true; // Matched again: refuses with a zero-byte grant
      }
      grant = E.win.take(q.bytes);
      if (grant < 0) return false; // window busy: grant later
      q.region = 1;
    } else {
      if (q.bytes > R.host_bytes) {
        q.err = SP_ERR_UNSUPPORTED;
        q.msg = "recv: message larger than the host region and not deliverable directly";
        return true; // Matched again: refuses with a zero-byte grant
      }
      grant = E.host.take(q.bytes);
      if (grant < 0) return false;
      q.region = 2;
    }
    q.grant = grant;
    if (q.method == SP_METHOD_STAGED && q.bytes > 0)
      cuda_check(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&q.rbuf_stage), static_cast<size_t>(q.bytes), engine_pool(), s),
                 "cudaMallocAsync(staged)");
    const uint8_t *packed = q.method == SP_METHOD_DEVICE   ? R.window + grant
                            : q.method == SP_METHOD_STAGED ? q.rbuf_stage
                                                           : R.host + grant;
    q.ranged = q.bytes > 0 && q.method != SP_METHOD_DIRECT && range_capable(*q.ct, q.bytes / q.ct->size, q.rbuf, packed);
    post(q.peer, Msg{kCTS, R.rank, static_cast<int32_t>(q.id), q.method, q.bytes, grant, static_cast<int64_t>(q.sreq)});
    q.st = St::Receiving;
    return true;
  }
  case St::Receiving: {
    bool moved = false;
    Msg m;
    while (take(kCHUNK, q.peer, q.id, m)) {
      moved = true;
      q.expect = m.method;
      ++q.got;
      const int64_t lo = m.offset, hi = m.bytes;
      if (q.bytes == 0 || q.method == SP_METHOD_DIRECT) continue;
      const int64_t n = q.bytes / q.ct->size;
      const uint8_t *src = q.method == SP_METHOD_DEVICE ? R.window + q.grant
                           : q.method == SP_METHOD_STAGED ? q.rbuf_stage
                                                          : R.host + q.grant;
      if (q.method == SP_METHOD_STAGED)
        cuda_check(cudaMemcpyAsync(q.rbuf_stage + lo, R.host + q.grant + lo, static_cast<size_t>(hi - lo),
                                   cudaMemcpyHostToDevice, s),
                   "staged H2D");
      if (q.ranged) {
        const BatchSpec spec{q.ct.get(), src, static_cast<uint64_t>(q.bytes), n, q.rbuf, q.buf_bytes, 0};
        range_execute(spec, true, static_cast<uint64_t>(lo), static_cast<uint64_t>(hi), s);
      } else if (q.got == q.expect) {
        PackArgs a{};
        a.ct = q.ct.get();
        a.src = src;
        a.src_bytes = static_cast<uint64_t>(q.bytes);
        a.dst = q.rbuf;
        a.dst_bytes = q.buf_bytes;
        a.count = n;
        a.stream = s;
        a.opt = sp_pack_options{1, SP_KERNEL_AUTO, 0};
        a.pack = false;
        execute(a);
      }
    }
    if (q.expect >= 0 && q.got == q.expect) {
      if (q.rbuf_stage) {
        cuda_check(cudaFreeAsync(q.rbuf_stage, s), "cudaFreeAsync(staged)");
        q.rbuf_stage = nullptr;
      }
      if (q.bytes > 0 && q.method != SP_METHOD_DIRECT) {
        q.last = get_event();
        cuda_check(cudaEventRecord(q.last, s), "cudaEventRecord");
      }
      // DIRECT (and an empty message) enqueued nothing here: the sender's
      // kernel had completed before its CHUNK was posted
      q.st = St::Draining;
      moved = true;
    }
    return moved;
  }
  case St::Draining: {
    if (q.last) {
      if (!event_done(q.last)) return false;
      put_event(q.last);
      q.last = nullptr;
    }
    if (q.region == 1) E.win.give(q.grant, q.bytes);
    if (q.region == 2) E.host.give(q.grant, q.bytes);
    if (q.region == 3) E.desc_used &= ~(1u << q.grant);
    q.region = 0;
    q.st = St::Done;
    return true;
  }
  default:
    return false;
  }
}

} // namespace

// one pass over every active request; requests that finish move to `done`
void rt_progress() {
  Engine &E = eng();
  if (E.in_progress) return;
  E.in_progress = true;
  struct Reset {
    bool &f;
    ~Reset() { f = false; }
  } reset{E.in_progress};
  drain();
  bool moved = true;
  while (moved) {
    moved = false;
    for (auto it = E.active.begin(); it != E.active.end();) {
      Req &q = **it;
      try {
        moved = (q.send ? step_send(q) : step_recv(q)) || moved;
      } catch (const Error &e) {
        q.err = e.code;
        q.msg = e.msg;
        q.st = St::Done;
      }
      if (q.st == St::Done) {
        E.done[q.id] = std::move(*it);
        it = E.active.erase(it);
        moved = true;
      } else {
        ++it;
      }
    }
    if (moved) drain();
  }
}

void engine_init(int64_t window_bytes, int64_t host_bytes) {
  delete g_eng;
  g_eng = new Engine;
  g_eng->win.reset(window_bytes);
  g_eng->host.reset(host_bytes);
  if (const char *c = std::getenv("TEMPI_CHUNK")) {
    const int64_t v = std::atoll(c);
    if (v >= 16 && v % 16 == 0) g_eng->chunk = v;
  }
}

void engine_fini() {
  if (!g_eng) return;
  for (cudaEvent_t e : g_eng->pool) cudaEventDestroy(e);
  delete g_eng;
  g_eng = nullptr;
}

uint64_t rt_isend(const void *buf, uint64_t buf_bytes, int64_t count, CommitPtr ct, int dest, int tag, int method) {
  Runtime &R = rt();
  Engine &E = eng();
  if (dest < 0 || dest >= R.size) fail(SP_ERR_INVALID_ARGUMENT, "send: bad destination rank");
  if (tag < 0) fail(SP_ERR_INVALID_ARGUMENT, "send: negative tag");
  const int64_t bytes = count * ct->size;
  // model-selected messages (method < 0) and explicit DIRECT offer the
  // fused copy to the receiver; the model's choice (DEVICE for an explicit
  // DIRECT) is the fallback when the receive buffer is not device memory.
  // On B200 the fused copy wins at every size measured (one kernel, no
  // window, no unpack; bench.py `send`), which the paper's three-term
  // model cannot express.
  // DIRECT is offered when asked for explicitly, or when the B200 model
  // (Eq. 4, the measured gpu_direct / gpu_direct_peer surface of the
  // receiver's GPU) puts it ahead of the reference's three methods
  const bool forced_direct = method == SP_METHOD_DIRECT;
  bool allow_direct = forced_direct || (method < 0 && model_prefers_direct(*ct, count, dest));
  if (method < 0) method = rt_choose(*ct, count);
  if (method == SP_METHOD_DIRECT) method = SP_METHOD_DEVICE;
  if (method != SP_METHOD_DEVICE && method != SP_METHOD_ONESHOT && method != SP_METHOD_STAGED)
    fail(SP_ERR_INVALID_ARGUMENT, "send: unknown method");
  if (!allow_direct && method == SP_METHOD_DEVICE && bytes > R.shm->slots[dest].window_bytes)
    fail(SP_ERR_UNSUPPORTED, "send: message larger than the receive window");
  if (!allow_direct && method != SP_METHOD_DEVICE && bytes > R.shm->slots[dest].host_bytes)
    fail(SP_ERR_UNSUPPORTED, "send: message larger than the receiver's host region");
  auto q = std::make_unique<Req>();
  q->id = E.next_id++;
  q->send = true;
  q->sbuf = buf;
  q->buf_bytes = buf_bytes;
  q->count = count;
  q->ct = std::move(ct);
  q->peer = dest;
  q->tag = tag;
  q->method = method;
  q->allow_direct = allow_direct;
  q->forced_direct = forced_direct;
  q->bytes = bytes;
  q->st = St::Start;
  const uint64_t id = q->id;
  E.active.push_back(std::move(q));
  rt_progress();
  return id;
}

uint64_t rt_irecv(void *buf, uint64_t buf_bytes, int64_t count, CommitPtr ct, int source, int tag) {
  Runtime &R = rt();
  Engine &E = eng();
  if (source >= R.size) fail(SP_ERR_INVALID_ARGUMENT, "recv: bad source rank");
  auto q = std::make_unique<Req>();
  q->id = E.next_id++;
  q->rbuf = buf;
  q->buf_bytes = buf_bytes;
  q->count = count;
  q->ct = std::move(ct);
  q->src_want = source;
  q->tag_want = tag;
  q->st = St::WaitRts;
  const uint64_t id = q->id;
  E.active.push_back(std::move(q));
  rt_progress();
  return id;
}

// completes (and frees) request `id` if it has finished; rethrows its error
bool rt_test(uint64_t id, RtStatus *st) {
  Engine &E = eng();
  rt_progress();
  auto it = E.done.find(id);
  if (it == E.done.end()) {
    bool known = false;
    for (auto &q : E.active) known = known || q->id == id;
    if (!known) fail(SP_ERR_INVALID_HANDLE, "unknown request");
    return false;
  }
  std::unique_ptr<Req> q = std::move(it->second);
  E.done.erase(it);
  if (st) {
    *st = q->send ? RtStatus{q->peer, q->tag, q->method, q->bytes} : q->status;
    if (!q->send) st->method = q->method;
  }
  if (q->err) fail(q->err, q->msg);
  return true;
}

void rt_wait(uint64_t id, RtStatus *st) {
  Waiter w("MPI_Wait");
  while (!rt_test(id, st)) w.pause();
}

void rt_set_chunk(int64_t bytes) {
  if (bytes < 16 || bytes % 16) fail(SP_ERR_INVALID_ARGUMENT, "chunk size must be a positive multiple of 16");
  eng().chunk = bytes;
}

void rt_send(const void *buf, uint64_t buf_bytes, int64_t count, CommitPtr ct, int dest, int tag, int method,
             RtTrace *trace) {
  RtStatus st{};
  rt_wait(rt_isend(buf, buf_bytes, count, std::move(ct), dest, tag, method), &st);
  if (trace) {
    trace->method = st.method;
    trace->bytes = st.bytes;
  }
}

void rt_recv(void *buf, uint64_t buf_bytes, int64_t count, CommitPtr ct, int source, int tag, RtStatus *st) {
  rt_wait(rt_irecv(buf, buf_bytes, count, std::move(ct), source, tag), st);
}

void rt_set_profile(sp_profile_s *p) {
  Runtime &R = rt();
  R.profile = p ? p->p : nullptr;
  R.direct_cache.clear();
  sp_model_cache_s *c = nullptr;
  if (p) {
    if (sp_model_cache_create(p, &c) != SP_OK) fail(SP_ERR_INTERNAL, "model cache");
  }
  R.cache.reset(c);
}

// model query of a message: object = packed bytes, block = contiguous run
// (halo.hpp:296 uses the same pair)
int rt_choose(const Committed &ct, int64_t count) {
  Runtime &R = rt();
  if (!R.cache || ct.size == 0) return SP_METHOD_DEVICE;
  const int64_t obj = ct.size * count;
  // block size of the model query (halo.hpp:296 uses counts[0]); a
  // block-list form contributes its mean run length
  const int64_t blk = ct.form == SP_FORM_STRIDED
                          ? std::min(ct.sb.counts[0], obj)
                          : std::max<int64_t>(1, ct.runs.empty() ? 1 : ct.size / static_cast<int64_t>(ct.runs.size()));
  int m = SP_METHOD_DEVICE;
  if (sp_model_cache_choose(R.cache.get(), obj, blk, &m) != SP_OK) return SP_METHOD_DEVICE;
  return m;
}

// B200 model (Eq. 4) on DIRECT for `count` objects of `ct` moving between
// this GPU and a device buffer of rank `peer` (same GPU or peer GPU, told
// apart by UUID: ordinals are per process): true when the measured
// DIRECT surface of that destination is at least as
// fast as the reference's best method; without a profile DIRECT is the
// default (it measured fastest on B200 at every size, bench.py `send`);
// with a profile that lacks the surface, never.
bool model_prefers_direct(const Committed &ct, int64_t count, int peer) {
  Runtime &R = rt();
  if (!R.profile) return true;
  if (ct.size == 0 || count < 1) return false;
  const int64_t obj = ct.size * count;
  const int64_t blk = ct.form == SP_FORM_STRIDED
                          ? std::min(ct.sb.counts[0], obj)
                          : std::max<int64_t>(1, ct.runs.empty() ? 1 : ct.size / static_cast<int64_t>(ct.runs.size()));
  const bool same = peer == R.rank || !std::memcmp(R.shm->slots[peer].uuid, R.shm->slots[R.rank].uuid, 16);
  const int kind = same ? kDstSameGpu : kDstPeerGpu;
  const auto key = std::make_tuple(obj, blk, kind);
  auto it = R.direct_cache.find(key);
  if (it != R.direct_cache.end()) return it->second;
  const bool yes = choose_method_b200(*R.profile, obj, blk, kind, nullptr) == SP_METHOD_DIRECT;
  if (R.direct_cache.size() > 4096) R.direct_cache.clear();
  R.direct_cache.emplace(key, yes);
  return yes;
}

void *rt_stream() { return rt().stream; }

// ------------------------------------------------------------ neighbour exchange
// MPI_Neighbor_alltoallv over a distributed graph: every rank publishes its
// receive buffer (CUDA IPC) and the (source, offset, bytes) of each in-edge;
// each rank then runs ONE batch launch that packs every out-edge block with
// the send type straight into the matching receiver's buffer (the k-th edge
// to a rank matches that rank's k-th edge from us, MPI-3.1 §7.6), and a
// barrier publishes completion. Batches are cached per call signature, so
// an iterative halo loop re-launches a persistent plan.
namespace {
struct NbrCacheEntry {
  std::string key;
  Batch *batch;
};
std::deque<NbrCacheEntry> g_nbr_cache;
} // namespace

// Publishes this rank's receive layout for a neighbour call (IPC handle of
// the receive buffer, in-edges, and for alltoallw the receive geometries)
// and bumps layout_ver when it differs from the previous call's.
void nbr_publish(uint8_t *recvbuf, const std::vector<int> &sources, const std::vector<int64_t> &disp_bytes,
                 const std::vector<int64_t> &bytes, const std::vector<const Desc *> *wdesc) {
  Runtime &R = rt();
  Slot &me = R.shm->slots[R.rank];
  cudaIpcMemHandle_t h{};
  int64_t off = 0;
  const bool any = recvbuf != nullptr && std::any_of(bytes.begin(), bytes.end(), [](int64_t b) { return b > 0; });
  uint64_t xr[2] = {0, 0};
  if (any) ipc_handle_of(recvbuf, &h, &off, xr);
  std::string lay(reinterpret_cast<const char *>(&h), sizeof(h));
  lay.append(reinterpret_cast<const char *>(&off), sizeof(off));
  lay.push_back(any ? 1 : 0);
  for (size_t j = 0; j < sources.size(); ++j) {
    const int64_t e[3] = {sources[j], disp_bytes[j], bytes[j]};
    lay.append(reinterpret_cast<const char *>(e), sizeof(e));
    if (wdesc && (*wdesc)[j]) lay.append(reinterpret_cast<const char *>((*wdesc)[j]), sizeof(Desc));
  }
  if (lay == R.nbr_layout) return; // unchanged: peers keep their cached plans
  me.xh = h;
  me.xoff = off;
  me.xr[0] = xr[0];
  me.xr[1] = xr[1];
  me.xbytes = any ? 1 : 0;
  me.nedges = static_cast<int32_t>(sources.size());
  for (size_t j = 0; j < sources.size(); ++j) {
    me.edges[j][0] = sources[j];
    me.edges[j][1] = disp_bytes[j];
    me.edges[j][2] = bytes[j];
    if (wdesc && (*wdesc)[j]) me.wdesc[j] = *(*wdesc)[j];
  }
  R.nbr_layout = std::move(lay);
  me.layout_ver.fetch_add(1, std::memory_order_release);
}

// Last call of each neighbour collective: when a call repeats it (same
// arguments, every out-neighbour's layout version unchanged) the cached
// batch is relaunched without rebuilding jobs or cache keys.
// An out-edge whose send type has no strided form (an irregular indexed or
// struct type) into a receive layout that is one dense run: the run-table
// kernel packs it straight into the receiver's buffer -- all such edges of
// a call in one launch (k_runs_multi) -- ahead of the call's batch on the
// same stream, whose completion flags then cover it (stream order puts its
// stores before the batch's release).
struct LooseOp {
  CommitPtr ct;
  const uint8_t *src;
  int64_t count;
  uint8_t *dst; // receiver's bytes for this edge, already at their offset
  // a dense send run scattered through the receiver's run table (ct null)
  bool unpack = false;
  const int64_t *psrc = nullptr, *pdst = nullptr;
  int64_t npieces = 0, size = 0, extent = 0;
  uint64_t align = 0;
};

// Local copies of peers' run tables (a scattered-ghost edge reads its
// table once per piece; a copy in this GPU's HBM keeps those reads off
// NVLink). Owned by the call record that uses them; freed when it is
// replaced (every call ends with a stream synchronisation, so no launch
// still reads them).
struct TableCopy {
  void *p = nullptr;
  TableCopy() = default;
  explicit TableCopy(size_t bytes) { cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(run table copy)"); }
  TableCopy(const TableCopy &) = delete;
  TableCopy &operator=(const TableCopy &) = delete;
  ~TableCopy() {
    if (p) cudaFree(p);
  }
};

struct NbrLast {
  std::string sig;
  std::vector<std::pair<int, uint64_t>> peer_ver;
  Batch *batch = nullptr;
  std::vector<LooseOp> loose;
  std::vector<std::shared_ptr<TableCopy>> tables;
  bool valid = false;
};

NbrLast g_last_v, g_last_w;

bool nbr_peers_unchanged(const NbrLast &last) {
  Runtime &R = rt();
  for (auto [d, v] : last.peer_ver)
    if (R.shm->slots[d].layout_ver.load(std::memory_order_acquire) != v) return false;
  return true;
}

bool nbr_last_hit(const NbrLast &last, const std::string &sig) {
  if (!last.valid || last.sig != sig) return false;
  Runtime &R = rt();
  for (auto [d, v] : last.peer_ver)
    if (R.shm->slots[d].layout_ver.load(std::memory_order_acquire) != v) return false;
  return true;
}

// Layout versions of the distinct out-neighbours, read BEFORE their
// layouts are: the record of a built call must carry the versions the
// build saw. Read after the launch instead, a receiver released by this
// call's READY flags could already have published its next layout, and
// its new version would then vouch for a batch built from the old one.
std::vector<std::pair<int, uint64_t>> peer_versions(const std::vector<int> &dests) {
  Runtime &R = rt();
  std::vector<std::pair<int, uint64_t>> out;
  std::vector<char> seen(R.size, 0);
  for (int d : dests)
    if (!seen[d]) {
      seen[d] = 1;
      out.emplace_back(d, R.shm->slots[d].layout_ver.load(std::memory_order_acquire));
    }
  return out;
}

void nbr_last_set(NbrLast &last, std::string sig, std::vector<std::pair<int, uint64_t>> vers, Batch *b,
                  std::vector<LooseOp> loose, std::vector<std::shared_ptr<TableCopy>> tables = {}) {
  last.sig = std::move(sig);
  last.loose = std::move(loose);
  last.tables = std::move(tables);
  last.peer_ver = std::move(vers);
  last.batch = b;
  last.valid = true;
}

template <class T> void append_bytes(std::string &s, const std::vector<T> &v) {
  s.append(reinterpret_cast<const char *>(v.data()), v.size() * sizeof(T));
}

// batch-cache key part of a committed type: its geometry (and, for a
// block-list form, which has no geometry to compare, the record itself --
// the cached call holds it, so the address cannot be reused meanwhile)
void append_type_key(std::string &key, const Committed &c) {
  const int64_t head[6] = {c.form, c.size, c.extent, c.span, c.sb.start,
                           c.form == SP_FORM_STRIDED ? 0 : reinterpret_cast<int64_t>(&c)};
  key.append(reinterpret_cast<const char *>(head), sizeof(head));
  key.append(reinterpret_cast<const char *>(c.sb.counts.data()), c.sb.counts.size() * sizeof(int64_t));
  key.append(reinterpret_cast<const char *>(c.sb.strides.data()), c.sb.strides.size() * sizeof(int64_t));
}

// Entering a neighbour collective without a barrier (call after this rank's
// layout is published): for every distinct in-neighbour s, count the call
// and announce it (slot.pair_entered[s]); for every distinct out-neighbour
// d, count the call and wait until d has entered it -- d's receive buffer
// then belongs to the call and its layout is readable. The returned signal
// set makes the data kernel publish READY to each out-neighbour (value =
// calls on that pair, 2^32 per launch) and wait, in block 0, for READY from each
// in-neighbour, so the call is complete when the kernel is: no host
// barrier before or after. Edges to self need no flags (stream order).
BatchSignal nbr_enter(const std::vector<int> &sources, const std::vector<int> &dests) {
  Runtime &R = rt();
  BatchSignal bs;
  std::vector<char> seen_s(R.size, 0), seen_d(R.size, 0);
  { // everything that can refuse the call is checked BEFORE it is counted
    // and announced: once entered, the peers' kernels wait for this rank
    int ns = 0, nd = 0;
    for (int s : sources) {
      if (s < 0 || s >= R.size) fail(SP_ERR_INVALID_ARGUMENT, "neighbour exchange: source rank out of range");
      if (s != R.rank && !seen_s[s]) seen_s[s] = 1, ++ns;
    }
    for (int d : dests) {
      if (d < 0 || d >= R.size) fail(SP_ERR_INVALID_ARGUMENT, "neighbour exchange: destination rank out of range");
      if (d != R.rank && !seen_d[d]) seen_d[d] = 1, ++nd;
    }
    if (ns > kMaxSignalPeers || nd > kMaxSignalPeers)
      fail(SP_ERR_UNSUPPORTED, "neighbour exchange: more than 32 distinct neighbours");
    std::fill(seen_s.begin(), seen_s.end(), 0);
    std::fill(seen_d.begin(), seen_d.end(), 0);
  }
  for (int s : sources) {
    if (s == R.rank || seen_s[s]) continue;
    seen_s[s] = 1;
    const uint64_t n = ++R.pair_recv[s];
    bs.post.push_back(R.nbr_flags + s);
    bs.post_values.push_back(n << 32); // a sender launch adds 2^32
  }
  std::atomic_thread_fence(std::memory_order_release); // layout before the announcement
  for (int s = 0; s < R.size; ++s)
    if (seen_s[s]) R.shm->slots[R.rank].pair_entered[s].store(R.pair_recv[s], std::memory_order_release);
  std::vector<int> outs;
  for (int d : dests) {
    if (d == R.rank || seen_d[d]) continue;
    seen_d[d] = 1;
    ++R.pair_sent[d];
    bs.signal.push_back(reinterpret_cast<uint64_t *>(R.peer_nbr_flags[d]) + R.rank);
    outs.push_back(d);
  }
  for (int d : outs) {
    Waiter w("neighbour collective entry", d);
    while (R.shm->slots[d].pair_entered[R.rank].load(std::memory_order_acquire) < R.pair_sent[d]) {
      rt_progress();
      w.pause();
    }
  }
  bs.sys_scope = R.nbr_remote;
  bs.err = R.err_dev;
  bs.timeout_ns = rt_device_timeout_ns();
  return bs;
}

void nbr_run(Batch *b, const std::vector<LooseOp> &loose, const BatchSignal &bs) {
  Runtime &R = rt();
  if (!loose.empty()) { // every irregular edge in one run-table launch
    std::vector<RunJob> jobs;
    jobs.reserve(loose.size());
    for (const LooseOp &op : loose)
      jobs.push_back({op.ct.get(), op.src, op.count, op.dst, op.unpack, op.psrc, op.pdst, op.npieces, op.size,
                      op.extent, op.align});
    runs_multi(jobs, R.stream);
  }
  if (b) {
    batch_execute_signaled(*b, R.stream, bs);
  } else {
    flags_signal_wait(bs, R.stream);
  }
  cuda_check(cudaStreamSynchronize(R.stream), "cudaStreamSynchronize(neighbor)");
  rt_check_device_error("neighbour collective");
}

// A call that fails after nbr_enter still completes the entry protocol:
// its READY flags go out (no data) and it waits for its senders, so the
// peers' kernels finish and the per-pair call counts stay in step; then the
// error is returned. Without this a refused argument on one rank would hang
// every neighbour's GPU.
template <class F> void nbr_guarded(const BatchSignal &bs, F &&body) {
  try {
    body();
  } catch (...) {
    Runtime &R = rt();
    try {
      flags_signal_wait(bs, R.stream);
      cudaStreamSynchronize(R.stream);
    } catch (...) {
    }
    throw;
  }
}

void rt_neighbor_alltoallv(const uint8_t *sendbuf, const std::vector<int64_t> &send_counts,
                           const std::vector<int64_t> &send_displs, const CommitPtr &stp, uint8_t *recvbuf,
                           const std::vector<int64_t> &recv_counts, const std::vector<int64_t> &recv_displs,
                           const Committed &rtp, const std::vector<int> &sources, const std::vector<int> &dests) {
  Runtime &R = rt();
  ipc_call_begin();
  const Committed &st = *stp;
  if (static_cast<int>(sources.size()) > kMaxEdges) fail(SP_ERR_UNSUPPORTED, "neighbour exchange: indegree > 256");
  const bool dense_recv = rtp.form == SP_FORM_STRIDED && rtp.sb.ndims() == 1 && rtp.sb.start == 0 &&
                          rtp.extent == rtp.size;
  if (!dense_recv && rtp.form != SP_FORM_EMPTY)
    fail(SP_ERR_UNSUPPORTED, "neighbour exchange: receive type must be contiguous bytes (e.g. MPI_PACKED)");
  {
    std::vector<int64_t> disp(sources.size()), bytes(sources.size());
    for (size_t j = 0; j < sources.size(); ++j) {
      disp[j] = recv_displs[j] * rtp.extent;
      bytes[j] = recv_counts[j] * rtp.size;
    }
    nbr_publish(recvbuf, sources, disp, bytes, nullptr);
  }
  const BatchSignal bs = nbr_enter(sources, dests); // replaces a barrier
  nbr_guarded(bs, [&] {
    std::string sig(reinterpret_cast<const char *>(&sendbuf), sizeof(sendbuf));
    sig.append(reinterpret_cast<const char *>(&recvbuf), sizeof(recvbuf));
    append_bytes(sig, send_counts);
    append_bytes(sig, send_displs);
    append_bytes(sig, dests);
    append_type_key(sig, st);
    if (nbr_last_hit(g_last_v, sig)) {
      nbr_run(g_last_v.batch, g_last_v.loose, bs);
      return;
    }
    auto vers = peer_versions(dests); // before any layout is read
    std::string key(reinterpret_cast<const char *>(&sendbuf), sizeof(sendbuf));
    std::vector<BatchSpec> jobs;
    std::vector<LooseOp> loose;
    const bool blocklist = st.form != SP_FORM_STRIDED; // irregular send type: run-table packs
    std::vector<int> seen(R.size, 0);
    for (size_t i = 0; i < dests.size(); ++i) {
      const int d = dests[i];
      const int occ = seen[d]++;
      const Slot &peer = R.shm->slots[d];
      int hit = -1;
      for (int j = 0, k = 0; j < peer.nedges; ++j)
        if (peer.edges[j][0] == R.rank && k++ == occ) {
          hit = j;
          break;
        }
      if (hit < 0) fail(SP_ERR_INVALID_ARGUMENT, "neighbour exchange: destination does not list this rank as source");
      const int64_t bytes = send_counts[i] * st.size;
      if (bytes > peer.edges[hit][2]) fail(SP_ERR_BUFFER_TOO_SMALL, "neighbour exchange: message truncated");
      if (bytes == 0) continue;
      uint8_t *base = d == R.rank ? recvbuf : open_ipc(peer.xh, d, peer.xr) + peer.xoff;
      if (blocklist) {
        loose.push_back({stp, sendbuf + send_displs[i] * st.extent, send_counts[i], base + peer.edges[hit][1]});
        continue;
      }
      jobs.push_back({&st, sendbuf + send_displs[i] * st.extent, UINT64_MAX, send_counts[i], base, UINT64_MAX,
                      peer.edges[hit][1]});
      const int64_t sig[4] = {reinterpret_cast<int64_t>(base), peer.edges[hit][1], send_counts[i], send_displs[i]};
      key.append(reinterpret_cast<const char *>(sig), sizeof(sig));
    }
    append_type_key(key, st); // geometry, not the address: a freed type's address can be reused
    Batch *b = nullptr;
    for (auto &e : g_nbr_cache)
      if (e.key == key) b = e.batch;
    if (!b && !jobs.empty()) {
      b = batch_create(jobs, false);
      g_nbr_cache.push_back({key, b});
      if (g_nbr_cache.size() > 16) {
        if (g_last_v.batch == g_nbr_cache.front().batch) g_last_v.valid = false;
        batch_destroy(g_nbr_cache.front().batch);
        g_nbr_cache.pop_front();
      }
    }
    nbr_run(b, loose, bs); // returns when every block addressed to this rank has landed
    nbr_last_set(g_last_v, std::move(sig), std::move(vers), b, std::move(loose));
  });
}

// MPI_Neighbor_alltoallw with per-edge datatypes on BOTH sides: each rank
// publishes, per in-edge, its receive buffer (IPC), the byte displacement
// and the canonical geometry of the receive type; each rank then runs ONE
// typed-copy launch that moves every out-edge block from its send type
// straight to its final strided place in the receiver's buffer over NVLink
// (no packed intermediate, no unpack, no per-neighbour launch). The 26
// region types of a halo exchange become a single kernel per rank.
namespace {
struct NbrWCacheEntry {
  std::string key;
  Batch *batch;
};
std::deque<NbrWCacheEntry> g_nbrw_cache;

struct WArgs {
  const uint8_t *sbuf;
  const uint8_t *rbuf;
  std::vector<int64_t> sc, sd, rc, rd;
  std::vector<int> sources, dests;
  std::vector<const Committed *> st, rtp;
  cudaIpcMemHandle_t h;
  int64_t off;
  bool operator==(const WArgs &o) const {
    return sbuf == o.sbuf && rbuf == o.rbuf && sc == o.sc && sd == o.sd && rc == o.rc && rd == o.rd &&
           sources == o.sources && dests == o.dests && st == o.st && rtp == o.rtp && off == o.off &&
           std::memcmp(&h, &o.h, sizeof(h)) == 0;
  }
};

// the previous call's arguments; the commit records are held so their
// addresses cannot be reused by other types while they are compared
struct WLastCall {
  WArgs args{};
  std::vector<CommitPtr> keep_s, keep_r;
  uint64_t my_ver = 0; // this rank's layout version right after that call
  bool valid = false;
};
WLastCall g_wlast;

void desc_of(const Committed &c, int64_t count, Desc &d) {
  if (c.form != SP_FORM_STRIDED) { // block-list: publish the device run table
    const DeviceRuns &dr = device_run_table(c);
    d.runs = 1;
    d.ndims = 0;
    d.size = c.size;
    d.extent = c.extent;
    d.span = c.span;
    d.count = count;
    d.npieces = dr.n;
    d.align = dr.align_or;
    d.raw_s = reinterpret_cast<uint64_t>(dr.d_src);
    d.raw_d = reinterpret_cast<uint64_t>(dr.d_dst);
    ipc_handle_of(dr.d_src, &d.hs, &d.os, d.sr);
    ipc_handle_of(dr.d_dst, &d.hd, &d.od, d.dr);
    return;
  }
  d.ndims = c.sb.ndims();
  d.start = c.sb.start;
  for (int i = 0; i < d.ndims; ++i) {
    d.counts[i] = c.sb.counts[i];
    d.strides[i] = c.sb.strides[i];
  }
  d.size = c.size;
  d.extent = c.extent;
  d.span = c.span;
  d.count = count;
}
} // namespace

void rt_neighbor_alltoallw_build(const uint8_t *sendbuf, const std::vector<int64_t> &send_counts,
                                 const std::vector<int64_t> &send_displs, const std::vector<CommitPtr> &send_types,
                                 uint8_t *recvbuf, const std::vector<int> &dests, const BatchSignal &bs);

// drops every cached neighbour launch and repeat-call record: they name IPC
// mappings and peers of the runtime being finalised
void nbr_reset() {
  g_last_v = NbrLast{};
  g_last_w = NbrLast{};
  g_wlast = WLastCall{};
  for (auto &e : g_nbr_cache) batch_destroy(e.batch);
  g_nbr_cache.clear();
  for (auto &e : g_nbrw_cache) batch_destroy(e.batch);
  g_nbrw_cache.clear();
}

void rt_neighbor_alltoallw(const uint8_t *sendbuf, const std::vector<int64_t> &send_counts,
                           const std::vector<int64_t> &send_displs, const std::vector<CommitPtr> &send_types,
                           uint8_t *recvbuf, const std::vector<int64_t> &recv_counts,
                           const std::vector<int64_t> &recv_displs, const std::vector<CommitPtr> &recv_types,
                           const std::vector<int> &sources, const std::vector<int> &dests) {
  ipc_call_begin();
  const Runtime &R = rt();
  if (static_cast<int>(sources.size()) > kMaxWEdges) fail(SP_ERR_UNSUPPORTED, "neighbour alltoallw: indegree > 64");
  // repeat of the previous call (same buffers, counts, displacements,
  // neighbours and commit records, and the receive buffer still the same
  // allocation): this rank's published layout and the cached launch are
  // current, so only the entry protocol and the launch remain
  WArgs args{sendbuf, recvbuf, send_counts, send_displs, recv_counts, recv_displs, sources, dests, {}, {}, {}, 0};
  args.st.reserve(send_types.size());
  for (const CommitPtr &t : send_types) args.st.push_back(t.get());
  args.rtp.reserve(recv_types.size());
  for (const CommitPtr &t : recv_types) args.rtp.push_back(t.get());
  if (recvbuf && std::any_of(recv_counts.begin(), recv_counts.end(), [](int64_t c) { return c > 0; }))
    ipc_handle_of(recvbuf, &args.h, &args.off);
  // (another neighbour call publishing a different layout in between moves
  // this rank's layout version and disables the repeat path)
  if (g_wlast.valid && g_wlast.args == args && g_last_w.valid &&
      R.shm->slots[R.rank].layout_ver.load(std::memory_order_relaxed) == g_wlast.my_ver) {
    const BatchSignal bs = nbr_enter(sources, dests);
    nbr_guarded(bs, [&] {
      if (nbr_peers_unchanged(g_last_w)) {
        nbr_run(g_last_w.batch, g_last_w.loose, bs);
        return;
      }
      g_wlast.valid = false; // a neighbour re-published: rebuild below (entered already)
      rt_neighbor_alltoallw_build(sendbuf, send_counts, send_displs, send_types, recvbuf, dests, bs);
      g_wlast = WLastCall{std::move(args), send_types, recv_types,
                          R.shm->slots[R.rank].layout_ver.load(std::memory_order_relaxed), true};
    });
    return;
  }
  g_wlast.valid = false;
  {
    std::vector<Desc> descs(sources.size(), Desc{});
    std::vector<const Desc *> dp(sources.size(), nullptr);
    std::vector<int64_t> bytes(sources.size());
    for (size_t j = 0; j < sources.size(); ++j) {
      const Committed &rt_ = *recv_types[j];
      bytes[j] = recv_counts[j] * rt_.size;
      // irregular (block-list) receive layouts: the device run table is
      // published through CUDA IPC (its upload has landed: copy_sync)
      const bool runs = rt_.form == SP_FORM_UNSUPPORTED && !rt_.overlapping;
      if (bytes[j] > 0 && !describable(rt_) && !runs)
        fail(SP_ERR_UNSUPPORTED, "neighbour alltoallw: receive types need a non-overlapping layout");
      if (bytes[j] > 0) {
        desc_of(rt_, recv_counts[j], descs[j]);
        dp[j] = &descs[j];
      }
    }
    nbr_publish(recvbuf, sources, recv_displs, bytes, &dp);
  }
  const BatchSignal bs = nbr_enter(sources, dests); // replaces a barrier
  nbr_guarded(bs, [&] {
    rt_neighbor_alltoallw_build(sendbuf, send_counts, send_displs, send_types, recvbuf, dests, bs);
    g_wlast = WLastCall{std::move(args), send_types, recv_types,
                        R.shm->slots[R.rank].layout_ver.load(std::memory_order_relaxed), true};
  });
}

// ---- persistent neighbour alltoallw (MPI-4 MPI_Neighbor_alltoallw_init)
// The call's typed-copy batch is built once, against the receivers'
// layouts published at creation, and every start is one signalled launch
// with the halo plans' device protocol instead of the host entry protocol:
// block 0 tells this rank's senders that the receive buffer is free for
// iteration n (FREE = n-1), every block waits for FREE = n-1 from its
// receivers, stores its blocks, adds its share of READY = n, and block 0
// waits for READY = n from its senders -- so the launch completes when
// this rank's receives have landed. Starts are numbered on the host, or on
// the device once captured into a CUDA graph (like the halo plans).
namespace {
constexpr int kPlanReady = 0, kPlanFree = 1;
bool all_ranks_ok(bool ok) { // every rank learns whether every rank succeeded
  Runtime &R = rt();
  constexpr int kTag = 0x7e5a;
  int32_t v = ok ? 1 : 0;
  if (R.rank == 0) {
    for (int r = 1; r < R.size; ++r) {
      int32_t o = 0;
      rt_host_recv(r, kTag, &o, sizeof(o));
      v &= o;
    }
    for (int r = 1; r < R.size; ++r) rt_host_send(r, kTag + 1, &v, sizeof(v));
  } else {
    rt_host_send(0, kTag, &v, sizeof(v));
    rt_host_recv(0, kTag + 1, &v, sizeof(v));
  }
  return v != 0;
}
} // namespace

struct NbrPlan {
  Batch *batch = nullptr;
  std::vector<std::unique_ptr<Committed>> dst_types; // the receivers' geometries
  std::vector<CommitPtr> keep;
  std::vector<cudaIpcMemHandle_t> pinned;            // peers' receive buffers
  uint64_t *flags = nullptr;                         // [READY n][FREE n]
  std::vector<uint8_t *> peer_flags;
  std::vector<int> out_peers, in_peers;
  uint64_t iter = 0, *dev_iter = nullptr;
  bool graph_mode = false;
  cudaEvent_t done = nullptr;
  ~NbrPlan() {
    for (const auto &h : pinned) ipc_pin_handle(h, -1);
    rt_pin_ptrs(peer_flags, -1);
    batch_destroy(batch);
    if (flags) cudaFree(flags);
    if (dev_iter) cudaFree(dev_iter);
    if (done) cudaEventDestroy(done);
  }
};

NbrPlan *rt_nbr_plan_create(const uint8_t *sendbuf, const std::vector<int64_t> &send_counts,
                            const std::vector<int64_t> &send_displs, const std::vector<CommitPtr> &send_types,
                            uint8_t *recvbuf, const std::vector<int64_t> &recv_counts,
                            const std::vector<int64_t> &recv_displs, const std::vector<CommitPtr> &recv_types,
                            const std::vector<int> &sources, const std::vector<int> &dests) {
  Runtime &R = rt();
  ipc_call_begin();
  auto p = std::make_unique<NbrPlan>();
  // local checks first, agreed by every rank before anything is published
  std::string why;
  std::vector<Desc> descs(sources.size(), Desc{});
  std::vector<const Desc *> dp(sources.size(), nullptr);
  std::vector<int64_t> bytes(sources.size());
  for (size_t j = 0; j < sources.size() && why.empty(); ++j) {
    const Committed &rt_ = *recv_types[j];
    bytes[j] = recv_counts[j] * rt_.size;
    if (bytes[j] > 0 && !describable(rt_)) why = "receive types need a strided non-overlapping layout";
    if (bytes[j] > 0 && why.empty()) {
      desc_of(rt_, recv_counts[j], descs[j]);
      dp[j] = &descs[j];
    }
  }
  for (size_t i = 0; i < dests.size() && why.empty(); ++i)
    if (send_counts[i] > 0 && send_types[i]->form != SP_FORM_STRIDED) why = "send types need a strided form";
  if (sources.size() > static_cast<size_t>(kMaxWEdges) || dests.size() > static_cast<size_t>(kMaxWEdges))
    why = "more than 64 edges";
  { // the start launch carries the protocol: a rank with peers must send something
    bool peer = false, sends = false;
    for (int d : dests) peer |= d != R.rank;
    for (int q : sources) peer |= q != R.rank;
    for (size_t i = 0; i < dests.size(); ++i) sends |= send_counts[i] > 0 && send_types[i]->size > 0;
    if (peer && !sends && why.empty()) why = "a rank with neighbours but nothing to send";
  }
  if (!all_ranks_ok(why.empty()))
    fail(SP_ERR_UNSUPPORTED, "persistent neighbour alltoallw: " + (why.empty() ? std::string("another rank's types") : why));
  nbr_publish(recvbuf, sources, recv_displs, bytes, &dp);
  rt_barrier(); // every receive layout published
  std::vector<CopySpec> jobs;
  std::vector<int> seen(R.size, 0);
  for (size_t i = 0; i < dests.size() && why.empty(); ++i) {
    const int d = dests[i];
    const int occ = seen[d]++;
    const Slot &peer = R.shm->slots[d];
    int hit = -1;
    for (int j = 0, k = 0; j < peer.nedges; ++j)
      if (peer.edges[j][0] == R.rank && k++ == occ) {
        hit = j;
        break;
      }
    const Committed &st = *send_types[i];
    const int64_t b = send_counts[i] * st.size;
    if (hit < 0) {
      why = "a destination does not list this rank as a source";
    } else if (b != peer.edges[hit][2]) {
      why = "send and receive describe different byte counts";
    } else if (b > 0) {
      const Desc &wd = peer.wdesc[hit];
      uint8_t *base = d == R.rank ? recvbuf : open_ipc(peer.xh, d, peer.xr) + peer.xoff;
      if (d != R.rank) {
        ipc_pin_handle(peer.xh, 1);
        p->pinned.push_back(peer.xh);
      }
      auto dc = std::make_unique<Committed>();
      committed_from(wd, *dc);
      jobs.push_back({&st, sendbuf + send_displs[i], UINT64_MAX, send_counts[i], dc.get(),
                      base + peer.edges[hit][1], UINT64_MAX, wd.count});
      p->dst_types.push_back(std::move(dc));
    }
  }
  rt_barrier(); // every layout read before a later call republishes
  if (!all_ranks_ok(why.empty())) fail(SP_ERR_INVALID_ARGUMENT, "persistent neighbour alltoallw: " + why);
  p->keep = send_types;
  if (!jobs.empty()) p->batch = copy_batch_create(jobs);
  const int n = R.size;
  cuda_check(cudaMalloc(&p->flags, 2 * n * sizeof(uint64_t)), "cudaMalloc(plan flags)");
  cuda_check(cudaMemset(p->flags, 0, 2 * n * sizeof(uint64_t)), "cudaMemset(plan flags)");
  cuda_check(cudaMalloc(&p->dev_iter, sizeof(uint64_t)), "cudaMalloc(plan counter)");
  cuda_check(cudaMemset(p->dev_iter, 0, sizeof(uint64_t)), "cudaMemset(plan counter)");
  cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  rt_exchange_ptr(p->flags, p->peer_flags);
  rt_pin_ptrs(p->peer_flags, 1);
  std::vector<char> so(n, 0), si(n, 0);
  for (int d : dests)
    if (d != R.rank && !so[d]) so[d] = 1, p->out_peers.push_back(d);
  for (int s : sources)
    if (s != R.rank && !si[s]) si[s] = 1, p->in_peers.push_back(s);
  cuda_check(cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming), "cudaEventCreate");
  return p.release();
}

void rt_nbr_plan_start(NbrPlan *p) {
  Runtime &R = rt();
  cudaStream_t s = R.stream;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(s, &cap), "cudaStreamIsCapturing");
  const bool peers = !p->out_peers.empty() || !p->in_peers.empty();
  if (cap != cudaStreamCaptureStatusNone) p->graph_mode = true;
  if (!p->batch) return; // nothing to move and no peer
  const int n = R.size, me = R.rank;
  const uint64_t it = ++p->iter;
  auto at = [&](uint8_t *base, int kind, int peer) {
    return reinterpret_cast<uint64_t *>(base + static_cast<size_t>(kind * n + peer) * sizeof(uint64_t));
  };
  uint8_t *mine = reinterpret_cast<uint8_t *>(p->flags);
  BatchSignal ks;
  for (int q : p->in_peers) {
    ks.pre.push_back(at(p->peer_flags[q], kPlanFree, me));
    ks.post.push_back(at(mine, kPlanReady, q));
  }
  ks.pre_value = it - 1;
  for (int q : p->out_peers) {
    ks.wait.push_back(at(mine, kPlanFree, q));
    ks.signal.push_back(at(p->peer_flags[q], kPlanReady, me));
  }
  ks.wait_value = it - 1;
  ks.post_value = it << 32;
  ks.sys_scope = R.nbr_remote;
  ks.stream_waits = rt_flag_waits_in_stream();
  ks.err = rt_device_err();
  ks.timeout_ns = rt_device_timeout_ns();
  if (p->graph_mode && peers) {
    iter_tick(p->dev_iter, s);
    ks.iter = p->dev_iter;
    ks.pre_add = -1;
    ks.wait_add = -1;
    ks.post_shift = 32;
  } else {
    ks.iter_store = p->dev_iter;
    ks.iter_value = it;
  }
  batch_execute_signaled(*p->batch, s, ks);
  if (cap == cudaStreamCaptureStatusNone) cuda_check(cudaEventRecord(p->done, s), "cudaEventRecord");
}

bool rt_nbr_plan_test(NbrPlan *p) {
  const cudaError_t e = cudaEventQuery(p->done);
  if (e == cudaErrorNotReady) {
    cudaGetLastError();
    rt_progress();
    return false;
  }
  cuda_check(e, "cudaEventQuery");
  rt_check_device_error("persistent neighbour alltoallw");
  return true;
}

void rt_nbr_plan_wait(NbrPlan *p) {
  rt_sync_event(p->done, "persistent neighbour alltoallw");
  rt_check_device_error("persistent neighbour alltoallw");
}

void rt_nbr_plan_free(NbrPlan *p) {
  if (p && p->done) cudaEventSynchronize(p->done);
  delete p;
}

// the send side of an alltoallw call once entered: find (or build) the
// typed-copy batch for the out-edges against the neighbours' published
// receive layouts, and run it
void rt_neighbor_alltoallw_build(const uint8_t *sendbuf, const std::vector<int64_t> &send_counts,
                                 const std::vector<int64_t> &send_displs, const std::vector<CommitPtr> &send_types,
                                 uint8_t *recvbuf, const std::vector<int> &dests, const BatchSignal &bs) {
  Runtime &R = rt();
  std::string sig(reinterpret_cast<const char *>(&sendbuf), sizeof(sendbuf));
  sig.append(reinterpret_cast<const char *>(&recvbuf), sizeof(recvbuf));
  append_bytes(sig, send_counts);
  append_bytes(sig, send_displs);
  append_bytes(sig, dests);
  for (const CommitPtr &t : send_types) append_type_key(sig, *t);
  if (nbr_last_hit(g_last_w, sig)) {
    nbr_run(g_last_w.batch, g_last_w.loose, bs);
    return;
  }
  auto vers = peer_versions(dests); // before any layout is read
  std::string key(reinterpret_cast<const char *>(&sendbuf), sizeof(sendbuf));
  std::vector<CopySpec> jobs;
  std::vector<LooseOp> loose;
  std::vector<std::shared_ptr<TableCopy>> tables;
  std::vector<std::unique_ptr<Committed>> dst_types;
  std::vector<int> seen(R.size, 0);
  for (size_t i = 0; i < dests.size(); ++i) {
    const int d = dests[i];
    const int occ = seen[d]++;
    const Slot &peer = R.shm->slots[d];
    int hit = -1;
    for (int j = 0, k = 0; j < peer.nedges; ++j)
      if (peer.edges[j][0] == R.rank && k++ == occ) {
        hit = j;
        break;
      }
    if (hit < 0) fail(SP_ERR_INVALID_ARGUMENT, "neighbour exchange: destination does not list this rank as source");
    const Committed &st = *send_types[i];
    const int64_t bytes = send_counts[i] * st.size;
    if (bytes > peer.edges[hit][2]) fail(SP_ERR_BUFFER_TOO_SMALL, "neighbour exchange: message truncated");
    if (bytes != peer.edges[hit][2])
      fail(SP_ERR_INVALID_ARGUMENT, "neighbour alltoallw: send and receive describe different byte counts");
    if (bytes == 0) continue;
    const Desc &wd = peer.wdesc[hit];
    uint8_t *base = (d == R.rank ? recvbuf : open_ipc(peer.xh, d, peer.xr) + peer.xoff) + peer.edges[hit][1];
    if (wd.runs) {
      // an irregular receive layout: a dense send run scattered through the
      // receiver's run table (read over NVLink from the receiver's HBM)
      const bool dense = st.form == SP_FORM_STRIDED && st.sb.ndims() == 1 &&
                         (send_counts[i] <= 1 || st.extent == st.size);
      if (!dense)
        fail(SP_ERR_UNSUPPORTED,
             "neighbour alltoallw: an irregular (block-list) receive type needs a contiguous send layout");
      LooseOp op{};
      op.src = sendbuf + send_displs[i] + st.sb.start;
      op.count = wd.count;
      op.dst = base;
      op.unpack = true;
      if (d == R.rank) {
        op.psrc = reinterpret_cast<const int64_t *>(wd.raw_s);
        op.pdst = reinterpret_cast<const int64_t *>(wd.raw_d);
      } else { // the peer's table, copied into this GPU's HBM once per call layout
        const size_t ns = static_cast<size_t>(wd.npieces) * sizeof(int64_t), nd = ns + sizeof(int64_t);
        auto cs = std::make_shared<TableCopy>(ns), cd = std::make_shared<TableCopy>(nd);
        copy_sync(cs->p, open_ipc(wd.hs, d, wd.sr) + wd.os, ns, "run table copy");
        copy_sync(cd->p, open_ipc(wd.hd, d, wd.dr) + wd.od, nd, "run table copy");
        op.psrc = static_cast<const int64_t *>(cs->p);
        op.pdst = static_cast<const int64_t *>(cd->p);
        tables.push_back(std::move(cs));
        tables.push_back(std::move(cd));
      }
      op.npieces = wd.npieces;
      op.size = wd.size;
      op.extent = wd.extent;
      op.align = wd.align;
      loose.push_back(op);
      continue;
    }
    if (st.form != SP_FORM_STRIDED) {
      // an irregular send type: the run-table kernel packs it in place when
      // the receive layout is one dense run; typed copies between two
      // irregular layouts are not offered
      if (wd.ndims != 1 || (wd.count > 1 && wd.extent != wd.size))
        fail(SP_ERR_UNSUPPORTED,
             "neighbour alltoallw: an irregular (block-list) send type needs a contiguous receive layout");
      loose.push_back({send_types[i], sendbuf + send_displs[i], send_counts[i], base + wd.start});
      continue;
    }
    auto dc = std::make_unique<Committed>();
    committed_from(wd, *dc);
    jobs.push_back({&st, sendbuf + send_displs[i], UINT64_MAX, send_counts[i], dc.get(), base, UINT64_MAX, wd.count});
    const int64_t sig[5] = {reinterpret_cast<int64_t>(base), send_counts[i], send_displs[i], wd.count, wd.start};
    key.append(reinterpret_cast<const char *>(sig), sizeof(sig));
    append_type_key(key, st);
    // the receiver's whole geometry: types with one canonical row may still
    // differ in extent (contiguous(4, DOUBLE) vs a 1-D subarray of it)
    const int64_t geo[4] = {wd.size, wd.extent, wd.span, wd.ndims};
    key.append(reinterpret_cast<const char *>(geo), sizeof(geo));
    key.append(reinterpret_cast<const char *>(wd.counts), sizeof(int64_t) * wd.ndims);
    key.append(reinterpret_cast<const char *>(wd.strides), sizeof(int64_t) * wd.ndims);
    dst_types.push_back(std::move(dc));
  }
  Batch *b = nullptr;
  for (auto &e : g_nbrw_cache)
    if (e.key == key) b = e.batch;
  if (!b && !jobs.empty()) {
    b = copy_batch_create(jobs);
    g_nbrw_cache.push_back({key, b});
    if (g_nbrw_cache.size() > 16) {
      if (g_last_w.batch == g_nbrw_cache.front().batch) g_last_w.valid = false;
      batch_destroy(g_nbrw_cache.front().batch);
      g_nbrw_cache.pop_front();
    }
  }
  nbr_run(b, loose, bs); // returns when every block addressed to this rank has landed
  nbr_last_set(g_last_w, std::move(sig), std::move(vers), b, std::move(loose), std::move(tables));
}

} // namespace spb
