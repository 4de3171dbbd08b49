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

#include <atomic>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "guard.hpp"
#include "model.hpp"
#include "rt.hpp"

namespace spb {

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

struct Slot {
  std::atomic<uint32_t> ready;
  int32_t pid;
  int32_t device;
  int32_t pad;
  cudaIpcMemHandle_t window;  // device receive window (DEVICE method)
  int64_t window_bytes;
  int64_t host_bytes;         // shared pinned host region (ONESHOT/STAGED)
  cudaIpcMemHandle_t xh;      // publication area of sp_rt_exchange_ptr
  int64_t xoff;
  int64_t xbytes;
  int32_t nedges;             // neighbour-exchange in-edges: (src, offset, bytes)
  int32_t pad2;
  int64_t edges[kMaxEdges][3];
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
  std::map<std::string, uint8_t *> ipc_cache; // handle bytes -> mapped base
  std::deque<Msg> unexpected;
  cudaStream_t stream = nullptr;
  std::unique_ptr<sp_model_cache_s, sp_status (*)(sp_model_cache_s *)> cache{nullptr, sp_model_cache_free};
  sp_profile_s *profile = nullptr;
  std::mutex mu; // the runtime serialises its own calls (MPI_THREAD_SERIALIZED)
};

Runtime *g_rt = nullptr;

Runtime &rt() {
  if (!g_rt) fail(SP_ERR_INVALID_ARGUMENT, "runtime not initialised (sp_rt_init)");
  return *g_rt;
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

void post(int dst, const Msg &m) {
  Runtime &R = rt();
  Mailbox &b = R.shm->box[dst][R.rank];
  const uint64_t t = b.tail.load(std::memory_order_relaxed);
  unsigned spins = 0;
  while (t - b.head.load(std::memory_order_acquire) >= kRing) pause_briefly(spins);
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
  unsigned spins = 0;
  for (;;) {
    drain();
    for (auto it = R.unexpected.begin(); it != R.unexpected.end(); ++it) {
      if (it->kind == kind && (src < 0 || it->src == src) && (tag < 0 || it->tag == tag)) {
        Msg m = *it;
        R.unexpected.erase(it);
        return m;
      }
    }
    pause_briefly(spins);
  }
}

uint8_t *open_ipc(const cudaIpcMemHandle_t &h) {
  Runtime &R = rt();
  const std::string key(reinterpret_cast<const char *>(&h), sizeof(h));
  auto it = R.ipc_cache.find(key);
  if (it != R.ipc_cache.end()) return it->second;
  void *p = nullptr;
  cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  R.ipc_cache[key] = static_cast<uint8_t *>(p);
  return static_cast<uint8_t *>(p);
}

uint8_t *peer_window(int r) {
  Runtime &R = rt();
  if (r == R.rank) return R.window;
  if (!R.peer_window[r]) R.peer_window[r] = open_ipc(R.shm->slots[r].window);
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

void ipc_handle_of(const void *ptr, cudaIpcMemHandle_t *h, int64_t *offset) {
  // handles name whole allocations; carry the offset inside it separately
  cudaPointerAttributes at{};
  cuda_check(cudaPointerGetAttributes(&at, ptr), "cudaPointerGetAttributes");
  if (at.type != cudaMemoryTypeDevice) fail(SP_ERR_INVALID_ARGUMENT, "IPC export needs device memory");
  void *base = nullptr;
  size_t range = 0;
  // the runtime API has no range query; find the base by probing the handle
  // of the pointer itself first (cudaMalloc'd bases), else via the driver
  using GetRange = int (*)(uint64_t *, size_t *, uint64_t);
  static GetRange get_range = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
    return reinterpret_cast<GetRange>(fn);
  }();
  uint64_t b = 0;
  if (!get_range || get_range(&b, &range, reinterpret_cast<uint64_t>(ptr)) != 0)
    fail(SP_ERR_CUDA, "cuMemGetAddressRange failed");
  base = reinterpret_cast<void *>(b);
  cuda_check(cudaIpcGetMemHandle(h, base), "cudaIpcGetMemHandle");
  *offset = static_cast<const uint8_t *>(ptr) - static_cast<const uint8_t *>(base);
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
    unsigned spins = 0;
    while (reinterpret_cast<std::atomic<uint64_t> *>(&G.shm->magic)->load(std::memory_order_acquire) != kMagic)
      pause_briefly(spins);
  }
  Slot &me = G.shm->slots[rank];
  me.pid = static_cast<int32_t>(getpid());
  me.device = device;
  if (device >= 0) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&G.stream, cudaStreamNonBlocking), "cudaStreamCreate");
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
  me.ready.store(1, std::memory_order_release);
  rt_barrier();
}

void rt_finalize() {
  if (!g_rt) return;
  rt_barrier();
  Runtime &R = *g_rt;
  for (auto &kv : R.ipc_cache) cudaIpcCloseMemHandle(kv.second);
  for (int r = 0; r < R.size; ++r)
    if (R.peer_host[r] && r != R.rank) {
      cudaHostUnregister(R.peer_host[r]);
      munmap(R.peer_host[r], static_cast<size_t>(R.shm->slots[r].host_bytes));
    }
  rt_barrier();
  if (R.window) cudaFree(R.window);
  if (R.host) {
    cudaHostUnregister(R.host);
    munmap(R.host, static_cast<size_t>(R.host_bytes));
    shm_unlink(host_name(R.name, R.rank).c_str());
  }
  if (R.stream) cudaStreamDestroy(R.stream);
  const bool last = R.rank == 0;
  const std::string nm = R.name;
  munmap(R.shm, R.shm_bytes);
  if (last) shm_unlink(nm.c_str());
  delete g_rt;
  g_rt = nullptr;
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
    unsigned spins = 0;
    while (R.shm->generation.load(std::memory_order_acquire) == gen) pause_briefly(spins);
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
  Slot &me = R.shm->slots[R.rank];
  if (local) {
    ipc_handle_of(local, &me.xh, &me.xoff);
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
      out[r] = open_ipc(R.shm->slots[r].xh) + R.shm->slots[r].xoff;
    }
  }
  rt_barrier();
}

// ------------------------------------------------------------ point to point
// Rendezvous: the sender announces (RTS), the receiver grants its window
// (CTS) once a matching receive is posted, the sender packs straight into
// the granted memory and signals completion (FIN), the receiver unpacks.
//   DEVICE : pack kernel -> receiver's device window through CUDA IPC
//            (NVLink); receiver unpacks from its own HBM
//   ONESHOT: pack kernel -> receiver's shared pinned host region (mapped);
//            receiver's unpack kernel reads host memory directly
//   STAGED : pack kernel -> local device scratch -> D2H copy into the
//            receiver's host region; receiver copies H2D, then unpacks
void rt_send(const void *buf, uint64_t buf_bytes, int64_t count, const Committed &ct, int dest, int tag,
             int method, RtTrace *trace) {
  Runtime &R = rt();
  if (dest < 0 || dest >= R.size) fail(SP_ERR_INVALID_ARGUMENT, "send: bad destination rank");
  if (tag < 0) fail(SP_ERR_INVALID_ARGUMENT, "send: negative tag");
  const int64_t bytes = count * ct.size;
  if (method < 0) method = rt_choose(ct, count);
  if (method == SP_METHOD_DEVICE && bytes > R.shm->slots[dest].window_bytes)
    fail(SP_ERR_UNSUPPORTED, "send: message larger than the receive window");
  if (method != SP_METHOD_DEVICE && bytes > R.shm->slots[dest].host_bytes)
    fail(SP_ERR_UNSUPPORTED, "send: message larger than the receiver's host region");
  post(dest, Msg{kRTS, R.rank, tag, method, bytes, 0, 0});
  wait_msg(kCTS, dest, tag);
  if (bytes > 0) {
    int64_t pos = 0;
    PackArgs a{};
    a.ct = &ct;
    a.src = buf;
    a.src_bytes = buf_bytes;
    a.count = count;
    a.stream = R.stream;
    a.opt = sp_pack_options{1, SP_KERNEL_AUTO, 0};
    a.pack = true;
    if (method == SP_METHOD_DEVICE) {
      a.dst = peer_window(dest);
      a.dst_bytes = static_cast<uint64_t>(bytes);
      execute(a);
    } else if (method == SP_METHOD_ONESHOT) {
      a.dst = peer_host(dest);
      a.dst_bytes = static_cast<uint64_t>(bytes);
      execute(a);
    } else {
      uint8_t *scratch = nullptr;
      cuda_check(cudaMallocAsync(reinterpret_cast<void **>(&scratch), static_cast<size_t>(bytes), R.stream),
                 "cudaMallocAsync");
      a.dst = scratch;
      a.dst_bytes = static_cast<uint64_t>(bytes);
      execute(a);
      cuda_check(cudaMemcpyAsync(peer_host(dest), scratch, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost,
                                 R.stream),
                 "staged D2H");
      cuda_check(cudaFreeAsync(scratch, R.stream), "cudaFreeAsync");
    }
    (void)pos;
    cuda_check(cudaStreamSynchronize(R.stream), "cudaStreamSynchronize(send)");
  }
  post(dest, Msg{kFIN, R.rank, tag, method, bytes, 0, 0});
  if (trace) {
    trace->method = method;
    trace->bytes = bytes;
  }
}

void rt_recv(void *buf, uint64_t buf_bytes, int64_t count, const Committed &ct, int source, int tag, RtStatus *st) {
  Runtime &R = rt();
  const Msg rts = wait_msg(kRTS, source, tag);
  const int64_t bytes = count * ct.size;
  if (rts.bytes > bytes) fail(SP_ERR_BUFFER_TOO_SMALL, "recv: message truncated (MPI_ERR_TRUNCATE)");
  post(rts.src, Msg{kCTS, R.rank, rts.tag, rts.method, rts.bytes, 0, 0});
  wait_msg(kFIN, rts.src, rts.tag);
  if (rts.bytes > 0) {
    if (ct.size == 0 || rts.bytes % ct.size) fail(SP_ERR_INVALID_ARGUMENT, "recv: message is not whole objects");
    const int64_t n = rts.bytes / ct.size;
    int64_t pos = 0;
    PackArgs a{};
    a.ct = &ct;
    a.dst = buf;
    a.dst_bytes = buf_bytes;
    a.count = n;
    a.position = pos;
    a.stream = R.stream;
    a.opt = sp_pack_options{1, SP_KERNEL_AUTO, 0};
    a.pack = false;
    uint8_t *scratch = nullptr;
    if (rts.method == SP_METHOD_DEVICE) {
      a.src = R.window;
    } else if (rts.method == SP_METHOD_ONESHOT) {
      a.src = R.host;
    } else {
      cuda_check(cudaMallocAsync(reinterpret_cast<void **>(&scratch), static_cast<size_t>(rts.bytes), R.stream),
                 "cudaMallocAsync");
      cuda_check(cudaMemcpyAsync(scratch, R.host, static_cast<size_t>(rts.bytes), cudaMemcpyHostToDevice, R.stream),
                 "staged H2D");
      a.src = scratch;
    }
    a.src_bytes = static_cast<uint64_t>(rts.bytes);
    execute(a);
    if (scratch) cuda_check(cudaFreeAsync(scratch, R.stream), "cudaFreeAsync");
    cuda_check(cudaStreamSynchronize(R.stream), "cudaStreamSynchronize(recv)");
  }
  if (st) {
    st->source = rts.src;
    st->tag = rts.tag;
    st->bytes = rts.bytes;
    st->method = rts.method;
  }
}

void rt_set_profile(sp_profile_s *p) {
  Runtime &R = rt();
  R.profile = p;
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
  const int64_t blk = ct.form == SP_FORM_STRIDED ? std::min(ct.sb.counts[0], obj) : 1;
  int m = SP_METHOD_DEVICE;
  if (sp_model_cache_choose(R.cache.get(), obj, blk, &m) != SP_OK) return SP_METHOD_DEVICE;
  return m;
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

void rt_neighbor_alltoallv(const uint8_t *sendbuf, const std::vector<int64_t> &send_counts,
                           const std::vector<int64_t> &send_displs, const Committed &st, uint8_t *recvbuf,
                           const std::vector<int64_t> &recv_counts, const std::vector<int64_t> &recv_displs,
                           const Committed &rtp, const std::vector<int> &sources, const std::vector<int> &dests) {
  Runtime &R = rt();
  if (static_cast<int>(sources.size()) > kMaxEdges) fail(SP_ERR_UNSUPPORTED, "neighbour exchange: indegree > 256");
  const bool dense_recv = rtp.form == SP_FORM_STRIDED && rtp.sb.ndims() == 1 && rtp.sb.start == 0 &&
                          rtp.extent == rtp.size;
  if (!dense_recv && rtp.form != SP_FORM_EMPTY)
    fail(SP_ERR_UNSUPPORTED, "neighbour exchange: receive type must be contiguous bytes (e.g. MPI_PACKED)");
  Slot &me = R.shm->slots[R.rank];
  if (recvbuf) {
    ipc_handle_of(recvbuf, &me.xh, &me.xoff);
    me.xbytes = 1;
  } else {
    me.xbytes = 0;
  }
  me.nedges = static_cast<int32_t>(sources.size());
  for (size_t j = 0; j < sources.size(); ++j) {
    me.edges[j][0] = sources[j];
    me.edges[j][1] = recv_displs[j] * rtp.extent;
    me.edges[j][2] = recv_counts[j] * rtp.size;
  }
  rt_barrier(); // layouts published, every receive buffer is owned by the call
  std::string key(reinterpret_cast<const char *>(&sendbuf), sizeof(sendbuf));
  std::vector<BatchSpec> jobs;
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
    uint8_t *base = d == R.rank ? recvbuf : open_ipc(peer.xh) + peer.xoff;
    jobs.push_back({&st, sendbuf + send_displs[i] * st.extent, UINT64_MAX, send_counts[i], base, UINT64_MAX,
                    peer.edges[hit][1]});
    const int64_t sig[4] = {reinterpret_cast<int64_t>(base), peer.edges[hit][1], send_counts[i], send_displs[i]};
    key.append(reinterpret_cast<const char *>(sig), sizeof(sig));
  }
  key.append(reinterpret_cast<const char *>(&st), sizeof(void *));
  Batch *b = nullptr;
  for (auto &e : g_nbr_cache)
    if (e.key == key) b = e.batch;
  if (!b && !jobs.empty()) {
    b = batch_create(jobs, false);
    g_nbr_cache.push_back({key, b});
    if (g_nbr_cache.size() > 16) {
      batch_destroy(g_nbr_cache.front().batch);
      g_nbr_cache.pop_front();
    }
  }
  if (b) {
    batch_execute(*b, R.stream);
    cuda_check(cudaStreamSynchronize(R.stream), "cudaStreamSynchronize(neighbor)");
  }
  rt_barrier(); // every block addressed to this rank has landed
}

} // namespace spb
