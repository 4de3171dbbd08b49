// capi_rt.cpp -- C-ABI of the node-local runtime, point-to-point messages
// and the multi-process halo exchange.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "guard.hpp"
#include "halo.hpp"
#include "rt.hpp"
#include "trace.hpp"

using namespace spb;

namespace {
CommitPtr committed_of(sp_type t) { return registry().committed(t); }

// The handle -> commit-record lookups of the previous neighbour call, kept
// while the registry is unchanged: an iterative exchange passes the same
// 2 x degree handles every call, and resolving them is most of the call's
// host cost at degree 26 (~45 ns each under the registry's lock).
struct TypeMemo {
  std::vector<sp_type> handles;
  std::vector<CommitPtr> types;
  uint64_t gen = ~uint64_t{0};
  const std::vector<CommitPtr> &resolve(const sp_type *h, int64_t n) {
    const uint64_t g = registry().generation();
    if (g != gen || static_cast<int64_t>(handles.size()) != n || !std::equal(h, h + n, handles.begin())) {
      std::vector<CommitPtr> t;
      t.reserve(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) t.push_back(committed_of(h[i]));
      types = std::move(t);
      handles.assign(h, h + n);
      gen = g;
    }
    return types;
  }
};
TypeMemo g_memo_ws, g_memo_wr; // neighbour calls run on the rank's one MPI thread, like the engine
} // namespace

// One rank's share of a distributed halo exchange: its padded allocation,
// a receive buffer every neighbour writes into through CUDA IPC, and two
// persistent batch launches (26 packs, 26 unpacks).
struct sp_halo_plan_s {
  HaloCfg cfg{};
  int method = SP_HALO_FUSED;
  int rank = 0;
  uint8_t *alloc = nullptr;
  uint8_t *recv = nullptr, *send = nullptr;
  int64_t seg_total = 0;
  std::vector<int64_t> seg_off;
  std::vector<CommitPtr> keep;
  Batch *pack = nullptr, *unpack = nullptr;
  std::vector<uint8_t *> peer_send; // COPY method: where to pull segments from
  std::vector<int64_t> copy_src_rank;
  cudaEvent_t ev[4] = {};
  // SP_HALO_FUSED_ASYNC: per-peer completion flags in device memory,
  // flags[READY + src] (data of iteration n has landed) and flags[FREE + dst]
  // (the receiver consumed iteration n); peers' arrays are IPC-mapped
  uint64_t *flags = nullptr;
  std::vector<uint8_t *> peer_flags;
  std::vector<int> out_peers, in_peers; // distinct neighbours
  uint64_t iter = 0;
  // device iteration number: recorded by every host-numbered launch,
  // advanced on the device (iter_tick) once the plan was captured into a CUDA
  // graph -- from then on every exchange is numbered on the device
  uint64_t *dev_iter = nullptr;
  bool graph_mode = false;
  bool remote_peers = true; // some neighbour's memory is on another GPU
  std::vector<uint8_t *> pinned; // peer mappings held for the plan's lifetime
  ~sp_halo_plan_s() {
    rt_pin_ptrs(pinned, -1);
    batch_destroy(pack);
    batch_destroy(unpack);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (recv) cudaFree(recv);
    if (send) cudaFree(send);
    if (flags) cudaFree(flags);
    if (dev_iter) cudaFree(dev_iter);
  }
};

namespace {

constexpr int kReady = 0, kFree = 1; // flags[kind * size + peer]

} // namespace

extern "C" {

sp_status sp_rt_init(int rank, int size, const char *job, int device, int64_t window_bytes, int64_t host_bytes) {
  return guarded([&] { rt_init(rank, size, job, device, window_bytes, host_bytes); });
}

sp_status sp_rt_finalize(void) {
  return guarded([&] { rt_finalize(); });
}

sp_status sp_rt_rank(int *rank) {
  return guarded([&] {
    need(rank);
    *rank = rt_rank();
  });
}

sp_status sp_rt_size(int *size) {
  return guarded([&] {
    need(size);
    *size = rt_size();
  });
}

sp_status sp_rt_barrier(void) {
  return guarded([&] { rt_barrier(); });
}

sp_status sp_rt_host_send(int dst, int tag, const void *data, int64_t bytes) {
  return guarded([&] { rt_host_send(dst, tag, data, bytes); });
}

sp_status sp_rt_host_recv(int src, int tag, void *data, int64_t cap, int64_t *bytes) {
  return guarded([&] {
    const int64_t n = rt_host_recv(src, tag, data, cap);
    if (bytes) *bytes = n;
  });
}

sp_status sp_rt_set_profile(sp_profile p) {
  return guarded([&] { rt_set_profile(p); });
}

sp_status sp_rt_stream(void **stream) {
  return guarded([&] {
    need(stream);
    *stream = rt_stream();
  });
}

sp_status sp_rt_exchange_ptr(void *local, void **peers) {
  return guarded([&] {
    need(peers);
    std::vector<uint8_t *> out;
    rt_exchange_ptr(local, out);
    for (size_t r = 0; r < out.size(); ++r) peers[r] = out[r];
  });
}

sp_status sp_rt_choose(sp_type t, int64_t count, int *method) {
  return guarded([&] {
    need(method);
    *method = rt_choose(*committed_of(t), count);
  });
}

sp_status sp_rt_send(const void *buf, uint64_t buf_bytes, int64_t count, sp_type t, int dest, int tag, int method,
                     int *used_method) {
  SPB_TRACE("sp_rt_send");
  return guarded([&] {
    if (count < 0) fail(SP_ERR_INVALID_ARGUMENT, "send: negative count");
    RtTrace tr{};
    rt_send(buf, buf_bytes, count, committed_of(t), dest, tag, method, &tr);
    if (used_method) *used_method = tr.method;
  });
}

sp_status sp_rt_recv(void *buf, uint64_t buf_bytes, int64_t count, sp_type t, int source, int tag,
                     int64_t status[4]) {
  SPB_TRACE("sp_rt_recv");
  return guarded([&] {
    if (count < 0) fail(SP_ERR_INVALID_ARGUMENT, "recv: negative count");
    RtStatus st{};
    rt_recv(buf, buf_bytes, count, committed_of(t), source, tag, &st);
    if (status) {
      status[0] = st.source;
      status[1] = st.tag;
      status[2] = st.bytes;
      status[3] = st.method;
    }
  });
}

namespace {
void fill_status(const RtStatus &st, int64_t status[4]) {
  if (!status) return;
  status[0] = st.source;
  status[1] = st.tag;
  status[2] = st.bytes;
  status[3] = st.method;
}
} // namespace

sp_status sp_rt_isend(const void *buf, uint64_t buf_bytes, int64_t count, sp_type t, int dest, int tag, int method,
                      sp_request *req) {
  SPB_TRACE("sp_rt_isend");
  return guarded([&] {
    need(req);
    if (count < 0) fail(SP_ERR_INVALID_ARGUMENT, "send: negative count");
    *req = rt_isend(buf, buf_bytes, count, committed_of(t), dest, tag, method);
  });
}

sp_status sp_rt_irecv(void *buf, uint64_t buf_bytes, int64_t count, sp_type t, int source, int tag,
                      sp_request *req) {
  SPB_TRACE("sp_rt_irecv");
  return guarded([&] {
    need(req);
    if (count < 0) fail(SP_ERR_INVALID_ARGUMENT, "recv: negative count");
    *req = rt_irecv(buf, buf_bytes, count, committed_of(t), source, tag);
  });
}

sp_status sp_rt_test(sp_request req, int *done, int64_t status[4]) {
  return guarded([&] {
    need(done);
    RtStatus st{};
    *done = 0;
    if (rt_test(req, &st)) {
      *done = 1;
      fill_status(st, status);
    }
  });
}

sp_status sp_rt_wait(sp_request req, int64_t status[4]) {
  SPB_TRACE("sp_rt_wait");
  return guarded([&] {
    RtStatus st{};
    rt_wait(req, &st);
    fill_status(st, status);
  });
}

sp_status sp_rt_set_chunk(int64_t bytes) {
  return guarded([&] { rt_set_chunk(bytes); });
}

sp_status sp_rt_neighbor_alltoallv(const void *sendbuf, const int64_t *sendcounts, const int64_t *sdispls,
                                   int64_t outdegree, const int *dests, sp_type sendtype, void *recvbuf,
                                   const int64_t *recvcounts, const int64_t *rdispls, int64_t indegree,
                                   const int *sources, sp_type recvtype) {
  SPB_TRACE("sp_rt_neighbor_alltoallv");
  return guarded([&] {
    if (outdegree < 0 || indegree < 0) fail(SP_ERR_INVALID_ARGUMENT, "negative degree");
    if ((outdegree && (!sendcounts || !sdispls || !dests)) || (indegree && (!recvcounts || !rdispls || !sources)))
      fail(SP_ERR_INVALID_ARGUMENT, "null neighbour arrays");
    std::vector<int64_t> sc(sendcounts, sendcounts + outdegree), sd(sdispls, sdispls + outdegree);
    std::vector<int64_t> rc(recvcounts, recvcounts + indegree), rd(rdispls, rdispls + indegree);
    std::vector<int> ds(dests, dests + outdegree), ss(sources, sources + indegree);
    const CommitPtr st = committed_of(sendtype), rtp = committed_of(recvtype);
    const bool dense_recv = rtp->form == SP_FORM_EMPTY ||
                            (rtp->form == SP_FORM_STRIDED && rtp->sb.ndims() == 1 && rtp->sb.start == 0 &&
                             rtp->extent == rtp->size);
    if (dense_recv) { // packed receive buffer: pack-to-peer batch
      rt_neighbor_alltoallv(static_cast<const uint8_t *>(sendbuf), sc, sd, st, static_cast<uint8_t *>(recvbuf), rc,
                            rd, *rtp, ss, ds);
      return;
    }
    // a strided receive type: the alltoallw path with that type on every
    // edge (displacements in extents become bytes) -- typed copies straight
    // into the receivers' strided buffers
    for (auto &d : sd) d *= st->extent;
    for (auto &d : rd) d *= rtp->extent;
    rt_neighbor_alltoallw(static_cast<const uint8_t *>(sendbuf), sc, sd, std::vector<CommitPtr>(sc.size(), st),
                          static_cast<uint8_t *>(recvbuf), rc, rd, std::vector<CommitPtr>(rc.size(), rtp), ss, ds);
  });
}

sp_status sp_rt_neighbor_alltoallw(const void *sendbuf, const int64_t *sendcounts, const int64_t *sdispls,
                                   const sp_type *sendtypes, int64_t outdegree, const int *dests, void *recvbuf,
                                   const int64_t *recvcounts, const int64_t *rdispls, const sp_type *recvtypes,
                                   int64_t indegree, const int *sources) {
  SPB_TRACE("sp_rt_neighbor_alltoallw");
  return guarded([&] {
    if (outdegree < 0 || indegree < 0) fail(SP_ERR_INVALID_ARGUMENT, "negative degree");
    if ((outdegree && (!sendcounts || !sdispls || !sendtypes || !dests)) ||
        (indegree && (!recvcounts || !rdispls || !recvtypes || !sources)))
      fail(SP_ERR_INVALID_ARGUMENT, "null neighbour arrays");
    std::vector<int64_t> sc(sendcounts, sendcounts + outdegree), sd(sdispls, sdispls + outdegree);
    std::vector<int64_t> rc(recvcounts, recvcounts + indegree), rd(rdispls, rdispls + indegree);
    std::vector<int> ds(dests, dests + outdegree), ss(sources, sources + indegree);
    const std::vector<CommitPtr> &st = g_memo_ws.resolve(sendtypes, outdegree);
    const std::vector<CommitPtr> &rtp = g_memo_wr.resolve(recvtypes, indegree);
    rt_neighbor_alltoallw(static_cast<const uint8_t *>(sendbuf), sc, sd, st, static_cast<uint8_t *>(recvbuf), rc, rd,
                          rtp, ss, ds);
  });
}

struct sp_nbr_plan_s {
  NbrPlan *p = nullptr;
  ~sp_nbr_plan_s() { rt_nbr_plan_free(p); }
};

sp_status sp_rt_neighbor_alltoallw_init(const void *sendbuf, const int64_t *sendcounts, const int64_t *sdispls,
                                        const sp_type *sendtypes, int64_t outdegree, const int *dests,
                                        void *recvbuf, const int64_t *recvcounts, const int64_t *rdispls,
                                        const sp_type *recvtypes, int64_t indegree, const int *sources,
                                        sp_nbr_plan *out) {
  SPB_TRACE("sp_rt_neighbor_alltoallw_init");
  return guarded([&] {
    need(out);
    if (outdegree < 0 || indegree < 0) fail(SP_ERR_INVALID_ARGUMENT, "negative degree");
    if ((outdegree && (!sendcounts || !sdispls || !sendtypes || !dests)) ||
        (indegree && (!recvcounts || !rdispls || !recvtypes || !sources)))
      fail(SP_ERR_INVALID_ARGUMENT, "null edge arrays");
    std::vector<int64_t> sc(sendcounts, sendcounts + outdegree), sd(sdispls, sdispls + outdegree);
    std::vector<int64_t> rc(recvcounts, recvcounts + indegree), rd(rdispls, rdispls + indegree);
    std::vector<CommitPtr> st, rtp;
    for (int64_t i = 0; i < outdegree; ++i) st.push_back(committed_of(sendtypes[i]));
    for (int64_t j = 0; j < indegree; ++j) rtp.push_back(committed_of(recvtypes[j]));
    std::vector<int> ds(dests, dests + outdegree), ss(sources, sources + indegree);
    auto h = std::make_unique<sp_nbr_plan_s>();
    h->p = rt_nbr_plan_create(static_cast<const uint8_t *>(sendbuf), sc, sd, st, static_cast<uint8_t *>(recvbuf), rc,
                              rd, rtp, ss, ds);
    *out = h.release();
  });
}

sp_status sp_nbr_plan_start(sp_nbr_plan p) {
  return guarded([&] {
    need(p);
    rt_nbr_plan_start(p->p);
  });
}

sp_status sp_nbr_plan_test(sp_nbr_plan p, int *done) {
  return guarded([&] {
    need(p);
    need(done);
    *done = rt_nbr_plan_test(p->p) ? 1 : 0;
  });
}

sp_status sp_nbr_plan_wait(sp_nbr_plan p) {
  return guarded([&] {
    need(p);
    rt_nbr_plan_wait(p->p);
  });
}

sp_status sp_nbr_plan_free(sp_nbr_plan p) {
  delete p;
  return SP_OK;
}

sp_status sp_halo_plan_create(const sp_halo_config *cfgp, void *alloc, int method, sp_halo_plan *out) {
  return guarded([&] {
    need(cfgp);
    need(alloc);
    need(out);
    if (method != SP_HALO_FUSED && method != SP_HALO_COPY && method != SP_HALO_FUSED_ASYNC &&
        method != SP_HALO_DIRECT)
      fail(SP_ERR_INVALID_ARGUMENT, "unknown halo method");
    HaloCfg c{};
    for (int a = 0; a < 3; ++a) {
      c.ranks[a] = cfgp->ranks[a];
      c.interior[a] = cfgp->interior[a];
    }
    c.radius = cfgp->radius;
    c.elem = cfgp->element_bytes;
    halo_validate(c);
    if (c.ranks[0] * c.ranks[1] * c.ranks[2] != rt_size())
      fail(SP_ERR_INVALID_ARGUMENT, "halo rank grid does not match the runtime size");
    require_device();
    auto p = std::make_unique<sp_halo_plan_s>();
    p->cfg = c;
    p->method = method;
    p->rank = rt_rank();
    p->alloc = static_cast<uint8_t *>(alloc);
    const auto regions = halo_regions(c);
    const int64_t pad = (c.interior[0] + 2 * c.radius) * (c.interior[1] + 2 * c.radius) *
                        (c.interior[2] + 2 * c.radius) * c.elem;
    std::vector<CommitPtr> sct, rct;
    p->seg_off.assign(27, 0);
    for (int k = 0; k < 26; ++k) {
      sct.push_back(commit_def(*regions[k].send));
      rct.push_back(commit_def(*regions[k].recv));
      p->seg_off[k + 1] = p->seg_off[k] + sct[k]->size;
    }
    p->keep = sct;
    p->keep.insert(p->keep.end(), rct.begin(), rct.end());
    p->seg_total = p->seg_off[26];
    std::vector<BatchSpec> packs, unpacks;
    if (method == SP_HALO_DIRECT) {
      // ghost writes: region j of this rank lands in region 25-j of the
      // padded allocation of the rank at +d_j, through its IPC mapping
      std::vector<uint8_t *> peer_alloc;
      rt_exchange_ptr(alloc, peer_alloc);
      rt_pin_ptrs(peer_alloc, 1);
      p->pinned.insert(p->pinned.end(), peer_alloc.begin(), peer_alloc.end());
      std::vector<CopySpec> copies;
      for (int j = 0; j < 26; ++j) {
        const int64_t to = halo_rank_of(c, p->rank, regions[j].dir);
        copies.push_back({sct[j].get(), alloc, static_cast<uint64_t>(pad), 1, rct[25 - j].get(), peer_alloc[to],
                          static_cast<uint64_t>(pad), 1});
      }
      p->pack = copy_batch_create(copies);
    } else {
    cuda_check(cudaMalloc(&p->recv, static_cast<size_t>(p->seg_total)), "cudaMalloc(halo recv)");
    if (method == SP_HALO_COPY) cuda_check(cudaMalloc(&p->send, static_cast<size_t>(p->seg_total)), "cudaMalloc");
    std::vector<uint8_t *> peer_recv;
    rt_exchange_ptr(p->recv, peer_recv);
    rt_pin_ptrs(peer_recv, 1);
    p->pinned.insert(p->pinned.end(), peer_recv.begin(), peer_recv.end());
    if (method == SP_HALO_COPY) {
      rt_exchange_ptr(p->send, p->peer_send);
      rt_pin_ptrs(p->peer_send, 1);
      p->pinned.insert(p->pinned.end(), p->peer_send.begin(), p->peer_send.end());
    }
    for (int j = 0; j < 26; ++j) {
      if (method != SP_HALO_COPY) {
        // segment j of this rank is segment 25-j of the rank at +d_j,
        // written straight into that rank's HBM (halo.hpp:237-254)
        const int64_t to = halo_rank_of(c, p->rank, regions[j].dir);
        packs.push_back({sct[j].get(), alloc, static_cast<uint64_t>(pad), 1, peer_recv[to],
                         static_cast<uint64_t>(p->seg_total), p->seg_off[25 - j]});
      } else {
        packs.push_back({sct[j].get(), alloc, static_cast<uint64_t>(pad), 1, p->send,
                         static_cast<uint64_t>(p->seg_total), p->seg_off[j]});
        p->copy_src_rank.push_back(halo_rank_of(c, p->rank, regions[j].dir));
      }
      unpacks.push_back({rct[j].get(), p->recv, static_cast<uint64_t>(p->seg_total), 1, alloc,
                         static_cast<uint64_t>(pad), p->seg_off[j]});
    }
    p->pack = batch_create(packs, false);
    p->unpack = batch_create(unpacks, true);
    }
    for (auto &e : p->ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    if (method == SP_HALO_FUSED_ASYNC || method == SP_HALO_DIRECT) {
      cuda_check(cudaMalloc(&p->dev_iter, sizeof(uint64_t)), "cudaMalloc(iteration counter)");
      cuda_check(cudaMemset(p->dev_iter, 0, sizeof(uint64_t)), "cudaMemset(iteration counter)");
      const int n = rt_size();
      cuda_check(cudaMalloc(&p->flags, 2 * n * sizeof(uint64_t)), "cudaMalloc(flags)");
      cuda_check(cudaMemset(p->flags, 0, 2 * n * sizeof(uint64_t)), "cudaMemset(flags)");
      cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
      rt_exchange_ptr(p->flags, p->peer_flags);
      rt_pin_ptrs(p->peer_flags, 1);
      p->pinned.insert(p->pinned.end(), p->peer_flags.begin(), p->peer_flags.end());
      int mydev = 0;
      cuda_check(cudaGetDevice(&mydev), "cudaGetDevice");
      p->remote_peers = rt_peers_remote();
      for (uint8_t *pf : p->peer_flags) {
        cudaPointerAttributes at{};
        if (pf && cudaPointerGetAttributes(&at, pf) == cudaSuccess && at.device != mydev) p->remote_peers = true;
      }
      cudaGetLastError();
      // edges to this rank itself need no flags: its own earlier launches
      // on the same stream (the previous iteration's consumers) have
      // completed before this one starts, and this launch's own stores are
      // complete when it ends -- so a 1x1x1 grid runs with no protocol and
      // the periodic self-neighbours of a 2x1x1 / 2x2x1 grid drop out
      std::vector<char> seen_out(n, 0), seen_in(n, 0);
      // SPB_HALO_SELF_FLAGS keeps the self edges in the protocol: a one-GPU
      // measurement of what the flags cost (scripts/protocol_cost.py)
      if (!std::getenv("SPB_HALO_SELF_FLAGS")) seen_out[p->rank] = seen_in[p->rank] = 1;
      for (int j = 0; j < 26; ++j) {
        const int64_t nb = halo_rank_of(c, p->rank, regions[j].dir);
        if (!seen_out[nb]) {
          seen_out[nb] = 1;
          p->out_peers.push_back(static_cast<int>(nb));
        }
        const int64_t from = halo_rank_of(c, p->rank, {-regions[j].dir[0], -regions[j].dir[1], -regions[j].dir[2]});
        if (!seen_in[from]) {
          seen_in[from] = 1;
          p->in_peers.push_back(static_cast<int>(from));
        }
      }
    }
    *out = p.release();
  });
}

// collective; times[0..3] = pack, exchange, unpack, whole iteration (s),
// measured with CUDA events on this rank's stream
sp_status sp_halo_plan_exchange(sp_halo_plan p, double times[4]) {
  SPB_TRACE("sp_halo_plan_exchange");
  return guarded([&] {
    need(p);
    cudaStream_t s = static_cast<cudaStream_t>(rt_stream());
    // The flag values of an exchange are per iteration (FREE=n-1, READY=n).
    // A launch captured into a CUDA graph is replayed with its parameters
    // frozen, so a captured exchange numbers its iterations on the device
    // instead: a one-thread tick kernel advances the plan's counter and the
    // copy kernels derive FREE/READY from it. With every rank on its own GPU
    // the waits are in the copy kernels as usual; with ranks sharing a GPU
    // (whose stream memory operations carry fixed values) a one-warp kernel
    // publishes and waits ahead of each launch instead. A plan with no peer
    // (a 1x1x1 grid) has no flags at all.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing(s, &cap), "cudaStreamIsCapturing");
    const bool capturing = cap != cudaStreamCaptureStatusNone;
    const bool peers = !p->out_peers.empty() || !p->in_peers.empty();
    if (capturing) {
      if (p->method != SP_HALO_DIRECT && p->method != SP_HALO_FUSED_ASYNC)
        fail(SP_ERR_UNSUPPORTED, "halo exchange capture: only the device-ordered methods (DIRECT, FUSED_ASYNC)");
      if (times) fail(SP_ERR_INVALID_ARGUMENT, "halo exchange capture: a captured exchange only enqueues (times == NULL)");
      p->graph_mode = true;
    }
    // one iteration's protocol values: host-numbered (recorded on the
    // device), or device-numbered after a tick
    auto number = [&](BatchSignal &b, int64_t pre_add, int64_t wait_add, int wait_shift, int64_t post_add,
                      int post_shift, uint64_t it, bool first) {
      if (p->graph_mode && peers) { // (no peer: no flag, nothing to number)
        b.iter = p->dev_iter;
        b.pre_add = pre_add;
        b.wait_add = wait_add;
        b.wait_shift = wait_shift;
        b.post_add = post_add;
        b.post_shift = post_shift;
      } else if (first) {
        b.iter_store = p->dev_iter;
        b.iter_value = it;
      }
    };
    if (p->graph_mode && peers) iter_tick(p->dev_iter, s);
    // the device-ordered methods record their events only for timings (an
    // enqueue-only call, captured or not, never reads them)
    auto mark = [&](int k) {
      if (times) cuda_check(cudaEventRecord(p->ev[k], s), "cudaEventRecord");
    };
    if (p->method == SP_HALO_DIRECT) {
      // one copy launch per iteration: block 0 first tells this rank's
      // senders that the ghosts of iteration n-1 are consumed (FREE=n-1;
      // everything earlier on the stream has completed), every block waits
      // for FREE=n-1 from its receivers, the regions are stored into the
      // receivers' ghost cells over NVLink, every block adds its share of
      // READY=n to each receiver once its stores are done, and block 0 then
      // waits for READY=n from this rank's senders, so later work on the
      // stream sees whole ghost shells.
      const int n = rt_size(), me = p->rank;
      const uint64_t it = ++p->iter;
      auto at = [&](uint8_t *base, int kind, int peer) {
        return reinterpret_cast<uint64_t *>(base + static_cast<size_t>(kind * n + peer) * sizeof(uint64_t));
      };
      uint8_t *mine = reinterpret_cast<uint8_t *>(p->flags);
      BatchSignal ks;
      std::vector<const uint64_t *> ready;
      for (int q : p->in_peers) {
        ks.pre.push_back(at(p->peer_flags[q], kFree, me));
        ready.push_back(at(mine, kReady, q));
      }
      ks.pre_value = it - 1;
      for (int q : p->out_peers) {
        ks.wait.push_back(at(mine, kFree, q));
        ks.signal.push_back(at(p->peer_flags[q], kReady, me));
      }
      ks.wait_value = it - 1;
      ks.sys_scope = p->remote_peers;
      // block 0, after adding its share of READY=n, waits for READY=n from
      // this rank's senders: the launch completes only when the ghost shell
      // is whole, so no separate wait kernel
      ks.stream_waits = rt_flag_waits_in_stream();
      ks.post = ready;
      ks.post_value = it << 32; // READY counts 2^32 per sender launch
      ks.err = rt_device_err();
      ks.timeout_ns = rt_device_timeout_ns();
      number(ks, -1, -1, 0, 0, 32, it, true); // FREE = n-1, READY = n << 32
      mark(0);
      batch_execute_signaled(*p->pack, s, ks);
      mark(3); // one launch: no phase boundaries
    } else if (p->method == SP_HALO_FUSED_ASYNC) {
      // device-ordered iteration, signalled from inside the kernels: the
      // pack batch waits (in every block) until each receiver has consumed
      // iteration n-1, stores the segments into the receivers' HBM, and its
      // blocks add their shares of READY=n to each receiver's counter; the
      // unpack batch waits for READY=n from each sender and releases FREE=n
      // back. No host barrier, no stream memory op, no host round trip.
      const int n = rt_size(), me = p->rank;
      const uint64_t it = ++p->iter;
      auto at = [&](uint8_t *base, int kind, int peer) {
        return reinterpret_cast<uint64_t *>(base + static_cast<size_t>(kind * n + peer) * sizeof(uint64_t));
      };
      uint8_t *mine = reinterpret_cast<uint8_t *>(p->flags);
      BatchSignal ps, us;
      for (int q : p->out_peers) {
        ps.wait.push_back(at(mine, kFree, q));
        ps.signal.push_back(at(p->peer_flags[q], kReady, me));
      }
      ps.wait_value = (it - 1) << 32; // FREE and READY count 2^32 per launch
      for (int q : p->in_peers) {
        us.wait.push_back(at(mine, kReady, q));
        us.signal.push_back(at(p->peer_flags[q], kFree, me));
      }
      us.wait_value = it << 32;
      ps.sys_scope = us.sys_scope = p->remote_peers;
      ps.stream_waits = us.stream_waits = rt_flag_waits_in_stream();
      ps.err = us.err = rt_device_err();
      ps.timeout_ns = us.timeout_ns = rt_device_timeout_ns();
      number(ps, 0, -1, 32, 0, 0, it, true); // the pack waits FREE = (n-1) << 32
      number(us, 0, 0, 32, 0, 0, it, false); // the unpack waits READY = n << 32
      mark(0);
      batch_execute_signaled(*p->pack, s, ps);
      mark(1);
      mark(2);
      batch_execute_signaled(*p->unpack, s, us);
      mark(3);
    } else {
    rt_barrier(); // every neighbour has consumed the previous iteration
    cuda_check(cudaEventRecord(p->ev[0], s), "cudaEventRecord");
    batch_execute(*p->pack, s);
    cuda_check(cudaEventRecord(p->ev[1], s), "cudaEventRecord");
    if (p->method == SP_HALO_COPY) {
      cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
      rt_barrier(); // all send buffers packed
      for (int k = 0; k < 26; ++k) {
        const int64_t from = p->copy_src_rank[k];
        cuda_check(cudaMemcpyAsync(p->recv + p->seg_off[k], p->peer_send[from] + p->seg_off[25 - k],
                                   static_cast<size_t>(p->seg_off[k + 1] - p->seg_off[k]), cudaMemcpyDefault, s),
                   "segment copy");
      }
    }
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    rt_barrier(); // every segment addressed to this rank has landed
    cuda_check(cudaEventRecord(p->ev[2], s), "cudaEventRecord");
    batch_execute(*p->unpack, s);
    cuda_check(cudaEventRecord(p->ev[3], s), "cudaEventRecord");
    }
    // device-ordered methods need no host synchronisation: without timings
    // the call only enqueues, and iterations pipeline on the runtime stream
    const bool async = !times && (p->method == SP_HALO_DIRECT || p->method == SP_HALO_FUSED_ASYNC);
    if (!async) rt_sync_event(p->ev[3], "halo exchange");
    // a flag wait of this (or, enqueue-only, an earlier) iteration gave up
    rt_check_device_error("halo exchange");
    if (times) {
      float a = 0, b = 0, d = 0, t = 0;
      cudaEventElapsedTime(&t, p->ev[0], p->ev[3]);
      if (p->method == SP_HALO_DIRECT) {
        a = t; // the copy is the whole iteration
      } else {
        cudaEventElapsedTime(&a, p->ev[0], p->ev[1]);
        cudaEventElapsedTime(&b, p->ev[1], p->ev[2]);
        cudaEventElapsedTime(&d, p->ev[2], p->ev[3]);
      }
      times[0] = a * 1e-3;
      times[1] = b * 1e-3;
      times[2] = d * 1e-3;
      times[3] = t * 1e-3;
    }
  });
}

sp_status sp_halo_plan_free(sp_halo_plan p) {
  delete p;
  return SP_OK;
}

} // extern "C"
