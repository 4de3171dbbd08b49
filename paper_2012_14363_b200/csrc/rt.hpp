// rt.hpp -- node-local multi-process runtime (internal).
#pragma once

#include <vector>

#include "core.hpp"
#include "model.hpp"

namespace spb {

struct RtTrace {
  int method;
  int64_t bytes;
};
struct RtStatus {
  int source, tag, method;
  int64_t bytes;
};

void rt_init(int rank, int size, const char *name, int device, int64_t window_bytes, int64_t host_bytes);
void rt_finalize();
// bounded device waits: the limit for in-kernel flag spins (0 = none), the
// flag such a spin sets when it gives up, and the host-side check that
// turns it into SP_ERR_TIMEOUT after a synchronisation
uint64_t rt_device_timeout_ns();
int *rt_device_err();
void rt_check_device_error(const char *what);
// halo / neighbour flag waits in the stream front end (ranks share a GPU)
// rather than in the kernel (every rank on its own GPU); TEMPI_FLAG_WAIT
bool rt_flag_waits_in_stream();
// true when any other rank runs on another GPU (compared by UUID)
bool rt_peers_remote();
// polls a completion event with the peer-liveness checks and TEMPI_TIMEOUT
// of a host wait (stream work that waits on peers' flags)
void rt_sync_event(cudaEvent_t e, const char *what);
int rt_rank();
int rt_size();
void rt_barrier();
void rt_host_send(int dst, int tag, const void *data, int64_t bytes);
int64_t rt_host_recv(int src, int tag, void *data, int64_t cap);
void rt_exchange_ptr(void *local, std::vector<uint8_t *> &out);
// hold (delta > 0) or release (delta < 0) the peer mappings rt_exchange_ptr
// returned: held mappings are never evicted as stale
void rt_pin_ptrs(const std::vector<uint8_t *> &ptrs, int delta);
void rt_send(const void *buf, uint64_t buf_bytes, int64_t count, CommitPtr ct, int dest, int tag, int method,
             RtTrace *trace);
void rt_recv(void *buf, uint64_t buf_bytes, int64_t count, CommitPtr ct, int source, int tag, RtStatus *st);
// non-blocking point to point: request ids, progressed by every runtime call
uint64_t rt_isend(const void *buf, uint64_t buf_bytes, int64_t count, CommitPtr ct, int dest, int tag, int method);
uint64_t rt_irecv(void *buf, uint64_t buf_bytes, int64_t count, CommitPtr ct, int source, int tag);
bool rt_test(uint64_t req, RtStatus *st); // true (and the request is freed) once complete
void rt_wait(uint64_t req, RtStatus *st);
void rt_progress();
void rt_set_chunk(int64_t bytes);
void rt_set_profile(sp_profile_s *p);
int rt_choose(const Committed &ct, int64_t count);
// the B200 model's verdict on DIRECT between this GPU and a device buffer
// on `peer_device` (Eq. 4 vs the reference's best of Eqs. 1-3)
bool model_prefers_direct(const Committed &ct, int64_t count, int peer_device);
void *rt_stream();
// persistent neighbour alltoallw (MPI-4 MPI_Neighbor_alltoallw_init):
// built once (collective), started as one signalled launch per call
struct NbrPlan;
NbrPlan *rt_nbr_plan_create(const uint8_t *sendbuf, const std::vector<int64_t> &send_counts,
                            const std::vector<int64_t> &send_displs, const std::vector<CommitPtr> &send_types,
                            uint8_t *recvbuf, const std::vector<int64_t> &recv_counts,
                            const std::vector<int64_t> &recv_displs, const std::vector<CommitPtr> &recv_types,
                            const std::vector<int> &sources, const std::vector<int> &dests);
void rt_nbr_plan_start(NbrPlan *p);
bool rt_nbr_plan_test(NbrPlan *p);
void rt_nbr_plan_wait(NbrPlan *p);
void rt_nbr_plan_free(NbrPlan *p);
void rt_neighbor_alltoallv(const uint8_t *sendbuf, const std::vector<int64_t> &send_counts,
                           const std::vector<int64_t> &send_displs, const CommitPtr &stp, uint8_t *recvbuf,
                           const std::vector<int64_t> &recv_counts, const std::vector<int64_t> &recv_displs,
                           const Committed &rtp, const std::vector<int> &sources, const std::vector<int> &dests);

void rt_neighbor_alltoallw(const uint8_t *sendbuf, const std::vector<int64_t> &send_counts,
                           const std::vector<int64_t> &send_displs, const std::vector<CommitPtr> &send_types,
                           uint8_t *recvbuf, const std::vector<int64_t> &recv_counts,
                           const std::vector<int64_t> &recv_displs, const std::vector<CommitPtr> &recv_types,
                           const std::vector<int> &sources, const std::vector<int> &dests);

} // namespace spb
