/*
 * mpi.h -- the MPI subset exported by libtempi_b200.so.
 *
 * TEMPI is an interposer: it exports part of the MPI interface and forwards
 * the rest to the system MPI through PMPI_* (PAPER.md:781-796). This image
 * has no MPI, so libtempi_b200.so carries both layers: MPI_* (the
 * datatype-accelerated entry points: commit-time canonicalisation,
 * sm_100a pack/unpack kernels, model-selected transfers, fused
 * pack-to-peer neighbour exchange) and PMPI_* (a node-local runtime: one
 * process per GPU, shared-memory control plane, CUDA IPC data plane).
 * Handles are plain ints (MPICH-style); sizes follow MPI-3.1.
 *
 * Launch: any launcher that sets RANK/WORLD_SIZE/LOCAL_RANK (torchrun) or
 * TEMPI_RANK/TEMPI_SIZE (tools/tempirun), plus a job id shared by the ranks
 * (TEMPI_JOB, TORCHELASTIC_RUN_ID or MASTER_PORT).
 */
#ifndef TEMPI_B200_MPI_H
#define TEMPI_B200_MPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int MPI_Datatype;
typedef int MPI_Comm;
typedef int MPI_Request;
typedef int MPI_Info;
typedef int64_t MPI_Aint;
typedef int64_t MPI_Count;

typedef struct {
  int MPI_SOURCE;
  int MPI_TAG;
  int MPI_ERROR;
  int method;      /* transfer method used (0 oneshot, 1 device, 2 staged) */
  int64_t bytes;   /* bytes received */
} MPI_Status;

#define MPI_SUCCESS 0
#define MPI_ERR_BUFFER 1
#define MPI_ERR_COUNT 2
#define MPI_ERR_TYPE 3
#define MPI_ERR_TAG 4
#define MPI_ERR_COMM 5
#define MPI_ERR_RANK 6
#define MPI_ERR_ARG 12
#define MPI_ERR_TRUNCATE 14
#define MPI_ERR_OTHER 15
#define MPI_ERR_INTERN 16
#define MPI_ERR_UNSUPPORTED_OPERATION 52
#define MPI_ERR_NO_MEM 34

#define MPI_COMM_NULL ((MPI_Comm)0)
#define MPI_COMM_WORLD ((MPI_Comm)1)
#define MPI_COMM_SELF ((MPI_Comm)2)

#define MPI_DATATYPE_NULL ((MPI_Datatype)0)
#define MPI_BYTE ((MPI_Datatype)1)
#define MPI_CHAR ((MPI_Datatype)2)
#define MPI_INT ((MPI_Datatype)3)
#define MPI_FLOAT ((MPI_Datatype)4)
#define MPI_DOUBLE ((MPI_Datatype)5)
#define MPI_PACKED ((MPI_Datatype)6)
#define MPI_UNSIGNED_CHAR ((MPI_Datatype)7)

#define MPI_ANY_SOURCE (-1)
#define MPI_ANY_TAG (-1)
#define MPI_PROC_NULL (-2)
#define MPI_UNDEFINED (-32766)
#define MPI_STATUS_IGNORE ((MPI_Status *)0)
#define MPI_STATUSES_IGNORE ((MPI_Status *)0)
#define MPI_REQUEST_NULL ((MPI_Request)0)
#define MPI_UNWEIGHTED ((int *)0)
#define MPI_INFO_NULL ((MPI_Info)0)
#define MPI_ORDER_C 56
#define MPI_ORDER_FORTRAN 57
#define MPI_THREAD_SINGLE 0
#define MPI_THREAD_FUNNELED 1
#define MPI_THREAD_SERIALIZED 2
#define MPI_THREAD_MULTIPLE 3
#define MPI_MAX_ERROR_STRING 256

/* runtime */
int MPI_Init(int *argc, char ***argv);
int MPI_Init_thread(int *argc, char ***argv, int required, int *provided);
int MPI_Initialized(int *flag);
int MPI_Finalize(void);
int MPI_Finalized(int *flag);
int MPI_Comm_rank(MPI_Comm comm, int *rank);
int MPI_Comm_size(MPI_Comm comm, int *size);
int MPI_Barrier(MPI_Comm comm);
int MPI_Abort(MPI_Comm comm, int errorcode);
double MPI_Wtime(void);
int MPI_Error_string(int errorcode, char *string, int *resultlen);
int MPI_Get_count(const MPI_Status *status, MPI_Datatype datatype, int *count);

/* derived datatypes (accelerated: canonicalised at commit) */
int MPI_Type_contiguous(int count, MPI_Datatype oldtype, MPI_Datatype *newtype);
int MPI_Type_vector(int count, int blocklength, int stride, MPI_Datatype oldtype, MPI_Datatype *newtype);
int MPI_Type_create_hvector(int count, int blocklength, MPI_Aint stride, MPI_Datatype oldtype,
                            MPI_Datatype *newtype);
int MPI_Type_create_subarray(int ndims, const int sizes[], const int subsizes[], const int starts[], int order,
                             MPI_Datatype oldtype, MPI_Datatype *newtype);
/* beyond the reference (MPI-3.1 4.1.4-4.1.7; TEMPI's future work): regular
 * index patterns canonicalise to strided kernels, irregular ones run on the
 * device run-table kernel; displacements must be nonnegative */
int MPI_Type_indexed(int count, const int blocklengths[], const int displacements[], MPI_Datatype oldtype,
                     MPI_Datatype *newtype);
int MPI_Type_create_hindexed(int count, const int blocklengths[], const MPI_Aint displacements[],
                             MPI_Datatype oldtype, MPI_Datatype *newtype);
int MPI_Type_create_indexed_block(int count, int blocklength, const int displacements[], MPI_Datatype oldtype,
                                  MPI_Datatype *newtype);
int MPI_Type_create_hindexed_block(int count, int blocklength, const MPI_Aint displacements[],
                                   MPI_Datatype oldtype, MPI_Datatype *newtype);
int MPI_Type_create_struct(int count, const int blocklengths[], const MPI_Aint displacements[],
                           const MPI_Datatype types[], MPI_Datatype *newtype);
int MPI_Type_create_resized(MPI_Datatype oldtype, MPI_Aint lb, MPI_Aint extent, MPI_Datatype *newtype);
int MPI_Type_commit(MPI_Datatype *datatype);
int MPI_Type_free(MPI_Datatype *datatype);
int MPI_Type_size(MPI_Datatype datatype, int *size);
int MPI_Type_get_extent(MPI_Datatype datatype, MPI_Aint *lb, MPI_Aint *extent);

/* packing (accelerated: sm_100a kernels) */
int MPI_Pack(const void *inbuf, int incount, MPI_Datatype datatype, void *outbuf, int outsize, int *position,
             MPI_Comm comm);
int MPI_Unpack(const void *inbuf, int insize, int *position, void *outbuf, int outcount, MPI_Datatype datatype,
               MPI_Comm comm);
int MPI_Pack_size(int incount, MPI_Datatype datatype, MPI_Comm comm, int *size);

/* point to point (accelerated: model-selected device/one-shot/staged) */
int MPI_Send(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm);
int MPI_Recv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
             MPI_Status *status);
/* non-blocking point to point: requests progressed by every MPI call;
 * messages above two chunks (TEMPI_CHUNK, default 4 MiB) are pipelined
 * chunk by chunk, device-to-device messages run as one fused copy kernel */
int MPI_Isend(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
              MPI_Request *request);
int MPI_Irecv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
              MPI_Request *request);
int MPI_Wait(MPI_Request *request, MPI_Status *status);
int MPI_Waitall(int count, MPI_Request requests[], MPI_Status statuses[]);
int MPI_Test(MPI_Request *request, int *flag, MPI_Status *status);
/* completion of any / some / all of a set (MPI-3.1 3.7.5); MPI_Request_free
 * of an active request completes it first */
int MPI_Waitany(int count, MPI_Request requests[], int *index, MPI_Status *status);
int MPI_Waitsome(int incount, MPI_Request requests[], int *outcount, int indices[], MPI_Status statuses[]);
int MPI_Testany(int count, MPI_Request requests[], int *index, int *flag, MPI_Status *status);
int MPI_Testall(int count, MPI_Request requests[], int *flag, MPI_Status statuses[]);
int MPI_Request_free(MPI_Request *request);
/* persistent requests (MPI-3.1 3.9): MPI_Start / MPI_Startall begin the
 * recorded operation; completion leaves the request inactive, not freed */
int MPI_Send_init(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
                  MPI_Request *request);
int MPI_Recv_init(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
                  MPI_Request *request);
int MPI_Start(MPI_Request *request);
int MPI_Startall(int count, MPI_Request requests[]);
int MPI_Sendrecv(const void *sendbuf, int sendcount, MPI_Datatype sendtype, int dest, int sendtag, void *recvbuf,
                 int recvcount, MPI_Datatype recvtype, int source, int recvtag, MPI_Comm comm,
                 MPI_Status *status);

/* topologies + neighbourhood exchange (accelerated: fused pack-to-peer) */
int MPI_Dist_graph_create_adjacent(MPI_Comm comm_old, int indegree, const int sources[],
                                   const int sourceweights[], int outdegree, const int destinations[],
                                   const int destweights[], MPI_Info info, int reorder, MPI_Comm *comm_dist_graph);
int MPI_Dist_graph_neighbors_count(MPI_Comm comm, int *indegree, int *outdegree, int *weighted);
int MPI_Dist_graph_neighbors(MPI_Comm comm, int maxindegree, int sources[], int sourceweights[],
                             int maxoutdegree, int destinations[], int destweights[]);
int MPI_Cart_create(MPI_Comm comm_old, int ndims, const int dims[], const int periods[], int reorder,
                    MPI_Comm *comm_cart);
int MPI_Cart_coords(MPI_Comm comm, int rank, int maxdims, int coords[]);
int MPI_Cart_rank(MPI_Comm comm, const int coords[], int *rank);
int MPI_Cart_shift(MPI_Comm comm, int direction, int disp, int *rank_source, int *rank_dest);
int MPI_Comm_free(MPI_Comm *comm);
int MPI_Neighbor_alltoallv(const void *sendbuf, const int sendcounts[], const int sdispls[],
                           MPI_Datatype sendtype, void *recvbuf, const int recvcounts[], const int rdispls[],
                           MPI_Datatype recvtype, MPI_Comm comm);

/* per-neighbour datatypes on both sides, byte displacements (accelerated:
 * one typed-copy launch per rank stores every block at its final strided
 * place in the receiver's buffer over NVLink) */
int MPI_Neighbor_alltoallw(const void *sendbuf, const int sendcounts[], const MPI_Aint sdispls[],
                           const MPI_Datatype sendtypes[], void *recvbuf, const int recvcounts[],
                           const MPI_Aint rdispls[], const MPI_Datatype recvtypes[], MPI_Comm comm);

/* persistent neighbourhood collectives (MPI-4.0 7.10.2): start with
 * MPI_Start / MPI_Startall, complete with the MPI_Wait family, release with
 * MPI_Request_free. Compiled once into one signalled typed-copy launch per
 * start (no host entry protocol); the starts capture into CUDA graphs on
 * sp_rt_stream. Types the engine cannot compile (irregular layouts) re-run
 * the collective at every start. */
int MPI_Neighbor_alltoallw_init(const void *sendbuf, const int sendcounts[], const MPI_Aint sdispls[],
                                const MPI_Datatype sendtypes[], void *recvbuf, const int recvcounts[],
                                const MPI_Aint rdispls[], const MPI_Datatype recvtypes[], MPI_Comm comm,
                                MPI_Info info, MPI_Request *request);
int MPI_Neighbor_alltoallv_init(const void *sendbuf, const int sendcounts[], const int sdispls[],
                                MPI_Datatype sendtype, void *recvbuf, const int recvcounts[], const int rdispls[],
                                MPI_Datatype recvtype, MPI_Comm comm, MPI_Info info, MPI_Request *request);

/* all-to-all with derived datatypes (beyond the paper, whose future work
 * lists collectives): the neighbour machinery over the
 * complete graph of the communicator -- one typed-copy launch per rank
 * stores every block at its final strided place in the receiver's buffer.
 * Alltoallv displacements are in extents, Alltoallw's in bytes (MPI-3.1
 * 5.8). */
int MPI_Alltoallv(const void *sendbuf, const int sendcounts[], const int sdispls[], MPI_Datatype sendtype,
                  void *recvbuf, const int recvcounts[], const int rdispls[], MPI_Datatype recvtype, MPI_Comm comm);
int MPI_Alltoallw(const void *sendbuf, const int sendcounts[], const int sdispls[], const MPI_Datatype sendtypes[],
                  void *recvbuf, const int recvcounts[], const int rdispls[], const MPI_Datatype recvtypes[],
                  MPI_Comm comm);

/* profiling interface: the base implementations under the interposer */
int PMPI_Init(int *argc, char ***argv);
int PMPI_Finalize(void);
int PMPI_Comm_rank(MPI_Comm comm, int *rank);
int PMPI_Comm_size(MPI_Comm comm, int *size);
int PMPI_Barrier(MPI_Comm comm);
int PMPI_Type_commit(MPI_Datatype *datatype);
int PMPI_Pack(const void *inbuf, int incount, MPI_Datatype datatype, void *outbuf, int outsize, int *position,
              MPI_Comm comm);
int PMPI_Unpack(const void *inbuf, int insize, int *position, void *outbuf, int outcount, MPI_Datatype datatype,
                MPI_Comm comm);
int PMPI_Send(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm);
int PMPI_Recv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
              MPI_Status *status);
int PMPI_Isend(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
               MPI_Request *request);
int PMPI_Irecv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
               MPI_Request *request);
int PMPI_Wait(MPI_Request *request, MPI_Status *status);
int PMPI_Neighbor_alltoallv(const void *sendbuf, const int sendcounts[], const int sdispls[],
                            MPI_Datatype sendtype, void *recvbuf, const int recvcounts[], const int rdispls[],
                            MPI_Datatype recvtype, MPI_Comm comm);
int PMPI_Neighbor_alltoallw(const void *sendbuf, const int sendcounts[], const MPI_Aint sdispls[],
                            const MPI_Datatype sendtypes[], void *recvbuf, const int recvcounts[],
                            const MPI_Aint rdispls[], const MPI_Datatype recvtypes[], MPI_Comm comm);

int PMPI_Alltoallv(const void *sendbuf, const int sendcounts[], const int sdispls[], MPI_Datatype sendtype,
                   void *recvbuf, const int recvcounts[], const int rdispls[], MPI_Datatype recvtype, MPI_Comm comm);
int PMPI_Alltoallw(const void *sendbuf, const int sendcounts[], const int sdispls[], const MPI_Datatype sendtypes[],
                   void *recvbuf, const int recvcounts[], const int rdispls[], const MPI_Datatype recvtypes[],
                   MPI_Comm comm);

/* TEMPI-specific controls (not MPI): force a transfer method for MPI_Send /
 * MPI_Isend (-1 = model-selected, the default; 0 one-shot, 1 device, 2
 * staged, 3 direct = fused copy into the receiver's device buffer), load a
 * machine profile. */
int TEMPI_Set_method(int method);
int TEMPI_Load_profile(const char *path);

#ifdef __cplusplus
}
#endif
#endif /* TEMPI_B200_MPI_H */
