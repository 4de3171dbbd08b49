/* TEST INFRASTRUCTURE: an Open MPI-style mpi.h (declarations only) --
 * opaque POINTER handles and predefined objects, a standard MPI_Status
 * without the engine's extra fields. tests/test_interpose.py compiles
 * paper_2012_14363_b200/csrc/interpose.cpp against it to show that the
 * interposer builds against a vendor header whose handles are not ints, as
 * a site rebuilding it for its own MPI would. Never linked. */
#ifndef OMPI_STYLE_MPI_H
#define OMPI_STYLE_MPI_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef struct ompi_datatype_t *MPI_Datatype;
typedef struct ompi_communicator_t *MPI_Comm;
typedef struct ompi_request_t *MPI_Request;
typedef struct ompi_info_t *MPI_Info;
typedef ptrdiff_t MPI_Aint;
typedef struct ompi_status_public_t {
  int MPI_SOURCE, MPI_TAG, MPI_ERROR;
  int _cancelled;
  size_t _ucount;
} MPI_Status;
extern struct ompi_predefined_datatype_t ompi_mpi_byte, ompi_mpi_char, ompi_mpi_unsigned_char, ompi_mpi_packed,
    ompi_mpi_int, ompi_mpi_float, ompi_mpi_double;
extern struct ompi_predefined_communicator_t ompi_mpi_comm_world;
#define MPI_BYTE ((MPI_Datatype)&ompi_mpi_byte)
#define MPI_CHAR ((MPI_Datatype)&ompi_mpi_char)
#define MPI_UNSIGNED_CHAR ((MPI_Datatype)&ompi_mpi_unsigned_char)
#define MPI_PACKED ((MPI_Datatype)&ompi_mpi_packed)
#define MPI_INT ((MPI_Datatype)&ompi_mpi_int)
#define MPI_FLOAT ((MPI_Datatype)&ompi_mpi_float)
#define MPI_DOUBLE ((MPI_Datatype)&ompi_mpi_double)
#define MPI_DATATYPE_NULL ((MPI_Datatype)0)
#define MPI_COMM_WORLD ((MPI_Comm)&ompi_mpi_comm_world)
#define MPI_REQUEST_NULL ((MPI_Request)0)
#define MPI_STATUS_IGNORE ((MPI_Status *)0)
#define MPI_SUCCESS 0
#define MPI_ERR_TYPE 3
#define MPI_ERR_ARG 13
#define MPI_ERR_TRUNCATE 15
#define MPI_ERR_INTERN 17
#define MPI_ERR_NO_MEM 34
#define MPI_ERR_UNSUPPORTED_OPERATION 52
#define MPI_UNDEFINED (-32766)
#define MPI_ORDER_C 0
int MPI_Init(int *, char ***);
int MPI_Init_thread(int *, char ***, int, int *);
int MPI_Finalize(void);
int MPI_Comm_rank(MPI_Comm, int *);
int MPI_Comm_size(MPI_Comm, int *);
int MPI_Comm_free(MPI_Comm *);
int MPI_Get_count(const MPI_Status *, MPI_Datatype, int *);
int MPI_Type_contiguous(int, MPI_Datatype, MPI_Datatype *);
int MPI_Type_vector(int, int, int, MPI_Datatype, MPI_Datatype *);
int MPI_Type_create_hvector(int, int, MPI_Aint, MPI_Datatype, MPI_Datatype *);
int MPI_Type_create_subarray(int, const int[], const int[], const int[], int, MPI_Datatype, MPI_Datatype *);
int MPI_Type_indexed(int, const int[], const int[], MPI_Datatype, MPI_Datatype *);
int MPI_Type_create_hindexed(int, const int[], const MPI_Aint[], MPI_Datatype, MPI_Datatype *);
int MPI_Type_create_indexed_block(int, int, const int[], MPI_Datatype, MPI_Datatype *);
int MPI_Type_create_hindexed_block(int, int, const MPI_Aint[], MPI_Datatype, MPI_Datatype *);
int MPI_Type_create_struct(int, const int[], const MPI_Aint[], const MPI_Datatype[], MPI_Datatype *);
int MPI_Type_create_resized(MPI_Datatype, MPI_Aint, MPI_Aint, MPI_Datatype *);
int MPI_Type_commit(MPI_Datatype *);
int MPI_Type_free(MPI_Datatype *);
int MPI_Pack(const void *, int, MPI_Datatype, void *, int, int *, MPI_Comm);
int MPI_Unpack(const void *, int, int *, void *, int, MPI_Datatype, MPI_Comm);
int MPI_Send(const void *, int, MPI_Datatype, int, int, MPI_Comm);
int MPI_Recv(void *, int, MPI_Datatype, int, int, MPI_Comm, MPI_Status *);
int MPI_Isend(const void *, int, MPI_Datatype, int, int, MPI_Comm, MPI_Request *);
int MPI_Irecv(void *, int, MPI_Datatype, int, int, MPI_Comm, MPI_Request *);
int MPI_Wait(MPI_Request *, MPI_Status *);
int MPI_Waitall(int, MPI_Request[], MPI_Status[]);
int MPI_Test(MPI_Request *, int *, MPI_Status *);
int MPI_Waitany(int, MPI_Request[], int *, MPI_Status *);
int MPI_Waitsome(int, MPI_Request[], int *, int[], MPI_Status[]);
int MPI_Testany(int, MPI_Request[], int *, int *, MPI_Status *);
int MPI_Testall(int, MPI_Request[], int *, MPI_Status[]);
int MPI_Request_free(MPI_Request *);
int MPI_Send_init(const void *, int, MPI_Datatype, int, int, MPI_Comm, MPI_Request *);
int MPI_Recv_init(void *, int, MPI_Datatype, int, int, MPI_Comm, MPI_Request *);
int MPI_Start(MPI_Request *);
int MPI_Startall(int, MPI_Request[]);
int MPI_Sendrecv(const void *, int, MPI_Datatype, int, int, void *, int, MPI_Datatype, int, int, MPI_Comm,
                 MPI_Status *);
int MPI_Dist_graph_create_adjacent(MPI_Comm, int, const int[], const int[], int, const int[], const int[], MPI_Info,
                                   int, MPI_Comm *);
int MPI_Cart_create(MPI_Comm, int, const int[], const int[], int, MPI_Comm *);
int MPI_Neighbor_alltoallv(const void *, const int[], const int[], MPI_Datatype, void *, const int[], const int[],
                           MPI_Datatype, MPI_Comm);
int MPI_Neighbor_alltoallw(const void *, const int[], const MPI_Aint[], const MPI_Datatype[], void *, const int[],
                           const MPI_Aint[], const MPI_Datatype[], MPI_Comm);
int MPI_Neighbor_alltoallw_init(const void *, const int[], const MPI_Aint[], const MPI_Datatype[], void *,
                                const int[], const MPI_Aint[], const MPI_Datatype[], MPI_Comm, MPI_Info,
                                MPI_Request *);
int MPI_Neighbor_alltoallv_init(const void *, const int[], const int[], MPI_Datatype, void *, const int[],
                                const int[], MPI_Datatype, MPI_Comm, MPI_Info, MPI_Request *);
int MPI_Alltoallv(const void *, const int[], const int[], MPI_Datatype, void *, const int[], const int[],
                  MPI_Datatype, MPI_Comm);
int MPI_Alltoallw(const void *, const int[], const int[], const MPI_Datatype[], void *, const int[], const int[],
                  const MPI_Datatype[], MPI_Comm);
#ifdef __cplusplus
}
#endif
#endif
