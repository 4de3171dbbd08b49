/* Non-blocking point to point on device buffers: every rank posts an
 * MPI_Irecv from its left and an MPI_Isend to its right for several
 * messages at once (3D subarrays of different shapes, every transfer
 * method, a message large enough to be pipelined in chunks), completes them
 * with MPI_Waitall / MPI_Test loops, then an MPI_Sendrecv; bytes checked on
 * the host against the MPI definition. Prints "OK". */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include <mpi.h>

#define CHECK(c) do { if (!(c)) { printf("FAIL rank %d line %d: %s\n", rank, __LINE__, #c); MPI_Abort(MPI_COMM_WORLD, 1); } } while (0)

static unsigned char pat(long i, int salt) { return (unsigned char)((i * 131 + salt * 29 + 3) >> 1); }

enum { NMSG = 5 };

int main(int argc, char **argv) {
  int rank = 0, size = 0;
  MPI_Init(&argc, &argv);
  MPI_Comm_rank(MPI_COMM_WORLD, &rank);
  MPI_Comm_size(MPI_COMM_WORLD, &size);
  const int right = (rank + 1) % size, left = (rank + size - 1) % size;
  /* (Z, Y, X) byte arrays, x fastest; message k uses shape k */
  const int shapes[NMSG][9] = {
      {16, 48, 256, 8, 32, 64, 3, 5, 64},        /* 16 KiB, 64-B rows */
      {64, 64, 1024, 40, 48, 512, 7, 9, 32},     /* 960 KiB, 512-B rows: chunked */
      {8, 16, 96, 5, 7, 24, 1, 2, 11},           /* odd start, 24-B rows */
      {32, 128, 512, 24, 100, 256, 2, 10, 100},  /* 600 KiB */
      {4, 4, 64, 2, 2, 8, 0, 0, 0},              /* tiny */
  };
  const int methods[NMSG] = {3, -1, 0, 2, 1};
  MPI_Datatype t[NMSG];
  unsigned char *d_src[NMSG], *d_dst[NMSG];
  long n[NMSG];
  for (int k = 0; k < NMSG; ++k) {
    const int *s = shapes[k];
    int sz[3] = {s[0], s[1], s[2]}, sub[3] = {s[3], s[4], s[5]}, st[3] = {s[6], s[7], s[8]};
    CHECK(MPI_Type_create_subarray(3, sz, sub, st, MPI_ORDER_C, MPI_BYTE, &t[k]) == MPI_SUCCESS);
    CHECK(MPI_Type_commit(&t[k]) == MPI_SUCCESS);
    n[k] = (long)s[0] * s[1] * s[2];
    unsigned char *h = malloc(n[k]);
    for (long i = 0; i < n[k]; ++i) h[i] = pat(i, rank * 8 + k);
    cudaMalloc((void **)&d_src[k], n[k]);
    cudaMalloc((void **)&d_dst[k], n[k]);
    cudaMemcpy(d_src[k], h, n[k], cudaMemcpyHostToDevice);
    cudaMemset(d_dst[k], 0xA5, n[k]); cudaDeviceSynchronize();
    free(h);
  }
  MPI_Request req[2 * NMSG];
  for (int k = 0; k < NMSG; ++k)
    CHECK(MPI_Irecv(d_dst[k], 1, t[k], left, 100 + k, MPI_COMM_WORLD, &req[k]) == MPI_SUCCESS);
  for (int k = NMSG - 1; k >= 0; --k) {
    CHECK(TEMPI_Set_method(methods[k]) == MPI_SUCCESS);
    CHECK(MPI_Isend(d_src[k], 1, t[k], right, 100 + k, MPI_COMM_WORLD, &req[NMSG + k]) == MPI_SUCCESS);
  }
  TEMPI_Set_method(-1);
  /* the first receive by MPI_Test polling, the rest by MPI_Waitall */
  int flag = 0;
  MPI_Status s0;
  while (!flag) CHECK(MPI_Test(&req[0], &flag, &s0) == MPI_SUCCESS);
  CHECK(req[0] == MPI_REQUEST_NULL && s0.MPI_SOURCE == left && s0.MPI_TAG == 100);
  MPI_Status sts[2 * NMSG];
  CHECK(MPI_Waitall(2 * NMSG, req, sts) == MPI_SUCCESS);
  for (int k = 1; k < NMSG; ++k) CHECK(sts[k].MPI_SOURCE == left && sts[k].MPI_TAG == 100 + k);
  for (int k = 0; k < NMSG; ++k) {
    const int *s = shapes[k];
    unsigned char *h = malloc(n[k]);
    cudaMemcpy(h, d_dst[k], n[k], cudaMemcpyDeviceToHost);
    for (long i = 0; i < n[k]; ++i) {
      const int z = (int)(i / ((long)s[1] * s[2])), y = (int)(i / s[2] % s[1]), x = (int)(i % s[2]);
      const int in = z >= s[6] && z < s[6] + s[3] && y >= s[7] && y < s[7] + s[4] && x >= s[8] && x < s[8] + s[5];
      CHECK(h[i] == (in ? pat(i, left * 8 + k) : 0xA5));
    }
    free(h);
  }
  /* MPI_Sendrecv around the ring with message 1's type */
  cudaMemset(d_dst[1], 0, n[1]); cudaDeviceSynchronize();
  MPI_Status ss;
  CHECK(MPI_Sendrecv(d_src[1], 1, t[1], right, 7, d_dst[1], 1, t[1], left, 7, MPI_COMM_WORLD, &ss) == MPI_SUCCESS);
  CHECK(ss.MPI_SOURCE == left && ss.MPI_TAG == 7);
  MPI_Request nul = MPI_REQUEST_NULL;
  CHECK(MPI_Wait(&nul, MPI_STATUS_IGNORE) == MPI_SUCCESS);
  MPI_Barrier(MPI_COMM_WORLD);
  for (int k = 0; k < NMSG; ++k) {
    MPI_Type_free(&t[k]);
    cudaFree(d_src[k]);
    cudaFree(d_dst[k]);
  }
  MPI_Finalize();
  if (rank == 0) printf("OK\n");
  return 0;
}
