/* Beyond the reference: an irregular MPI_Type_indexed of doubles (a sparse
 * gather list, the typical unstructured-mesh halo) and a struct type on
 * device buffers through MPI_Pack / MPI_Unpack, then MPI_Send with the
 * indexed type received as a contiguous run of doubles, every transfer
 * method. Bytes checked on the host against the MPI typemap definition.
 * Prints "OK". */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include <mpi.h>

#define CHECK(c) do { if (!(c)) { printf("FAIL rank %d line %d: %s\n", rank, __LINE__, #c); MPI_Abort(MPI_COMM_WORLD, 1); } } while (0)

int main(int argc, char **argv) {
  int rank = 0, size = 0;
  MPI_Init(&argc, &argv);
  MPI_Comm_rank(MPI_COMM_WORLD, &rank);
  MPI_Comm_size(MPI_COMM_WORLD, &size);
  /* 4096 blocks of 1..7 doubles at scrambled, non-overlapping displacements */
  enum { NB = 4096, SLOT = 8 };
  int *bl = malloc(NB * sizeof(int)), *dp = malloc(NB * sizeof(int));
  long total = 0;
  for (int i = 0; i < NB; ++i) {
    const int slot = (int)((i * 2654435761u) % NB); /* a permutation of the slots */
    bl[i] = 1 + (i * 7 + 3) % 7;
    dp[i] = slot * SLOT;
    total += bl[i];
  }
  MPI_Datatype ix;
  CHECK(MPI_Type_indexed(NB, bl, dp, MPI_DOUBLE, &ix) == MPI_SUCCESS);
  CHECK(MPI_Type_commit(&ix) == MPI_SUCCESS);
  int tsize;
  MPI_Aint lb, ext;
  CHECK(MPI_Type_size(ix, &tsize) == MPI_SUCCESS && tsize == total * 8);
  CHECK(MPI_Type_get_extent(ix, &lb, &ext) == MPI_SUCCESS);
  const long N = (long)NB * SLOT; /* doubles in the source array */
  double *h = malloc(N * 8), *want = malloc(total * 8), *hp = malloc(total * 8), *d, *dpk;
  cudaMalloc((void **)&d, N * 8);
  cudaMalloc((void **)&dpk, total * 8);
  for (long i = 0; i < N; ++i) h[i] = (double)i * 0.5 + rank;
  long k = 0; /* typemap order: block by block, in definition order */
  for (int i = 0; i < NB; ++i)
    for (int j = 0; j < bl[i]; ++j) want[k++] = h[dp[i] + j];
  cudaMemcpy(d, h, N * 8, cudaMemcpyHostToDevice);
  int pos = 0;
  CHECK(MPI_Pack(d, 1, ix, dpk, (int)(total * 8), &pos, MPI_COMM_WORLD) == MPI_SUCCESS && pos == total * 8);
  cudaMemcpy(hp, dpk, total * 8, cudaMemcpyDeviceToHost);
  CHECK(memcmp(hp, want, total * 8) == 0);
  cudaMemset(d, 0, N * 8); cudaDeviceSynchronize();
  pos = 0;
  CHECK(MPI_Unpack(dpk, (int)(total * 8), &pos, d, 1, ix, MPI_COMM_WORLD) == MPI_SUCCESS);
  double *back = malloc(N * 8);
  cudaMemcpy(back, d, N * 8, cudaMemcpyDeviceToHost);
  char *hit = calloc(N, 1);
  for (int i = 0; i < NB; ++i)
    for (int j = 0; j < bl[i]; ++j) hit[dp[i] + j] = 1;
  for (long i = 0; i < N; ++i) CHECK(back[i] == (hit[i] ? h[i] : 0.0));
  /* a struct {int; double[2]} resized to 32 bytes, 64 of them */
  int sbl[2] = {1, 2};
  MPI_Aint sd[2] = {0, 8};
  MPI_Datatype stt[2] = {MPI_INT, MPI_DOUBLE}, st, rs;
  CHECK(MPI_Type_create_struct(2, sbl, sd, stt, &st) == MPI_SUCCESS);
  CHECK(MPI_Type_create_resized(st, 0, 32, &rs) == MPI_SUCCESS && MPI_Type_commit(&rs) == MPI_SUCCESS);
  unsigned char *hs = malloc(64 * 32), *hsp = malloc(64 * 20), *ds, *dsp;
  for (int i = 0; i < 64 * 32; ++i) hs[i] = (unsigned char)(i * 13 + 1);
  cudaMalloc((void **)&ds, 64 * 32);
  cudaMalloc((void **)&dsp, 64 * 20);
  cudaMemcpy(ds, hs, 64 * 32, cudaMemcpyHostToDevice);
  pos = 0;
  CHECK(MPI_Pack(ds, 64, rs, dsp, 64 * 20, &pos, MPI_COMM_WORLD) == MPI_SUCCESS && pos == 64 * 20);
  cudaMemcpy(hsp, dsp, 64 * 20, cudaMemcpyDeviceToHost);
  for (int o = 0; o < 64; ++o) {
    CHECK(memcmp(hsp + o * 20, hs + o * 32, 4) == 0);
    CHECK(memcmp(hsp + o * 20 + 4, hs + o * 32 + 8, 16) == 0);
  }
  /* Send with the indexed type, receive as contiguous doubles */
  if (size >= 2) {
    MPI_Datatype flat;
    CHECK(MPI_Type_contiguous((int)total, MPI_DOUBLE, &flat) == MPI_SUCCESS && MPI_Type_commit(&flat) == MPI_SUCCESS);
    for (int m = -1; m <= 3; ++m) {
      CHECK(TEMPI_Set_method(m) == MPI_SUCCESS);
      if (rank == 0) {
        cudaMemcpy(d, h, N * 8, cudaMemcpyHostToDevice);
        CHECK(MPI_Send(d, 1, ix, 1, 70 + m, MPI_COMM_WORLD) == MPI_SUCCESS);
      } else if (rank == 1) {
        MPI_Status s;
        cudaMemset(dpk, 0, total * 8); cudaDeviceSynchronize();
        CHECK(MPI_Recv(dpk, 1, flat, 0, 70 + m, MPI_COMM_WORLD, &s) == MPI_SUCCESS);
        /* the irregular send lands by DIRECT (run-table pack straight into the
           contiguous receive buffer) when offered: explicitly and by the model */
        if (m == 3 || m == -1) CHECK(s.method == 3);
        cudaMemcpy(hp, dpk, total * 8, cudaMemcpyDeviceToHost);
        k = 0;
        for (int i = 0; i < NB; ++i)
          for (int j = 0; j < bl[i]; ++j) {
            CHECK(hp[k] == (double)(dp[i] + j) * 0.5 + 0);
            ++k;
          }
      }
    }
    MPI_Type_free(&flat);
  }
  MPI_Barrier(MPI_COMM_WORLD);
  MPI_Type_free(&ix);
  MPI_Type_free(&rs);
  MPI_Finalize();
  if (rank == 0) printf("OK\n");
  return 0;
}
