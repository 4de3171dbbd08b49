/* MPI_Alltoallv / MPI_Alltoallw with derived datatypes on device memory
 * (MPI-3.1 5.8), portable: the same source runs on libtempi_b200.so and on
 * a system MPI with the interposer in front. Values are doubles
 * v = rank * 1e6 + index, so every received element names its sender and
 * source position; checked on the host.
 *  1. alltoallv, strided send (vector(B,1,2)) -> contiguous receive;
 *  2. alltoallv, contiguous send -> strided receive (every other slot; the
 *     slots between keep their sentinel);
 *  3. alltoallw, per-peer types (strided to even peers, contiguous to odd
 *     ones), byte displacements.
 * Prints "OK". */
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime.h>
#include <mpi.h>

static int rank = 0, size = 1;
#define CHECK(c) do { if (!(c)) { printf("FAIL rank %d line %d: %s\n", rank, __LINE__, #c); fflush(stdout); MPI_Abort(MPI_COMM_WORLD, 1); } } while (0)
#define B 4096

static double *dev_fill(long n, double base, int sentinel) {
  double *h = malloc(sizeof(double) * n), *d = NULL;
  for (long k = 0; k < n; ++k) h[k] = sentinel ? -1.0 : base + (double)k;
  CHECK(cudaMalloc((void **)&d, sizeof(double) * n) == cudaSuccess);
  cudaMemcpy(d, h, sizeof(double) * n, cudaMemcpyHostToDevice);
  free(h);
  return d;
}

static double *host_copy(const double *d, long n) {
  double *h = malloc(sizeof(double) * n);
  cudaMemcpy(h, d, sizeof(double) * n, cudaMemcpyDeviceToHost);
  return h;
}

int main(int argc, char **argv) {
  MPI_Init(&argc, &argv);
  MPI_Comm_rank(MPI_COMM_WORLD, &rank);
  MPI_Comm_size(MPI_COMM_WORLD, &size);
  const int n = size;
  MPI_Datatype strided, dense;
  CHECK(MPI_Type_vector(B, 1, 2, MPI_DOUBLE, &strided) == MPI_SUCCESS);
  CHECK(MPI_Type_contiguous(B, MPI_DOUBLE, &dense) == MPI_SUCCESS);
  CHECK(MPI_Type_commit(&strided) == MPI_SUCCESS && MPI_Type_commit(&dense) == MPI_SUCCESS);
  const long ext = 2 * B - 1; /* strided extent in doubles */
  int *ones = malloc(sizeof(int) * n), *disp = malloc(sizeof(int) * n), *sdb = malloc(sizeof(int) * n),
      *rdb = malloc(sizeof(int) * n);
  MPI_Datatype *st = malloc(sizeof(MPI_Datatype) * n), *rt = malloc(sizeof(MPI_Datatype) * n);
  for (int i = 0; i < n; ++i) {
    ones[i] = 1;
    disp[i] = i;
  }
  const double me = rank * 1e6;

  /* 1. strided -> contiguous */
  {
    double *s = dev_fill(n * ext, me, 0), *r = dev_fill((long)n * B, 0, 1);
    CHECK(MPI_Alltoallv(s, ones, disp, strided, r, ones, disp, dense, MPI_COMM_WORLD) == MPI_SUCCESS);
    double *h = host_copy(r, (long)n * B);
    for (int j = 0; j < n; ++j)
      for (int b = 0; b < B; ++b) CHECK(h[(long)j * B + b] == j * 1e6 + rank * ext + 2.0 * b);
    free(h);
    cudaFree(s);
    cudaFree(r);
  }
  /* 2. contiguous -> strided (sentinels between the received slots) */
  {
    double *s = dev_fill((long)n * B, me, 0), *r = dev_fill(n * ext, 0, 1);
    CHECK(MPI_Alltoallv(s, ones, disp, dense, r, ones, disp, strided, MPI_COMM_WORLD) == MPI_SUCCESS);
    double *h = host_copy(r, n * ext);
    for (int j = 0; j < n; ++j)
      for (long k = 0; k < ext; ++k)
        CHECK(h[j * ext + k] == (k % 2 ? -1.0 : j * 1e6 + (double)rank * B + k / 2));
    free(h);
    cudaFree(s);
    cudaFree(r);
  }
  /* 3. alltoallw: strided to even peers, contiguous to odd ones; the send
   * blocks sit 2B doubles apart, received blocks B doubles apart */
  {
    double *s = dev_fill((long)n * 2 * B, me, 0), *r = dev_fill((long)n * B, 0, 1);
    for (int i = 0; i < n; ++i) {
      st[i] = i % 2 ? dense : strided;
      rt[i] = dense;
      sdb[i] = (int)(sizeof(double) * 2 * B * i);
      rdb[i] = (int)(sizeof(double) * B * i);
    }
    CHECK(MPI_Alltoallw(s, ones, sdb, st, r, ones, rdb, rt, MPI_COMM_WORLD) == MPI_SUCCESS);
    double *h = host_copy(r, (long)n * B);
    for (int j = 0; j < n; ++j) /* j sent me its block `rank`, strided iff rank is even */
      for (int b = 0; b < B; ++b)
        CHECK(h[(long)j * B + b] == j * 1e6 + 2.0 * B * rank + (rank % 2 ? b : 2.0 * b));
    free(h);
    cudaFree(s);
    cudaFree(r);
  }
  MPI_Barrier(MPI_COMM_WORLD);
  MPI_Type_free(&strided);
  MPI_Type_free(&dense);
  free(ones);
  free(disp);
  free(sdb);
  free(rdb);
  free(st);
  free(rt);
  MPI_Finalize();
  if (rank == 0) printf("OK\n");
  return 0;
}
