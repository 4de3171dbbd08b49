/* Beyond the reference: an unstructured-mesh exchange written purely
 * against MPI. Each rank of a ring sends an irregular MPI_Type_indexed
 * gather list of doubles (different per neighbour) and receives (a) into
 * contiguous ghost runs and (b) with the roles swapped, contiguous sends
 * scattered into irregular ghost slots -- one MPI_Neighbor_alltoallw each,
 * on device memory. Values checked on the host. Prints "OK".
 * argv[1]: "a" gather only, "b" scatter only, "ab" both in sequence;
 * argv[2]: iterations (default 1). Every iteration builds FRESH types from
 * lists that change with the iteration, so each one uploads and publishes
 * new device run tables and every call re-publishes its receive layout. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include <mpi.h>

#define CHECK(c) do { if (!(c)) { printf("FAIL rank %d line %d: %s\n", rank, __LINE__, #c); fflush(stdout); MPI_Abort(MPI_COMM_WORLD, 1); } } while (0)

enum { NB = 300, SLOTS = 1024 };

/* the gather list rank `from` uses for neighbour `to`: NB blocks of 1-3
 * doubles at distinct 4-double slots (a deterministic permutation) */
static int g_it = 0; /* current iteration: varies every list */
static void glist(int from, int to, int *bl, int *dp) {
  for (int i = 0; i < NB; ++i) {
    bl[i] = 1 + (i * 5 + from * 3 + to + g_it) % 3;
    /* distinct slots: i -> 389 i + c is a bijection mod SLOTS (389 odd) */
    dp[i] = (int)(((unsigned)i * 389u + (unsigned)(from * 7 + to + 13 * g_it)) % SLOTS) * 4;
  }
}

static int one_iteration(int rank, int size, MPI_Comm g, const char *mode);

static double val(int r, int i) { return r * 100000.0 + i * 0.5; }

int main(int argc, char **argv) {
  int rank = 0, size = 0;
  MPI_Init(&argc, &argv);
  MPI_Comm_rank(MPI_COMM_WORLD, &rank);
  MPI_Comm_size(MPI_COMM_WORLD, &size);
  const char *mode = argc > 1 ? argv[1] : "ab";
  const int iters = argc > 2 ? atoi(argv[2]) : 1;
  const int right = (rank + 1) % size, left = (rank + size - 1) % size;
  int nbrs[2] = {right, left}, srcs[2] = {left, right};
  MPI_Comm g;
  CHECK(MPI_Dist_graph_create_adjacent(MPI_COMM_WORLD, 2, srcs, MPI_UNWEIGHTED, 2, nbrs, MPI_UNWEIGHTED,
                                       MPI_INFO_NULL, 0, &g) == MPI_SUCCESS);
  for (g_it = 0; g_it < iters; ++g_it) CHECK(one_iteration(rank, size, g, mode) == 0);
  MPI_Barrier(MPI_COMM_WORLD);
  MPI_Finalize();
  if (rank == 0) printf("OK\n");
  return 0;
}

static int one_iteration(int rank, int size, MPI_Comm g, const char *mode) {
  const int right = (rank + 1) % size, left = (rank + size - 1) % size;
  int nbrs[2] = {right, left}, srcs[2] = {left, right};
  const int N = SLOTS * 4;
  int bl[2][NB], dp[2][NB], blin[2][NB], dpin[2][NB], n_out[2] = {0, 0}, n_in[2] = {0, 0};
  MPI_Datatype gather[2], ghost[2];
  for (int k = 0; k < 2; ++k) {
    glist(rank, nbrs[k], bl[k], dp[k]);  /* what I send to nbrs[k] */
    glist(srcs[k], rank, blin[k], dpin[k]); /* what srcs[k] sends me */
    for (int i = 0; i < NB; ++i) { n_out[k] += bl[k][i]; n_in[k] += blin[k][i]; }
    CHECK(MPI_Type_indexed(NB, bl[k], dp[k], MPI_DOUBLE, &gather[k]) == MPI_SUCCESS);
    CHECK(MPI_Type_commit(&gather[k]) == MPI_SUCCESS);
    CHECK(MPI_Type_contiguous(n_in[k], MPI_DOUBLE, &ghost[k]) == MPI_SUCCESS);
    CHECK(MPI_Type_commit(&ghost[k]) == MPI_SUCCESS);
  }
  double *h = malloc(N * sizeof(double)), *d_field, *d_ghost;
  for (int i = 0; i < N; ++i) h[i] = val(rank, i);
  cudaMalloc((void **)&d_field, N * sizeof(double));
  cudaMalloc((void **)&d_ghost, (n_in[0] + n_in[1]) * sizeof(double));
  cudaMemcpy(d_field, h, N * sizeof(double), cudaMemcpyHostToDevice);
  /* (a) irregular sends, contiguous ghost runs */
  int ones[2] = {1, 1};
  MPI_Aint sd[2] = {0, 0}, rd[2] = {0, (MPI_Aint)(n_in[0] * sizeof(double))};
  if (strchr(mode, 'a')) {
    CHECK(MPI_Neighbor_alltoallw(d_field, ones, sd, gather, d_ghost, ones, rd, ghost, g) == MPI_SUCCESS);
    double *hg = malloc((n_in[0] + n_in[1]) * sizeof(double));
    cudaMemcpy(hg, d_ghost, (n_in[0] + n_in[1]) * sizeof(double), cudaMemcpyDeviceToHost);
    for (int k = 0, at = 0; k < 2; ++k)
      for (int i = 0; i < NB; ++i)
        for (int j = 0; j < blin[k][i]; ++j) CHECK(hg[at++] == val(srcs[k], dpin[k][i] + j));
    free(hg);
  }
  /* (b) contiguous sends scattered into irregular ghost slots: I receive
     through the lists my neighbours used, into a fresh field */
  MPI_Datatype flat[2], scatter[2];
  for (int k = 0; k < 2; ++k) {
    CHECK(MPI_Type_contiguous(n_out[k], MPI_DOUBLE, &flat[k]) == MPI_SUCCESS && MPI_Type_commit(&flat[k]) == MPI_SUCCESS);
    CHECK(MPI_Type_indexed(NB, blin[k], dpin[k], MPI_DOUBLE, &scatter[k]) == MPI_SUCCESS);
    CHECK(MPI_Type_commit(&scatter[k]) == MPI_SUCCESS);
  }
  double *d_src, *d_out;
  double *hs = malloc((n_out[0] + n_out[1]) * sizeof(double));
  for (int i = 0; i < n_out[0] + n_out[1]; ++i) hs[i] = val(rank, i) + 0.25;
  cudaMalloc((void **)&d_src, (n_out[0] + n_out[1]) * sizeof(double));
  cudaMalloc((void **)&d_out, 2 * N * sizeof(double));
  cudaMemcpy(d_src, hs, (n_out[0] + n_out[1]) * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemset(d_out, 0, 2 * N * sizeof(double)); cudaDeviceSynchronize();
  MPI_Aint sd2[2] = {0, (MPI_Aint)(n_out[0] * sizeof(double))}, rd2[2] = {0, (MPI_Aint)(N * sizeof(double))};
  if (!strchr(mode, 'b')) goto done;
  CHECK(MPI_Neighbor_alltoallw(d_src, ones, sd2, flat, d_out, ones, rd2, scatter, g) == MPI_SUCCESS);
  double *ho = malloc(2 * N * sizeof(double));
  cudaMemcpy(ho, d_out, 2 * N * sizeof(double), cudaMemcpyDeviceToHost);
  for (int k = 0; k < 2; ++k) {
    /* srcs[k] sent me its flat run for me: its k-th out edge is to me when
       its nbrs[k'] == rank; k' = k because right/left mirror */
    int at = 0;
    int from_n0 = 0; /* the sender's first-edge length when I am its second neighbour */
    int bl0[NB], dp0[NB];
    glist(srcs[k], (srcs[k] + 1) % size, bl0, dp0);
    for (int i = 0; i < NB; ++i) from_n0 += bl0[i];
    const int base = (k == 0) ? 0 : from_n0; /* left sends me its edge 0 (to its right); right sends edge 1 */
    for (int i = 0; i < NB; ++i)
      for (int j = 0; j < blin[k][i]; ++j) {
        if (ho[k * N + dpin[k][i] + j] != val(srcs[k], base + at) + 0.25)
          printf("rank %d k %d i %d j %d got %.2f want %.2f (base %d at %d)\n", rank, k, i, j,
                 ho[k * N + dpin[k][i] + j], val(srcs[k], base + at) + 0.25, base, at);
        CHECK(ho[k * N + dpin[k][i] + j] == val(srcs[k], base + at) + 0.25);
        ++at;
      }
  }
  free(ho);
done:
  for (int k = 0; k < 2; ++k) {
    MPI_Type_free(&gather[k]);
    MPI_Type_free(&ghost[k]);
    MPI_Type_free(&flat[k]);
    MPI_Type_free(&scatter[k]);
  }
  cudaFree(d_field);
  cudaFree(d_ghost);
  cudaFree(d_src);
  cudaFree(d_out);
  free(h);
  free(hs);
  return 0;
}
