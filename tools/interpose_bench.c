/* interpose_bench -- the paper's MPI_Pack / MPI_Send comparison (PAPER.md:
 * 704-760): the same portable MPI program timed on the system MPI alone and
 * with TEMPI interposed (LD_PRELOAD=libtempi_interpose.so). Device buffers,
 * cold L2 is NOT forced (the system-MPI leg is latency bound), best of R
 * calls after one warm-up. Prints one JSON object per measurement:
 *   {"what": ..., "bytes": B, "us": T}
 * usage: interpose_bench [max_seconds_per_case]
 * rank 0 alone runs the pack cases; with 2 ranks, rank 0 -> 1 Send/Recv of
 * the cfg1 object (one-way time = half a ping-pong). */
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime.h>
#include <mpi.h>

static double best_of(double budget, int (*op)(void *), void *arg) {
  double best = 1e30, spent = 0;
  op(arg); /* warm-up (the interposer's commit-time plan and scratch) */
  for (int r = 0; r < 5 && spent < budget; ++r) {
    cudaDeviceSynchronize();
    const double t0 = MPI_Wtime();
    if (op(arg) != MPI_SUCCESS) return -1;
    cudaDeviceSynchronize();
    const double t = MPI_Wtime() - t0;
    spent += t;
    if (t < best) best = t;
  }
  return best;
}

typedef struct {
  MPI_Datatype t;
  void *obj, *packed;
  int bytes;
} Case;

static int do_pack(void *a) {
  Case *c = a;
  int pos = 0;
  return MPI_Pack(c->obj, 1, c->t, c->packed, c->bytes, &pos, MPI_COMM_WORLD);
}

static int do_unpack(void *a) {
  Case *c = a;
  int pos = 0;
  return MPI_Unpack(c->packed, c->bytes, &pos, c->obj, 1, c->t, MPI_COMM_WORLD);
}

int main(int argc, char **argv) {
  MPI_Init(&argc, &argv);
  int rank = 0, size = 1;
  MPI_Comm_rank(MPI_COMM_WORLD, &rank);
  MPI_Comm_size(MPI_COMM_WORLD, &size);
  const double budget = argc > 1 ? atof(argv[1]) : 3.0;
  /* cfg1: vector(131072,1,64,DOUBLE); cfg2: 1 MiB subarray of a 1024^3 B
   * allocation with E0 = 64 and 512 (smaller E0 on the system MPI's
   * per-run copies would take minutes) */
  unsigned char *big = NULL, *packed = NULL;
  cudaMalloc((void **)&big, (size_t)1 << 30);
  cudaMalloc((void **)&packed, 1 << 20);
  cudaMemset(big, 7, (size_t)1 << 30);
  MPI_Datatype cfg1;
  MPI_Type_vector(131072, 1, 64, MPI_DOUBLE, &cfg1);
  MPI_Type_commit(&cfg1);
  if (rank == 0) {
    struct { const char *name; MPI_Datatype t; } cs[3];
    cs[0].name = "cfg1 vector(131072,1,64,DOUBLE)";
    cs[0].t = cfg1;
    const int e0s[2] = {64, 512};
    char names[2][64];
    for (int i = 0; i < 2; ++i) {
      const int e0 = e0s[i], e2 = e0 == 64 ? 128 : 64, e1 = (1 << 20) / (e0 * e2);
      const int sizes[3] = {1024, 1024, 1024}, subs[3] = {e2, e1, e0}, starts[3] = {0, 0, 0};
      MPI_Type_create_subarray(3, sizes, subs, starts, MPI_ORDER_C, MPI_BYTE, &cs[i + 1].t);
      MPI_Type_commit(&cs[i + 1].t);
      snprintf(names[i], sizeof names[i], "cfg2 subarray E0=%d", e0);
      cs[i + 1].name = names[i];
    }
    for (int i = 0; i < 3; ++i) {
      Case c = {cs[i].t, big, packed, 1 << 20};
      const double tp = best_of(budget, do_pack, &c), tu = best_of(budget, do_unpack, &c);
      printf("{\"what\": \"MPI_Pack %s\", \"bytes\": %d, \"us\": %.2f}\n", cs[i].name, c.bytes, tp * 1e6);
      printf("{\"what\": \"MPI_Unpack %s\", \"bytes\": %d, \"us\": %.2f}\n", cs[i].name, c.bytes, tu * 1e6);
      fflush(stdout);
    }
  }
  if (size >= 2 && rank < 2) {
    double best = 1e30;
    for (int r = 0; r < 4; ++r) { /* r = 0 warms up */
      MPI_Barrier(MPI_COMM_WORLD);
      const double t0 = MPI_Wtime();
      if (rank == 0) {
        MPI_Send(big, 1, cfg1, 1, 1, MPI_COMM_WORLD);
        MPI_Recv(big, 1, cfg1, 1, 2, MPI_COMM_WORLD, MPI_STATUS_IGNORE);
      } else {
        MPI_Recv(big, 1, cfg1, 0, 1, MPI_COMM_WORLD, MPI_STATUS_IGNORE);
        MPI_Send(big, 1, cfg1, 0, 2, MPI_COMM_WORLD);
      }
      const double t = (MPI_Wtime() - t0) / 2;
      if (r && t < best) best = t;
    }
    if (rank == 0)
      printf("{\"what\": \"MPI_Send/Recv cfg1 one-way\", \"bytes\": %d, \"us\": %.2f}\n", 1 << 20, best * 1e6);
  }
  MPI_Type_free(&cfg1);
  cudaFree(big);
  cudaFree(packed);
  MPI_Finalize();
  return 0;
}
