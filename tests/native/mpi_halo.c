/* The paper's 3D halo exchange written against the MPI surface
 * (PAPER.md:1029-1041): 26 subarray types per rank, MPI_Pack of every
 * region into one device buffer, MPI_Neighbor_alltoallv over a distributed
 * graph of the 26 neighbours, MPI_Unpack into the ghost shell. Verified
 * with the reference's fill_cell pattern (sp_halo_fill / sp_halo_verify).
 * With MODE = 1 the exchange is ONE MPI_Neighbor_alltoallw call on the
 * padded allocation itself: send types = the interior regions, receive
 * types = the ghost regions, byte displacements 0 (ghost writes, no packed
 * buffers). MODE = 2 is the same exchange as an MPI-4 persistent
 * collective: MPI_Neighbor_alltoallw_init once, then MPI_Start + MPI_Wait
 * per iteration (the ghosts reset before the last one). MODE = 3 is mode 0
 * with the MPI_Neighbor_alltoallv of the packed segments made persistent
 * (MPI_Neighbor_alltoallv_init once, MPI_Start + MPI_Wait per iteration).
 * usage: mpi_halo RX RY RZ N RADIUS ELEM ITERS [MODE]  (RX*RY*RZ == ranks)
 * prints per-phase wall times of the last iteration and "OK". */
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime.h>
#include <mpi.h>
#include "stridepack_b200.h"

/* MPI-4 (modes 2, 3): weak, so the program still links against an MPI-3 library */
#pragma weak MPI_Neighbor_alltoallw_init
#pragma weak MPI_Neighbor_alltoallv_init

#define CHECK(c) do { if (!(c)) { printf("FAIL rank %d line %d: %s\n", rank, __LINE__, #c); MPI_Abort(MPI_COMM_WORLD, 1); } } while (0)

static int rank_of(const int R[3], const int c[3]) {
  int w[3];
  for (int a = 0; a < 3; ++a) w[a] = ((c[a] % R[a]) + R[a]) % R[a];
  return (w[2] * R[1] + w[1]) * R[0] + w[0];
}

int main(int argc, char **argv) {
  int rank = 0, size = 0;
  MPI_Init(&argc, &argv);
  MPI_Comm_rank(MPI_COMM_WORLD, &rank);
  MPI_Comm_size(MPI_COMM_WORLD, &size);
  const int R[3] = {atoi(argv[1]), atoi(argv[2]), atoi(argv[3])};
  const int n = atoi(argv[4]), r = atoi(argv[5]), e = atoi(argv[6]);
  int iters = atoi(argv[7]);
  const int mode = argc > 8 ? atoi(argv[8]) : 0;
  CHECK(R[0] * R[1] * R[2] == size);
  const int p = n + 2 * r;
  const long alloc_bytes = (long)p * p * p * e;
  const int me[3] = {rank % R[0], rank / R[0] % R[1], rank / (R[0] * R[1])};
  MPI_Datatype send_t[26], recv_t[26];
  int dir[26][3], k = 0, sizes[26];
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (!dx && !dy && !dz) continue;
        const int d[3] = {dx, dy, dz};
        int ssub[3], sst[3], rsub[3], rst[3], full[3] = {p, p, p * e};
        for (int a = 0; a < 3; ++a) { /* C order: index 0 = z, 2 = x (bytes) */
          const int i = 2 - a, m = a == 0 ? e : 1;
          const int sb = d[a] < 0 ? r : d[a] > 0 ? n : r, sl = d[a] ? r : n;
          const int rb = d[a] < 0 ? 0 : d[a] > 0 ? r + n : r;
          ssub[i] = sl * m; sst[i] = sb * m; rsub[i] = sl * m; rst[i] = rb * m;
        }
        CHECK(MPI_Type_create_subarray(3, full, ssub, sst, MPI_ORDER_C, MPI_BYTE, &send_t[k]) == MPI_SUCCESS);
        CHECK(MPI_Type_create_subarray(3, full, rsub, rst, MPI_ORDER_C, MPI_BYTE, &recv_t[k]) == MPI_SUCCESS);
        MPI_Type_commit(&send_t[k]);
        MPI_Type_commit(&recv_t[k]);
        MPI_Type_size(send_t[k], &sizes[k]);
        dir[k][0] = dx; dir[k][1] = dy; dir[k][2] = dz;
        ++k;
      }
  int off[27], srcs[26], dsts[26];
  off[0] = 0;
  for (int i = 0; i < 26; ++i) {
    off[i + 1] = off[i] + sizes[i];
    int plus[3], minus[3];
    for (int a = 0; a < 3; ++a) { plus[a] = me[a] + dir[i][a]; minus[a] = me[a] - dir[i][a]; }
    dsts[i] = rank_of(R, plus);   /* my region i goes to the rank at +d_i */
    srcs[i] = rank_of(R, minus);  /* edge i brings that rank's region i   */
  }
  MPI_Comm g;
  CHECK(MPI_Dist_graph_create_adjacent(MPI_COMM_WORLD, 26, srcs, MPI_UNWEIGHTED, 26, dsts, MPI_UNWEIGHTED,
                                       MPI_INFO_NULL, 0, &g) == MPI_SUCCESS);
  unsigned char *alloc, *sbuf, *rbuf;
  CHECK(cudaMalloc((void **)&alloc, alloc_bytes) == cudaSuccess);
  CHECK(cudaMalloc((void **)&sbuf, off[26]) == cudaSuccess);
  CHECK(cudaMalloc((void **)&rbuf, off[26]) == cudaSuccess);
  sp_halo_config cfg = {{R[0], R[1], R[2]}, {n, n, n}, r, e};
  CHECK(sp_halo_fill(&cfg, rank, alloc, NULL) == SP_OK);
  cudaDeviceSynchronize();
  double tp = 0, tx = 0, tu = 0;
  if ((mode == 2 && !MPI_Neighbor_alltoallw_init) || (mode == 3 && !MPI_Neighbor_alltoallv_init)) {
    if (rank == 0) printf("MPI-4 persistent collectives: not in this MPI library\nOK\n");
    MPI_Finalize();
    return 0;
  }
  if (mode == 2) {
    int ones[26];
    MPI_Aint zeros[26];
    MPI_Datatype rtypes[26];
    for (int i = 0; i < 26; ++i) {
      ones[i] = 1;
      zeros[i] = 0;
      rtypes[i] = recv_t[25 - i];
    }
    MPI_Request req;
    CHECK(MPI_Neighbor_alltoallw_init(alloc, ones, zeros, send_t, alloc, ones, zeros, rtypes, g, MPI_INFO_NULL, &req) ==
          MPI_SUCCESS);
    for (int it = 0; it < iters; ++it) {
      if (it + 1 == iters) CHECK(sp_halo_fill(&cfg, rank, alloc, NULL) == SP_OK && cudaDeviceSynchronize() == cudaSuccess);
      MPI_Barrier(MPI_COMM_WORLD);
      const double t0 = MPI_Wtime();
      CHECK(MPI_Start(&req) == MPI_SUCCESS);
      CHECK(MPI_Wait(&req, MPI_STATUS_IGNORE) == MPI_SUCCESS);
      tx = MPI_Wtime() - t0;
      CHECK(req != MPI_REQUEST_NULL); /* inactive, reusable */
    }
    CHECK(MPI_Request_free(&req) == MPI_SUCCESS && req == MPI_REQUEST_NULL);
    iters = 0;
  }
  if (mode == 1) {
    /* edge i brings the neighbour's region i into my ghost region 25-i */
    int ones[26];
    MPI_Aint zeros[26];
    MPI_Datatype rtypes[26];
    for (int i = 0; i < 26; ++i) {
      ones[i] = 1;
      zeros[i] = 0;
      rtypes[i] = recv_t[25 - i];
    }
    for (int it = 0; it < iters; ++it) {
      if (it + 1 == iters) CHECK(sp_halo_fill(&cfg, rank, alloc, NULL) == SP_OK && cudaDeviceSynchronize() == cudaSuccess);
      MPI_Barrier(MPI_COMM_WORLD);
      const double t0 = MPI_Wtime();
      CHECK(MPI_Neighbor_alltoallw(alloc, ones, zeros, send_t, alloc, ones, zeros, rtypes, g) == MPI_SUCCESS);
      tx = MPI_Wtime() - t0;
    }
    iters = 0;
  }
  MPI_Request vreq = MPI_REQUEST_NULL;
  if (mode == 3)
    CHECK(MPI_Neighbor_alltoallv_init(sbuf, sizes, off, MPI_PACKED, rbuf, sizes, off, MPI_PACKED, g, MPI_INFO_NULL,
                                      &vreq) == MPI_SUCCESS);
  for (int it = 0; it < iters; ++it) {
    MPI_Barrier(MPI_COMM_WORLD);
    const double t0 = MPI_Wtime();
    int pos = 0;
    for (int i = 0; i < 26; ++i) CHECK(MPI_Pack(alloc, 1, send_t[i], sbuf, off[26], &pos, MPI_COMM_WORLD) == MPI_SUCCESS);
    const double t1 = MPI_Wtime();
    if (mode == 3) {
      CHECK(MPI_Start(&vreq) == MPI_SUCCESS && MPI_Wait(&vreq, MPI_STATUS_IGNORE) == MPI_SUCCESS);
    } else {
      CHECK(MPI_Neighbor_alltoallv(sbuf, sizes, off, MPI_PACKED, rbuf, sizes, off, MPI_PACKED, g) == MPI_SUCCESS);
    }
    const double t2 = MPI_Wtime();
    pos = 0;
    for (int i = 0; i < 26; ++i) {
      /* edge i carries the neighbour's region i: my ghost on side -d_i */
      pos = off[i];
      CHECK(MPI_Unpack(rbuf, off[26], &pos, alloc, 1, recv_t[25 - i], MPI_COMM_WORLD) == MPI_SUCCESS);
    }
    const double t3 = MPI_Wtime();
    tp = t1 - t0; tx = t2 - t1; tu = t3 - t2;
  }
  if (vreq != MPI_REQUEST_NULL) CHECK(MPI_Request_free(&vreq) == MPI_SUCCESS);
  int64_t bad = -1;
  CHECK(sp_halo_verify(&cfg, rank, alloc, NULL, &bad) == SP_OK);
  CHECK(bad == 0);
  MPI_Barrier(MPI_COMM_WORLD);
  if (rank == 0) printf("pack %.1f us alltoallv %.1f us unpack %.1f us bytes/rank %d\nOK\n", tp * 1e6, tx * 1e6, tu * 1e6, off[26]);
  MPI_Finalize();
  return 0;
}
