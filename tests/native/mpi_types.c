/* Datatype construction and queries through the MPI surface (no GPU needed):
 * the cfg1 vector, a C-order and a Fortran-order 3D subarray of the same
 * cuboid (must canonicalise identically), hvector-of-vector, sizes,
 * extents, Pack_size, error codes. Prints "OK" on success. */
#include <stdio.h>
#include <mpi.h>
#include "stridepack_b200.h"

#define CHECK(c) do { if (!(c)) { printf("FAIL line %d: %s\n", __LINE__, #c); return 1; } } while (0)

int main(int argc, char **argv) {
  CHECK(MPI_Init(&argc, &argv) == MPI_SUCCESS);
  int rank, size;
  MPI_Comm_rank(MPI_COMM_WORLD, &rank);
  MPI_Comm_size(MPI_COMM_WORLD, &size);
  MPI_Datatype v, sc, sf, hv, row, x;
  CHECK(MPI_Type_vector(131072, 1, 64, MPI_DOUBLE, &v) == MPI_SUCCESS);
  CHECK(MPI_Type_commit(&v) == MPI_SUCCESS);
  int s; MPI_Aint lb, ext;
  CHECK(MPI_Type_size(v, &s) == MPI_SUCCESS && s == 1048576);
  CHECK(MPI_Type_get_extent(v, &lb, &ext) == MPI_SUCCESS && lb == 0 && ext == 67108360);
  /* C order: slowest dimension first */
  int sizes_c[3] = {1024, 512, 512}, sub_c[3] = {47, 13, 400}, st_c[3] = {0, 0, 0};
  CHECK(MPI_Type_create_subarray(3, sizes_c, sub_c, st_c, MPI_ORDER_C, MPI_BYTE, &sc) == MPI_SUCCESS);
  int sizes_f[3] = {512, 512, 1024}, sub_f[3] = {400, 13, 47};
  CHECK(MPI_Type_create_subarray(3, sizes_f, sub_f, st_c, MPI_ORDER_FORTRAN, MPI_BYTE, &sf) == MPI_SUCCESS);
  CHECK(MPI_Type_contiguous(400, MPI_BYTE, &row) == MPI_SUCCESS);
  MPI_Datatype plane;
  CHECK(MPI_Type_create_hvector(13, 1, 512, row, &plane) == MPI_SUCCESS);
  CHECK(MPI_Type_create_hvector(47, 1, 262144, plane, &hv) == MPI_SUCCESS);
  MPI_Datatype all[3] = {sc, sf, hv};
  for (int i = 0; i < 3; ++i) {
    CHECK(MPI_Type_commit(&all[i]) == MPI_SUCCESS);
    CHECK(MPI_Type_size(all[i], &s) == MPI_SUCCESS && s == 400 * 13 * 47);
  }
  CHECK(MPI_Pack_size(3, sc, MPI_COMM_WORLD, &s) == MPI_SUCCESS && s == 3 * 244400);
  /* beyond the reference: indexed / hindexed / indexed_block / struct / resized */
  MPI_Datatype ix, hx, ib, st, rs, rv;
  int bl[3] = {2, 3, 1}, dp[3] = {1, 5, 10};
  CHECK(MPI_Type_indexed(3, bl, dp, MPI_DOUBLE, &ix) == MPI_SUCCESS && MPI_Type_commit(&ix) == MPI_SUCCESS);
  CHECK(MPI_Type_size(ix, &s) == MPI_SUCCESS && s == 48);
  CHECK(MPI_Type_get_extent(ix, &lb, &ext) == MPI_SUCCESS && lb == 8 && ext == 80);
  MPI_Aint hd[2] = {64, 67};
  int hbl[2] = {3, 5};
  CHECK(MPI_Type_create_hindexed(2, hbl, hd, MPI_BYTE, &hx) == MPI_SUCCESS && MPI_Type_commit(&hx) == MPI_SUCCESS);
  CHECK(MPI_Type_get_extent(hx, &lb, &ext) == MPI_SUCCESS && lb == 64 && ext == 8);
  int ibd[4] = {0, 16, 32, 48};
  CHECK(MPI_Type_create_indexed_block(4, 4, ibd, MPI_FLOAT, &ib) == MPI_SUCCESS && MPI_Type_commit(&ib) == MPI_SUCCESS);
  CHECK(MPI_Type_size(ib, &s) == MPI_SUCCESS && s == 64);
  CHECK(MPI_Type_get_extent(ib, &lb, &ext) == MPI_SUCCESS && lb == 0 && ext == 208);
  int sbl[2] = {1, 2};
  MPI_Aint sd[2] = {0, 8};
  MPI_Datatype stt[2] = {MPI_INT, MPI_DOUBLE};
  CHECK(MPI_Type_create_struct(2, sbl, sd, stt, &st) == MPI_SUCCESS && MPI_Type_commit(&st) == MPI_SUCCESS);
  CHECK(MPI_Type_size(st, &s) == MPI_SUCCESS && s == 20);
  CHECK(MPI_Type_get_extent(st, &lb, &ext) == MPI_SUCCESS && lb == 0 && ext == 24);
  CHECK(MPI_Type_create_resized(st, 0, 32, &rs) == MPI_SUCCESS);
  CHECK(MPI_Type_contiguous(4, rs, &rv) == MPI_SUCCESS && MPI_Type_commit(&rv) == MPI_SUCCESS);
  CHECK(MPI_Type_get_extent(rv, &lb, &ext) == MPI_SUCCESS && lb == 0 && ext == 128);
  MPI_Aint neg[1] = {-8};
  int one[1] = {1};
  CHECK(MPI_Type_create_hindexed(1, one, neg, MPI_BYTE, &x) == MPI_ERR_ARG);
  /* errors */
  int bad_sizes[1] = {8}, bad_sub[1] = {4}, bad_st[1] = {6};
  CHECK(MPI_Type_create_subarray(1, bad_sizes, bad_sub, bad_st, MPI_ORDER_C, MPI_BYTE, &x) == MPI_ERR_ARG);
  CHECK(MPI_Type_size(12345, &s) == MPI_ERR_TYPE);
  CHECK(MPI_Type_free(&sc) == MPI_SUCCESS && sc == MPI_DATATYPE_NULL);
  /* topology bookkeeping */
  MPI_Comm g;
  int srcs[2] = {(rank + size - 1) % size, (rank + 1) % size};
  CHECK(MPI_Dist_graph_create_adjacent(MPI_COMM_WORLD, 2, srcs, MPI_UNWEIGHTED, 2, srcs, MPI_UNWEIGHTED,
                                       MPI_INFO_NULL, 0, &g) == MPI_SUCCESS);
  int indeg, outdeg, w;
  CHECK(MPI_Dist_graph_neighbors_count(g, &indeg, &outdeg, &w) == MPI_SUCCESS && indeg == 2 && outdeg == 2);
  CHECK(MPI_Barrier(MPI_COMM_WORLD) == MPI_SUCCESS);
  CHECK(MPI_Finalize() == MPI_SUCCESS);
  if (rank == 0) printf("OK\n");
  return 0;
}
