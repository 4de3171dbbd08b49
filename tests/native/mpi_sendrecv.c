/* MPI_Send/MPI_Recv of a 3D subarray between two ranks, device buffers,
 * every transfer method (TEMPI_Set_method) plus the model's choice, and
 * MPI_Pack/MPI_Unpack round trips; bytes checked on the host against the
 * MPI definition (C order: last dimension fastest). Prints "OK". */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include <mpi.h>

#define CHECK(c) do { if (!(c)) { printf("FAIL rank %d line %d: %s\n", rank, __LINE__, #c); MPI_Abort(MPI_COMM_WORLD, 1); } } while (0)

static unsigned char pat(long i, int salt) { return (unsigned char)((i * 131 + salt * 17 + 7) >> 1); }

int main(int argc, char **argv) {
  int rank = 0, size = 0;
  MPI_Init(&argc, &argv);
  MPI_Comm_rank(MPI_COMM_WORLD, &rank);
  MPI_Comm_size(MPI_COMM_WORLD, &size);
  /* a 3D subarray of a (Z,Y,X) byte array, x fastest: E0=64-byte rows */
  const int Z = 16, Y = 48, X = 256, sz[3] = {Z, Y, X}, sub[3] = {8, 32, 64}, st[3] = {3, 5, 64};
  MPI_Datatype t;
  CHECK(MPI_Type_create_subarray(3, sz, sub, st, MPI_ORDER_C, MPI_BYTE, &t) == MPI_SUCCESS);
  CHECK(MPI_Type_commit(&t) == MPI_SUCCESS);
  const long N = (long)Z * Y * X, P = 8L * 32 * 64;
  unsigned char *h = malloc(N), *hp = malloc(P), *want = malloc(P), *d, *dp;
  cudaMalloc((void **)&d, N);
  cudaMalloc((void **)&dp, P);
  /* expected packed bytes of the source pattern */
  long k = 0;
  for (int z = 0; z < 8; ++z)
    for (int y = 0; y < 32; ++y)
      for (int x = 0; x < 64; ++x) want[k++] = pat(((long)(z + 3) * Y + (y + 5)) * X + (x + 64), 0);
  /* MPI_Pack / MPI_Unpack on device memory */
  for (long i = 0; i < N; ++i) h[i] = pat(i, 0);
  cudaMemcpy(d, h, N, cudaMemcpyHostToDevice);
  int pos = 0;
  CHECK(MPI_Pack(d, 1, t, dp, (int)P, &pos, MPI_COMM_WORLD) == MPI_SUCCESS && pos == P);
  cudaMemcpy(hp, dp, P, cudaMemcpyDeviceToHost);
  CHECK(memcmp(hp, want, P) == 0);
  cudaMemset(d, 0xCD, N); cudaDeviceSynchronize();
  pos = 0;
  CHECK(MPI_Unpack(dp, (int)P, &pos, d, 1, t, MPI_COMM_WORLD) == MPI_SUCCESS && pos == P);
  cudaMemcpy(h, d, N, cudaMemcpyDeviceToHost);
  for (long i = 0; i < N; ++i) {
    const int z = (int)(i / (Y * X)), y = (int)(i / X % Y), x = (int)(i % X);
    const int in = z >= 3 && z < 11 && y >= 5 && y < 37 && x >= 64 && x < 128;
    CHECK(h[i] == (in ? pat(i, 0) : 0xCD));
  }
  /* Send/Recv, every method, ring of two */
  if (size >= 2) {
    for (int m = -1; m <= 3; ++m) {
      CHECK(TEMPI_Set_method(m) == MPI_SUCCESS);
      if (rank == 0) {
        for (long i = 0; i < N; ++i) h[i] = pat(i, m + 2);
        cudaMemcpy(d, h, N, cudaMemcpyHostToDevice);
        CHECK(MPI_Send(d, 1, t, 1, 40 + m, MPI_COMM_WORLD) == MPI_SUCCESS);
      } else if (rank == 1) {
        MPI_Status s;
        cudaMemset(d, 0x5A, N); cudaDeviceSynchronize();
        CHECK(MPI_Recv(d, 1, t, MPI_ANY_SOURCE, 40 + m, MPI_COMM_WORLD, &s) == MPI_SUCCESS);
        CHECK(s.MPI_SOURCE == 0 && s.MPI_TAG == 40 + m && s.bytes == P);
        if (m >= 0) CHECK(s.method == m);
        int cnt = -1;
        CHECK(MPI_Get_count(&s, t, &cnt) == MPI_SUCCESS && cnt == 1);
        cudaMemcpy(h, d, N, cudaMemcpyDeviceToHost);
        for (long i = 0; i < N; ++i) {
          const int z = (int)(i / (Y * X)), y = (int)(i / X % Y), x = (int)(i % X);
          const int in = z >= 3 && z < 11 && y >= 5 && y < 37 && x >= 64 && x < 128;
          CHECK(h[i] == (in ? pat(i, m + 2) : 0x5A));
        }
      }
    }
  }
  MPI_Barrier(MPI_COMM_WORLD);
  MPI_Type_free(&t);
  MPI_Finalize();
  if (rank == 0) printf("OK\n");
  return 0;
}
