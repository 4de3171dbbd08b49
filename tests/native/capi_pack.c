/* The engine's C-ABI from plain C (no Python, no MPI): a 3-D subarray of a
 * device array packed with sp_pack, unpacked with sp_unpack into a
 * sentinel-filled copy, and moved directly with sp_copy into a differently
 * shaped destination type of the same size; every byte checked on the host
 * against the C-order definition. Prints "OK". */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include "stridepack_b200.h"

#define CHECK(c) do { if (!(c)) { printf("FAIL line %d: %s (%s)\n", __LINE__, #c, sp_last_error()); return 1; } } while (0)

int main(void) {
  CHECK(sp_abi_version() == SP_ABI_VERSION);
  /* reference order: dim 0 innermost (type_def.hpp:75) */
  const int64_t sizes[3] = {96, 40, 24}, subs[3] = {32, 8, 4}, offs[3] = {3, 5, 7};
  sp_type byte, sub, row, dst_t;
  CHECK(sp_type_named(SP_BYTE, &byte) == SP_OK);
  CHECK(sp_type_subarray(3, sizes, subs, offs, byte, SP_ORDER_C, &sub) == SP_OK);
  CHECK(sp_type_commit(sub) == SP_OK);
  sp_type_info info;
  int64_t counts[8], strides[8];
  CHECK(sp_type_query(sub, &info, counts, strides, 8) == SP_OK);
  CHECK(info.form == SP_FORM_STRIDED && info.size == 32 * 8 * 4 && info.ndims == 3);
  CHECK(counts[0] == 32 && counts[1] == 8 && counts[2] == 4 && strides[1] == 96 && strides[2] == 96 * 40);
  /* destination: 32 rows of 32 B at a 48-B pitch (same 1024 bytes) */
  CHECK(sp_type_contiguous(32, byte, &row) == SP_OK);
  CHECK(sp_type_hvector(32, 1, 48, row, &dst_t) == SP_OK);
  CHECK(sp_type_commit(dst_t) == SP_OK);

  const long n = 96L * 40 * 24;
  unsigned char *h = malloc(n), *hp = malloc(info.size), *hb = malloc(n), *hd = malloc(2048);
  for (long i = 0; i < n; ++i) h[i] = (unsigned char)(i * 37 + 11);
  unsigned char *d, *dp, *db, *dd;
  CHECK(cudaMalloc((void **)&d, n) == cudaSuccess);
  CHECK(cudaMalloc((void **)&dp, info.size) == cudaSuccess);
  CHECK(cudaMalloc((void **)&db, n) == cudaSuccess);
  CHECK(cudaMalloc((void **)&dd, 2048) == cudaSuccess);
  cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
  cudaMemset(db, 0xC3, n);
  cudaMemset(dd, 0x5A, 2048);

  int64_t pos = 0;
  CHECK(sp_pack(d, n, sub, 1, dp, info.size, &pos, NULL) == SP_OK && pos == info.size);
  pos = 0;
  CHECK(sp_unpack(dp, info.size, &pos, sub, 1, db, n, NULL) == SP_OK && pos == info.size);
  sp_copy_job job = {d, (uint64_t)n, sub, 1, dd, 2048, dst_t, 1};
  CHECK(sp_copy(&job, NULL) == SP_OK);
  CHECK(cudaDeviceSynchronize() == cudaSuccess);
  cudaMemcpy(hp, dp, info.size, cudaMemcpyDeviceToHost);
  cudaMemcpy(hb, db, n, cudaMemcpyDeviceToHost);
  cudaMemcpy(hd, dd, 2048, cudaMemcpyDeviceToHost);

  long k = 0; /* packed order: dim 0 fastest */
  for (int z = 0; z < 4; ++z)
    for (int y = 0; y < 8; ++y)
      for (int x = 0; x < 32; ++x, ++k) {
        const long src = ((long)(z + 7) * 40 + (y + 5)) * 96 + (x + 3);
        CHECK(hp[k] == h[src]);
      }
  for (long i = 0; i < n; ++i) {
    const long x = i % 96, y = i / 96 % 40, z = i / (96 * 40);
    const int in = x >= 3 && x < 35 && y >= 5 && y < 13 && z >= 7 && z < 11;
    CHECK(hb[i] == (in ? h[i] : 0xC3));
  }
  for (long i = 0; i < 2048; ++i) {
    const long r = i / 48, c = i % 48;
    CHECK(hd[i] == ((r < 32 && c < 32) ? hp[r * 32 + c] : 0x5A));
  }
  /* the error contract: a too-small destination reports BufferTooSmall */
  pos = 0;
  CHECK(sp_pack(d, n, sub, 1, dp, info.size - 1, &pos, NULL) == SP_ERR_BUFFER_TOO_SMALL);
  CHECK(strstr(sp_last_error(), "need") != NULL);
  sp_type_free(sub);
  sp_type_free(row);
  sp_type_free(dst_t);
  sp_type_free(byte);
  printf("OK\n");
  return 0;
}
