/* A portable MPI program for the interposer (libtempi_interpose.so) over a
 * system MPI (tests/native/minimpi.c). Nothing here is TEMPI-specific except
 * TEMPI_Set_method: the same source links against any MPI.
 *
 * Every device-memory result is checked against the SYSTEM MPI's own host
 * implementation on the same bytes: MPI_Pack / MPI_Unpack of a host copy
 * (pageable memory, so the interposer forwards those calls untouched).
 *  1. MPI_Pack / MPI_Unpack of six derived types (vector, 3-D subarray,
 *     hvector, irregular indexed, resized struct, and an hindexed with a
 *     negative displacement that the engine rejects and the system MPI
 *     keeps) on device memory, into device and pinned packed buffers;
 *  2. with 2+ ranks: MPI_Send / MPI_Recv rank 0 -> 1 for every transfer
 *     method and the model's choice (status.method reports the receiver's),
 *     a receive into HOST memory with the derived type (the wire format is
 *     the type signature, so a receiver without the interposer reads it),
 *     MPI_Isend / MPI_Irecv / MPI_Waitall in both directions, MPI_Sendrecv,
 *     the set completions (Waitany, Waitsome, Testall, Testany,
 *     Request_free) on device receives of every type, and persistent
 *     requests (Send_init / Recv_init / Startall) over three rounds.
 * Without a GPU only the host paths run (everything is forwarded): the same
 * types packed, unpacked and sent between ranks from host memory.
 * As with any CUDA-aware MPI, a device buffer is ready (its cudaMemset has
 * completed) before it is handed to an MPI call: a peer may write it
 * directly.
 * Prints "OK". */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include <mpi.h>

/* weak: present when the interposer is loaded (linked or LD_PRELOADed) */
int TEMPI_Set_method(int method) __attribute__((weak));

static int rank = 0, size = 1;
#define CHECK(c) do { if (!(c)) { printf("FAIL rank %d line %d: %s\n", rank, __LINE__, #c); fflush(stdout); MPI_Abort(MPI_COMM_WORLD, 1); } } while (0)

#define NT 6
#define COUNT 3

static unsigned char pat(long i, int salt) { return (unsigned char)((i * 131 + salt * 17 + (i >> 9)) & 0xff); }

int main(int argc, char **argv) {
  MPI_Init(&argc, &argv);
  MPI_Comm_rank(MPI_COMM_WORLD, &rank);
  MPI_Comm_size(MPI_COMM_WORLD, &size);
  int ndev = 0;
  const int gpu = cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0;
  MPI_Datatype t[NT], tmp;
  CHECK(MPI_Type_vector(4096, 1, 64, MPI_DOUBLE, &t[0]) == MPI_SUCCESS);
  {
    const int sizes[3] = {64, 64, 256}, subs[3] = {16, 32, 64}, starts[3] = {3, 5, 64};
    CHECK(MPI_Type_create_subarray(3, sizes, subs, starts, MPI_ORDER_C, MPI_BYTE, &t[1]) == MPI_SUCCESS);
  }
  CHECK(MPI_Type_create_hvector(64, 3, 200, MPI_FLOAT, &t[2]) == MPI_SUCCESS);
  {
    const int bl[4] = {2, 1, 3, 1}, d[4] = {9, 0, 4, 14};
    CHECK(MPI_Type_indexed(4, bl, d, MPI_DOUBLE, &t[3]) == MPI_SUCCESS);
  }
  {
    const int bl[2] = {1, 2};
    const MPI_Aint d[2] = {0, 8};
    const MPI_Datatype ty[2] = {MPI_INT, MPI_DOUBLE};
    CHECK(MPI_Type_create_struct(2, bl, d, ty, &tmp) == MPI_SUCCESS);
    CHECK(MPI_Type_create_resized(tmp, 0, 32, &t[4]) == MPI_SUCCESS);
    CHECK(MPI_Type_free(&tmp) == MPI_SUCCESS);
  }
  int nt = NT;
  {
    const int bl[3] = {16, 8, 4};
    const MPI_Aint d[3] = {64, -32, 200};
    /* an MPI that refuses negative displacements (the engine's own library
     * does) runs the other five */
    if (MPI_Type_create_hindexed(3, bl, d, MPI_BYTE, &t[5]) != MPI_SUCCESS) nt = NT - 1;
  }
  for (int k = 0; k < nt; ++k) CHECK(MPI_Type_commit(&t[k]) == MPI_SUCCESS);

  for (int k = 0; k < nt; ++k) {
    int tsize = 0;
    MPI_Aint lb = 0, ext = 0;
    CHECK(MPI_Type_size(t[k], &tsize) == MPI_SUCCESS && MPI_Type_get_extent(t[k], &lb, &ext) == MPI_SUCCESS);
    const long base = lb < 0 ? -lb : 0;                       /* buffer start -> MPI address 0 */
    const long span = base + COUNT * ext + (lb > 0 ? lb : 0) + 64; /* every byte any object touches */
    const int P = tsize * COUNT;
    unsigned char *h = malloc(span), *hp = malloc(P), *hd = malloc(span), *back = malloc(span);
    unsigned char *d = NULL, *dp = NULL, *dd = NULL, *pin = NULL, *got = malloc(P);
    for (long i = 0; i < span; ++i) h[i] = pat(i, k);
    if (gpu) CHECK(cudaMalloc((void **)&d, span) == cudaSuccess && cudaMalloc((void **)&dp, P) == cudaSuccess &&
          cudaMalloc((void **)&dd, span) == cudaSuccess && cudaMallocHost((void **)&pin, P) == cudaSuccess);
    if (gpu) cudaMemcpy(d, h, span, cudaMemcpyHostToDevice);
    /* the system MPI on host memory: the expected packed bytes and unpack */
    int pos = 0;
    CHECK(MPI_Pack(h + base, COUNT, t[k], hp, P, &pos, MPI_COMM_WORLD) == MPI_SUCCESS && pos == P);
    memset(hd, 0xCD, span);
    pos = 0;
    CHECK(MPI_Unpack(hp, P, &pos, hd + base, COUNT, t[k], MPI_COMM_WORLD) == MPI_SUCCESS && pos == P);
    if (!gpu) { /* host only: the round trip, and host messages below */
      memset(back, 0xCD, span);
      for (long i = 0; i < span; ++i) if (hd[i] != 0xCD) back[i] = h[i];
      CHECK(memcmp(back, hd, span) == 0);
      if (size >= 2 && rank < 2) {
        if (rank == 0) {
          CHECK(MPI_Send(h + base, COUNT, t[k], 1, 5, MPI_COMM_WORLD) == MPI_SUCCESS);
        } else {
          memset(back, 0xCD, span);
          CHECK(MPI_Recv(back + base, COUNT, t[k], 0, 5, MPI_COMM_WORLD, MPI_STATUS_IGNORE) == MPI_SUCCESS);
          CHECK(memcmp(back, hd, span) == 0);
        }
      }
      goto next;
    }
    /* device -> device packed */
    cudaMemset(dp, 0, P); cudaDeviceSynchronize();
    pos = 0;
    CHECK(MPI_Pack(d + base, COUNT, t[k], dp, P, &pos, MPI_COMM_WORLD) == MPI_SUCCESS && pos == P);
    cudaMemcpy(got, dp, P, cudaMemcpyDeviceToHost);
    CHECK(memcmp(got, hp, P) == 0);
    /* device -> pinned host packed */
    memset(pin, 0, P);
    pos = 0;
    CHECK(MPI_Pack(d + base, COUNT, t[k], pin, P, &pos, MPI_COMM_WORLD) == MPI_SUCCESS && pos == P);
    CHECK(memcmp(pin, hp, P) == 0);
    /* unpack into device memory: described bytes written, the rest kept */
    cudaMemset(dd, 0xCD, span); cudaDeviceSynchronize();
    pos = 0;
    CHECK(MPI_Unpack(dp, P, &pos, dd + base, COUNT, t[k], MPI_COMM_WORLD) == MPI_SUCCESS && pos == P);
    cudaMemcpy(back, dd, span, cudaMemcpyDeviceToHost);
    CHECK(memcmp(back, hd, span) == 0);
    /* a truncated packed buffer is an error, not an overrun */
    pos = 0;
    CHECK(MPI_Pack(d + base, COUNT, t[k], dp, P - 1, &pos, MPI_COMM_WORLD) != MPI_SUCCESS);

    if (size >= 2 && rank < 2) {
      /* Send/Recv 0 -> 1, every method and the model's choice */
      for (int m = -1; m <= 2; ++m) {
        if (m >= 0 && !TEMPI_Set_method) continue;
        if (TEMPI_Set_method) CHECK(TEMPI_Set_method(m) == MPI_SUCCESS);
        if (rank == 0) {
          CHECK(MPI_Send(d + base, COUNT, t[k], 1, 100 + m, MPI_COMM_WORLD) == MPI_SUCCESS);
        } else {
          MPI_Status s;
          cudaMemset(dd, 0xCD, span); cudaDeviceSynchronize();
          CHECK(MPI_Recv(dd + base, COUNT, t[k], 0, 100 + m, MPI_COMM_WORLD, &s) == MPI_SUCCESS);
          CHECK(s.MPI_SOURCE == 0 && s.MPI_TAG == 100 + m);
          int cnt = -1;
          CHECK(MPI_Get_count(&s, t[k], &cnt) == MPI_SUCCESS && cnt == COUNT);
          /* a system MPI that cannot read device memory gets staged messages */
          const int aware = !getenv("TEMPI_CUDA_AWARE") || atoi(getenv("TEMPI_CUDA_AWARE"));
          if (m >= 0 && k != 5) CHECK(s.method == (m == 1 && !aware ? 2 : m));
          cudaMemcpy(back, dd, span, cudaMemcpyDeviceToHost);
          CHECK(memcmp(back, hd, span) == 0);
        }
      }
      if (TEMPI_Set_method) TEMPI_Set_method(-1);
      /* device sender, HOST receiver with the derived type: the system MPI
       * unpacks the interposer's packed bytes */
      if (rank == 0) {
        CHECK(MPI_Send(d + base, COUNT, t[k], 1, 7, MPI_COMM_WORLD) == MPI_SUCCESS);
      } else {
        unsigned char *hr = malloc(span);
        memset(hr, 0xCD, span);
        CHECK(MPI_Recv(hr + base, COUNT, t[k], 0, 7, MPI_COMM_WORLD, MPI_STATUS_IGNORE) == MPI_SUCCESS);
        CHECK(memcmp(hr, hd, span) == 0);
        free(hr);
      }
      /* Isend/Irecv both ways at once */
      {
        const int peer = 1 - rank;
        MPI_Request rq[2];
        MPI_Status st[2];
        cudaMemset(dd, 0xCD, span); cudaDeviceSynchronize();
        CHECK(MPI_Irecv(dd + base, COUNT, t[k], peer, 8, MPI_COMM_WORLD, &rq[0]) == MPI_SUCCESS);
        CHECK(MPI_Isend(d + base, COUNT, t[k], peer, 8, MPI_COMM_WORLD, &rq[1]) == MPI_SUCCESS);
        CHECK(MPI_Waitall(2, rq, st) == MPI_SUCCESS);
        CHECK(rq[0] == MPI_REQUEST_NULL && rq[1] == MPI_REQUEST_NULL);
        cudaMemcpy(back, dd, span, cudaMemcpyDeviceToHost);
        CHECK(memcmp(back, hd, span) == 0);
      }
      /* Sendrecv */
      {
        const int peer = 1 - rank;
        cudaMemset(dd, 0xCD, span); cudaDeviceSynchronize();
        CHECK(MPI_Sendrecv(d + base, COUNT, t[k], peer, 9, dd + base, COUNT, t[k], peer, 9, MPI_COMM_WORLD,
                           MPI_STATUS_IGNORE) == MPI_SUCCESS);
        cudaMemcpy(back, dd, span, cudaMemcpyDeviceToHost);
        CHECK(memcmp(back, hd, span) == 0);
      }
      /* the set completions (MPI-3.1 3.7.5): receives by Waitany, sends by
       * Waitsome; then receives by Testall polling, sends by Testany; then a
       * send released with MPI_Request_free */
      {
        const int peer = 1 - rank;
        unsigned char *r3[3];
        MPI_Request rr[3], sr[3];
        for (int i = 0; i < 3; ++i) {
          CHECK(cudaMalloc((void **)&r3[i], span) == cudaSuccess);
          cudaMemset(r3[i], 0xCD, span); cudaDeviceSynchronize();
          CHECK(MPI_Irecv(r3[i] + base, COUNT, t[k], peer, 30 + i, MPI_COMM_WORLD, &rr[i]) == MPI_SUCCESS);
        }
        for (int i = 0; i < 3; ++i)
          CHECK(MPI_Isend(d + base, COUNT, t[k], peer, 30 + i, MPI_COMM_WORLD, &sr[i]) == MPI_SUCCESS);
        int seen = 0;
        for (int i = 0; i < 3; ++i) {
          int idx = -1;
          MPI_Status st;
          CHECK(MPI_Waitany(3, rr, &idx, &st) == MPI_SUCCESS && idx >= 0 && idx < 3 && rr[idx] == MPI_REQUEST_NULL);
          CHECK(st.MPI_TAG == 30 + idx && !(seen & (1 << idx)));
          seen |= 1 << idx;
        }
        int idx = 0;
        CHECK(MPI_Waitany(3, rr, &idx, MPI_STATUS_IGNORE) == MPI_SUCCESS && idx == MPI_UNDEFINED);
        for (int left = 3; left > 0;) {
          int n = 0, ind[3];
          CHECK(MPI_Waitsome(3, sr, &n, ind, MPI_STATUSES_IGNORE) == MPI_SUCCESS && n >= 1);
          left -= n;
        }
        for (int i = 0; i < 3; ++i) {
          cudaMemcpy(back, r3[i], span, cudaMemcpyDeviceToHost);
          CHECK(memcmp(back, hd, span) == 0);
          cudaMemset(r3[i], 0xCD, span); cudaDeviceSynchronize();
        }
        for (int i = 0; i < 2; ++i)
          CHECK(MPI_Irecv(r3[i] + base, COUNT, t[k], peer, 40 + i, MPI_COMM_WORLD, &rr[i]) == MPI_SUCCESS);
        for (int i = 0; i < 2; ++i)
          CHECK(MPI_Isend(d + base, COUNT, t[k], peer, 40 + i, MPI_COMM_WORLD, &sr[i]) == MPI_SUCCESS);
        int flag = 0;
        MPI_Status st2[2];
        while (!flag) CHECK(MPI_Testall(2, rr, &flag, st2) == MPI_SUCCESS);
        CHECK(rr[0] == MPI_REQUEST_NULL && rr[1] == MPI_REQUEST_NULL && st2[1].MPI_TAG == 41);
        for (int done = 0; done < 2;) {
          int f = 0, ix = -1;
          CHECK(MPI_Testany(2, sr, &ix, &f, MPI_STATUS_IGNORE) == MPI_SUCCESS);
          if (f && ix != MPI_UNDEFINED) ++done;
        }
        for (int i = 0; i < 2; ++i) {
          cudaMemcpy(back, r3[i], span, cudaMemcpyDeviceToHost);
          CHECK(memcmp(back, hd, span) == 0);
        }
        cudaMemset(r3[2], 0xCD, span); cudaDeviceSynchronize();
        CHECK(MPI_Irecv(r3[2] + base, COUNT, t[k], peer, 50, MPI_COMM_WORLD, &rr[2]) == MPI_SUCCESS);
        CHECK(MPI_Isend(d + base, COUNT, t[k], peer, 50, MPI_COMM_WORLD, &sr[2]) == MPI_SUCCESS);
        CHECK(MPI_Request_free(&sr[2]) == MPI_SUCCESS && sr[2] == MPI_REQUEST_NULL);
        CHECK(MPI_Wait(&rr[2], MPI_STATUS_IGNORE) == MPI_SUCCESS);
        cudaMemcpy(back, r3[2], span, cudaMemcpyDeviceToHost);
        CHECK(memcmp(back, hd, span) == 0);
        /* a datatype freed while a receive using it is pending (MPI-3.1
         * 4.1.9: the operation completes normally) */
        MPI_Datatype tmp2;
        CHECK(MPI_Type_contiguous(1, t[k], &tmp2) == MPI_SUCCESS && MPI_Type_commit(&tmp2) == MPI_SUCCESS);
        cudaMemset(r3[1], 0xCD, span); cudaDeviceSynchronize();
        CHECK(MPI_Irecv(r3[1] + base, COUNT, tmp2, peer, 60, MPI_COMM_WORLD, &rr[1]) == MPI_SUCCESS);
        CHECK(MPI_Type_free(&tmp2) == MPI_SUCCESS);
        CHECK(MPI_Send(d + base, COUNT, t[k], peer, 60, MPI_COMM_WORLD) == MPI_SUCCESS);
        CHECK(MPI_Wait(&rr[1], MPI_STATUS_IGNORE) == MPI_SUCCESS);
        cudaMemcpy(back, r3[1], span, cudaMemcpyDeviceToHost);
        CHECK(memcmp(back, hd, span) == 0);
        /* persistent requests (MPI-3.1 3.9): three rounds of Startall +
         * Waitall on the same requests, the send data changing between
         * rounds (each MPI_Start packs the current contents) */
        MPI_Request pr[2];
        CHECK(MPI_Recv_init(r3[0] + base, COUNT, t[k], peer, 70, MPI_COMM_WORLD, &pr[0]) == MPI_SUCCESS);
        CHECK(MPI_Send_init(d + base, COUNT, t[k], peer, 70, MPI_COMM_WORLD, &pr[1]) == MPI_SUCCESS);
        for (int round = 0; round < 3; ++round) {
          for (long i = 0; i < span; ++i) h[i] = pat(i, k + 7 * round + 1);
          cudaMemcpy(d, h, span, cudaMemcpyHostToDevice);
          cudaMemset(r3[0], 0xCD, span); cudaDeviceSynchronize();
          MPI_Barrier(MPI_COMM_WORLD);
          CHECK(MPI_Startall(2, pr) == MPI_SUCCESS);
          MPI_Status ps[2];
          CHECK(MPI_Waitall(2, pr, ps) == MPI_SUCCESS);
          CHECK(pr[0] != MPI_REQUEST_NULL && pr[1] != MPI_REQUEST_NULL); /* inactive, not freed */
          /* expected: the host unpack of this round's pattern */
          int q = 0;
          unsigned char *hp2 = malloc(P), *exp2 = malloc(span);
          CHECK(MPI_Pack(h + base, COUNT, t[k], hp2, P, &q, MPI_COMM_WORLD) == MPI_SUCCESS);
          memset(exp2, 0xCD, span);
          q = 0;
          CHECK(MPI_Unpack(hp2, P, &q, exp2 + base, COUNT, t[k], MPI_COMM_WORLD) == MPI_SUCCESS);
          cudaMemcpy(back, r3[0], span, cudaMemcpyDeviceToHost);
          CHECK(memcmp(back, exp2, span) == 0);
          free(hp2);
          free(exp2);
        }
        int f2 = 0;
        CHECK(MPI_Test(&pr[0], &f2, MPI_STATUS_IGNORE) == MPI_SUCCESS && f2); /* inactive: complete */
        CHECK(MPI_Request_free(&pr[0]) == MPI_SUCCESS && pr[0] == MPI_REQUEST_NULL);
        CHECK(MPI_Request_free(&pr[1]) == MPI_SUCCESS && pr[1] == MPI_REQUEST_NULL);
        for (long i = 0; i < span; ++i) h[i] = pat(i, k); /* restore the source */
        cudaMemcpy(d, h, span, cudaMemcpyHostToDevice);
        for (int i = 0; i < 3; ++i) cudaFree(r3[i]);
      }
    }
  next:
    MPI_Barrier(MPI_COMM_WORLD);
    if (gpu) {
      cudaFree(d);
      cudaFree(dp);
      cudaFree(dd);
      cudaFreeHost(pin);
    }
    free(h);
    free(hp);
    free(hd);
    free(back);
    free(got);
  }
  for (int k = 0; k < nt; ++k) CHECK(MPI_Type_free(&t[k]) == MPI_SUCCESS);
  MPI_Finalize();
  if (rank == 0) printf("OK\n");
  return 0;
}
