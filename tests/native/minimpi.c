/* minimpi.c -- TEST INFRASTRUCTURE: a small stand-in for "the system MPI".
 *
 * TEMPI is an interposer: it exports the MPI_* entry points it accelerates
 * and forwards everything else, and its own transport, to the system MPI
 * through PMPI_* (PAPER.md:781-796). This image ships no MPI library, so the
 * interposer (paper_2012_14363_b200/libtempi_interpose.so) is tested over
 * this one: libminimpi.so, built from this file by the tests, written
 * against include/mpi.h (MPICH-style int handles).
 *
 * What it is:
 *  * a complete, slow, obviously-correct MPI subset: every PMPI_* has an
 *    MPI_* alias, and internal calls never go through MPI_* (so an
 *    interposer sees only the application's calls, as with MPICH/Open MPI);
 *  * datatypes as flattened typemaps (offset, length) runs, MPI-3.1 4.1
 *    semantics (lb/ub from the displacements, subarray resized to the full
 *    array);
 *  * CUDA-aware the way a generic MPI is for derived types on device
 *    memory: one cudaMemcpy per contiguous run on the device, the packed
 *    bytes then crossing to or from host memory in one copy (the per-block
 *    path TEMPI replaces); contiguous data in one copy;
 *  * transport: UNIX-domain sockets under /tmp/minimpi-<job>/, one
 *    reader thread per incoming connection feeding a FIFO mailbox; every
 *    send is eager (buffered), so MPI_Send never blocks on the receiver.
 * Neighbourhood collectives follow MPI-3.1 7.6: the k-th message between a
 * pair of ranks in one call matches the k-th edge between them.
 * Launch with tools/tempirun.py (TEMPI_RANK / TEMPI_SIZE / TEMPI_JOB).
 */
#define _GNU_SOURCE
#include <cuda_runtime.h>
#include <errno.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/stat.h>
#include <sys/un.h>
#include <time.h>
#include <unistd.h>

#include "mpi.h"

#define ALIAS(name) __attribute__((alias("P" #name)))

/* ------------------------------------------------------------ datatypes */
typedef struct {
  int used, committed;
  int64_t size, lb, extent, nruns;
  int64_t *off, *len;
} Type;

static Type *g_types;
static int g_ntypes, g_captypes;

static Type *type_of(MPI_Datatype t) {
  return (t > 0 && t < g_ntypes && g_types[t].used) ? &g_types[t] : NULL;
}

static int new_type(Type *tmpl, MPI_Datatype *out) {
  if (g_ntypes == g_captypes) {
    g_captypes = g_captypes ? 2 * g_captypes : 64;
    g_types = realloc(g_types, sizeof(Type) * g_captypes);
  }
  g_types[g_ntypes] = *tmpl;
  g_types[g_ntypes].used = 1;
  *out = g_ntypes++;
  return MPI_SUCCESS;
}

/* builder: runs of a new typemap, merged when contiguous */
typedef struct {
  int64_t n, cap, size;
  int64_t *off, *len;
  int any;
  int64_t lb, ub;
} Build;

static void push_run(Build *b, int64_t off, int64_t len) {
  if (len <= 0) return;
  if (b->n && b->off[b->n - 1] + b->len[b->n - 1] == off) {
    b->len[b->n - 1] += len;
  } else {
    if (b->n == b->cap) {
      b->cap = b->cap ? 2 * b->cap : 16;
      b->off = realloc(b->off, sizeof(int64_t) * b->cap);
      b->len = realloc(b->len, sizeof(int64_t) * b->cap);
    }
    b->off[b->n] = off;
    b->len[b->n] = len;
    ++b->n;
  }
  b->size += len;
}

/* one copy of `t` displaced by `d` bytes */
static void push_type(Build *b, const Type *t, int64_t d) {
  for (int64_t i = 0; i < t->nruns; ++i) push_run(b, d + t->off[i], t->len[i]);
  const int64_t lo = d + t->lb, hi = d + t->lb + t->extent;
  if (!b->any || lo < b->lb) b->lb = lo;
  if (!b->any || hi > b->ub) b->ub = hi;
  b->any = 1;
}

static int finish(Build *b, MPI_Datatype *out) {
  Type t = {0};
  t.size = b->size;
  t.lb = b->any ? b->lb : 0;
  t.extent = b->any ? b->ub - b->lb : 0;
  t.nruns = b->n;
  t.off = b->off;
  t.len = b->len;
  return new_type(&t, out);
}

/* ------------------------------------------------------------ CUDA-aware copies */
static int is_device(const void *p) {
  struct cudaPointerAttributes a;
  if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static void copy_bytes(void *dst, const void *src, int64_t n, int dev) {
  if (n <= 0) return;
  if (dev)
    cudaMemcpy(dst, src, (size_t)n, cudaMemcpyDefault);
  else
    memcpy(dst, src, (size_t)n);
}

/* a cudaMemcpy from pageable memory may return before its DMA into device
 * memory has landed: the data must be in place when an MPI call returns,
 * also for a consumer on a non-blocking stream */
static void settle(int dev) {
  if (dev) cudaStreamSynchronize(0);
}

/* one run that fills its extent: `count` objects are one contiguous block
 * (every MPI takes this path for contiguous data) */
static int dense(const Type *t) { return t->nruns == 1 && t->off[0] == 0 && t->len[0] == t->extent; }

/* gather `count` objects of `t` at buf into out (type-signature byte order).
 * Device data moves one cudaMemcpy per run on the device; when the other
 * side is host memory the packed bytes then cross in one copy (what a
 * CUDA-aware MPI without datatype kernels does) */
static void gather(const Type *t, const void *buf, int64_t count, uint8_t *out) {
  const int dbuf = is_device(buf), dout = is_device(out), dev = dbuf || dout;
  if (dense(t)) {
    copy_bytes(out, buf, count * t->extent, dev);
    settle(dev);
    return;
  }
  uint8_t *dst = out, *stage = NULL;
  if (dbuf && !dout && count * t->size > 0 && cudaMalloc((void **)&stage, (size_t)(count * t->size)) == cudaSuccess)
    dst = stage;
  int64_t pos = 0;
  for (int64_t e = 0; e < count; ++e)
    for (int64_t i = 0; i < t->nruns; ++i) {
      copy_bytes(dst + pos, (const uint8_t *)buf + e * t->extent + t->off[i], t->len[i], dev);
      pos += t->len[i];
    }
  if (stage) {
    cudaMemcpy(out, stage, (size_t)pos, cudaMemcpyDeviceToHost);
    cudaFree(stage);
  }
  settle(dev);
}

static void scatter(const Type *t, const uint8_t *in, int64_t count, void *buf) {
  const int dbuf = is_device(buf), din = is_device(in), dev = dbuf || din;
  if (dense(t)) {
    copy_bytes(buf, in, count * t->extent, dev);
    settle(dev);
    return;
  }
  uint8_t *stage = NULL;
  const uint8_t *src = in;
  if (dbuf && !din && count * t->size > 0 && cudaMalloc((void **)&stage, (size_t)(count * t->size)) == cudaSuccess) {
    cudaMemcpy(stage, in, (size_t)(count * t->size), cudaMemcpyHostToDevice);
    src = stage;
  }
  int64_t pos = 0;
  for (int64_t e = 0; e < count; ++e)
    for (int64_t i = 0; i < t->nruns; ++i) {
      copy_bytes((uint8_t *)buf + e * t->extent + t->off[i], src + pos, t->len[i], dev);
      pos += t->len[i];
    }
  if (stage) cudaFree(stage);
  settle(dev);
}

/* ------------------------------------------------------------ processes, comms */
typedef struct {
  int used, kind; /* 0 world/self, 1 dist graph, 2 cartesian */
  int nsrc, ndst, ndims;
  int *src, *dst, *dims, *periods;
} Comm;

static struct {
  int init, fin, rank, size;
  char dir[96];
  int lfd;
  int *fds;
  pthread_mutex_t send_mu;
  Comm comms[256];
  int ncomms;
} G = {.send_mu = PTHREAD_MUTEX_INITIALIZER};

typedef struct Msg {
  int src, tag, ctx;
  int64_t bytes;
  uint8_t *data;
  struct Msg *next;
} Msg;

static Msg *g_head, *g_tail;
static pthread_mutex_t g_mu = PTHREAD_MUTEX_INITIALIZER;
static pthread_cond_t g_cv = PTHREAD_COND_INITIALIZER;

static int read_full(int fd, void *p, size_t n) {
  uint8_t *b = p;
  while (n) {
    ssize_t k = read(fd, b, n);
    if (k <= 0) {
      if (k < 0 && errno == EINTR) continue;
      return -1;
    }
    b += k;
    n -= (size_t)k;
  }
  return 0;
}

static int write_full(int fd, const void *p, size_t n) {
  const uint8_t *b = p;
  while (n) {
    ssize_t k = write(fd, b, n);
    if (k <= 0) {
      if (k < 0 && errno == EINTR) continue;
      return -1;
    }
    b += k;
    n -= (size_t)k;
  }
  return 0;
}

typedef struct {
  int src, tag, ctx, pad;
  int64_t bytes;
} Header;

static void *reader(void *arg) {
  const int fd = (int)(intptr_t)arg;
  for (;;) {
    Header h;
    if (read_full(fd, &h, sizeof h)) break;
    Msg *m = calloc(1, sizeof(Msg));
    m->src = h.src;
    m->tag = h.tag;
    m->ctx = h.ctx;
    m->bytes = h.bytes;
    m->data = malloc(h.bytes ? (size_t)h.bytes : 1);
    if (read_full(fd, m->data, (size_t)h.bytes)) break;
    pthread_mutex_lock(&g_mu);
    if (g_tail) g_tail->next = m; else g_head = m;
    g_tail = m;
    pthread_cond_broadcast(&g_cv);
    pthread_mutex_unlock(&g_mu);
  }
  close(fd);
  return NULL;
}

static void *acceptor(void *arg) {
  (void)arg;
  for (;;) {
    int fd = accept(G.lfd, NULL, NULL);
    if (fd < 0) {
      if (errno == EINTR) continue;
      return NULL;
    }
    pthread_t t;
    pthread_create(&t, NULL, reader, (void *)(intptr_t)fd);
    pthread_detach(t);
  }
}

static void sock_path(int rank, struct sockaddr_un *a) {
  memset(a, 0, sizeof *a);
  a->sun_family = AF_UNIX;
  snprintf(a->sun_path, sizeof a->sun_path, "%s/%d", G.dir, rank);
}

static int conn(int dest) {
  if (G.fds[dest] >= 0) return G.fds[dest];
  struct sockaddr_un a;
  sock_path(dest, &a);
  for (int tries = 0; tries < 120000; ++tries) { /* up to ~2 min for the peer to start */
    int fd = socket(AF_UNIX, SOCK_STREAM, 0);
    if (connect(fd, (struct sockaddr *)&a, sizeof a) == 0) return G.fds[dest] = fd;
    close(fd);
    usleep(1000);
  }
  return -1;
}

/* an eager message of packed bytes to world rank `dest` */
static int post(int dest, int tag, int ctx, const void *data, int64_t bytes) {
  Header h = {G.rank, tag, ctx, 0, bytes};
  pthread_mutex_lock(&G.send_mu);
  const int fd = conn(dest);
  int rc = fd < 0 || write_full(fd, &h, sizeof h) || write_full(fd, data, (size_t)bytes);
  pthread_mutex_unlock(&G.send_mu);
  return rc ? MPI_ERR_OTHER : MPI_SUCCESS;
}

static Msg *match_locked(int src, int tag, int ctx, int take) {
  Msg *prev = NULL;
  for (Msg *m = g_head; m; prev = m, m = m->next)
    if (m->ctx == ctx && (src == MPI_ANY_SOURCE || m->src == src) && (tag == MPI_ANY_TAG || m->tag == tag)) {
      if (take) {
        if (prev) prev->next = m->next; else g_head = m->next;
        if (g_tail == m) g_tail = prev;
      }
      return m;
    }
  return NULL;
}

static Msg *fetch(int src, int tag, int ctx) {
  pthread_mutex_lock(&g_mu);
  Msg *m;
  while (!(m = match_locked(src, tag, ctx, 1))) pthread_cond_wait(&g_cv, &g_mu);
  pthread_mutex_unlock(&g_mu);
  return m;
}

static int env_int(const char *a, const char *b, int dflt) {
  const char *v = getenv(a);
  if (!v) v = getenv(b);
  return v ? atoi(v) : dflt;
}

static Comm *comm_of(MPI_Comm c) {
  if (c == MPI_COMM_WORLD || c == MPI_COMM_SELF) return &G.comms[0];
  return (c >= 100 && c - 100 < G.ncomms && G.comms[c - 100].used) ? &G.comms[c - 100] : NULL;
}

/* point-to-point context of a communicator (collectives use ctx + 1) */
static int ctx_of(MPI_Comm c) { return c == MPI_COMM_SELF ? 4 : c == MPI_COMM_WORLD ? 2 : 2 * c; }
static int world_rank(MPI_Comm c, int r) { return c == MPI_COMM_SELF ? G.rank : r; }

/* ------------------------------------------------------------ runtime */
int PMPI_Init(int *argc, char ***argv) {
  (void)argc;
  (void)argv;
  if (G.init) return MPI_ERR_OTHER;
  G.rank = env_int("TEMPI_RANK", "RANK", 0);
  G.size = env_int("TEMPI_SIZE", "WORLD_SIZE", 1);
  const char *job = getenv("TEMPI_JOB") ? getenv("TEMPI_JOB") : getenv("MASTER_PORT");
  char jb[64];
  if (!job) {
    snprintf(jb, sizeof jb, "single%d", (int)getpid());
    job = jb;
  }
  /* not $TMPDIR: a socket path must fit sun_path (108 bytes) */
  snprintf(G.dir, sizeof G.dir, "/tmp/minimpi-%.64s", job);
  mkdir(G.dir, 0700);
  G.fds = malloc(sizeof(int) * G.size);
  for (int i = 0; i < G.size; ++i) G.fds[i] = -1;
  struct sockaddr_un a;
  sock_path(G.rank, &a);
  unlink(a.sun_path);
  G.lfd = socket(AF_UNIX, SOCK_STREAM, 0);
  if (bind(G.lfd, (struct sockaddr *)&a, sizeof a) || listen(G.lfd, 64)) return MPI_ERR_OTHER;
  pthread_t t;
  pthread_create(&t, NULL, acceptor, NULL);
  pthread_detach(t);
  /* predefined types 1..7 (mpi.h) */
  const int64_t named[] = {0, 1, 1, 4, 4, 8, 1, 1};
  for (int i = 0; i < 8; ++i) {
    Build b = {0};
    if (i) {
      push_run(&b, 0, named[i]);
      b.any = 1;
      b.lb = 0;
      b.ub = named[i];
    }
    MPI_Datatype h;
    finish(&b, &h);
    g_types[h].used = i > 0;
    g_types[h].committed = 1;
  }
  G.comms[0].used = 1;
  G.ncomms = 1;
  G.init = 1;
  return MPI_SUCCESS;
}
int MPI_Init(int *argc, char ***argv) ALIAS(MPI_Init);

int PMPI_Init_thread(int *argc, char ***argv, int required, int *provided) {
  (void)required;
  if (provided) *provided = MPI_THREAD_SERIALIZED;
  return PMPI_Init(argc, argv);
}
int MPI_Init_thread(int *argc, char ***argv, int required, int *provided) ALIAS(MPI_Init_thread);

int PMPI_Initialized(int *flag) {
  *flag = G.init;
  return MPI_SUCCESS;
}
int MPI_Initialized(int *flag) ALIAS(MPI_Initialized);

int PMPI_Finalized(int *flag) {
  *flag = G.fin;
  return MPI_SUCCESS;
}
int MPI_Finalized(int *flag) ALIAS(MPI_Finalized);

int PMPI_Comm_rank(MPI_Comm comm, int *rank) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  *rank = comm == MPI_COMM_SELF ? 0 : G.rank;
  return MPI_SUCCESS;
}
int MPI_Comm_rank(MPI_Comm comm, int *rank) ALIAS(MPI_Comm_rank);

int PMPI_Comm_size(MPI_Comm comm, int *size) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  *size = comm == MPI_COMM_SELF ? 1 : G.size;
  return MPI_SUCCESS;
}
int MPI_Comm_size(MPI_Comm comm, int *size) ALIAS(MPI_Comm_size);

int PMPI_Barrier(MPI_Comm comm) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (comm == MPI_COMM_SELF || G.size == 1) return MPI_SUCCESS;
  const int ctx = 1; /* the barrier context */
  char z = 0;
  if (G.rank == 0) {
    for (int r = 1; r < G.size; ++r) {
      Msg *m = fetch(r, 0, ctx);
      free(m->data);
      free(m);
    }
    for (int r = 1; r < G.size; ++r)
      if (post(r, 1, ctx, &z, 1)) return MPI_ERR_OTHER;
  } else {
    if (post(0, 0, ctx, &z, 1)) return MPI_ERR_OTHER;
    Msg *m = fetch(0, 1, ctx);
    free(m->data);
    free(m);
  }
  return MPI_SUCCESS;
}
int MPI_Barrier(MPI_Comm comm) ALIAS(MPI_Barrier);

int PMPI_Finalize(void) {
  if (!G.init || G.fin) return MPI_ERR_OTHER;
  PMPI_Barrier(MPI_COMM_WORLD);
  pthread_mutex_lock(&G.send_mu);
  for (int i = 0; i < G.size; ++i)
    if (G.fds[i] >= 0) close(G.fds[i]);
  pthread_mutex_unlock(&G.send_mu);
  struct sockaddr_un a;
  sock_path(G.rank, &a);
  unlink(a.sun_path);
  rmdir(G.dir); /* the last rank out removes it */
  G.fin = 1;
  return MPI_SUCCESS;
}
int MPI_Finalize(void) ALIAS(MPI_Finalize);

int PMPI_Abort(MPI_Comm comm, int code) {
  (void)comm;
  fprintf(stderr, "minimpi: MPI_Abort(%d) on rank %d\n", code, G.rank);
  fflush(NULL); /* the caller's diagnostics on a piped stdout */
  _exit(code ? code : 1);
}
int MPI_Abort(MPI_Comm comm, int code) ALIAS(MPI_Abort);

double PMPI_Wtime(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
double MPI_Wtime(void) ALIAS(MPI_Wtime);

int PMPI_Error_string(int code, char *s, int *len) {
  *len = snprintf(s, MPI_MAX_ERROR_STRING, "minimpi error %d", code);
  return MPI_SUCCESS;
}
int MPI_Error_string(int code, char *s, int *len) ALIAS(MPI_Error_string);

int PMPI_Get_count(const MPI_Status *st, MPI_Datatype dt, int *count) {
  const Type *t = type_of(dt);
  if (!t || !st || !count) return MPI_ERR_ARG;
  *count = t->size ? (st->bytes % t->size ? MPI_UNDEFINED : (int)(st->bytes / t->size)) : 0;
  return MPI_SUCCESS;
}
int MPI_Get_count(const MPI_Status *st, MPI_Datatype dt, int *count) ALIAS(MPI_Get_count);

/* ------------------------------------------------------------ type constructors */
#define OLD(h, var)                                                                                          \
  const Type *var = type_of(h);                                                                              \
  if (!var) return MPI_ERR_TYPE

int PMPI_Type_vector(int count, int bl, int stride, MPI_Datatype old, MPI_Datatype *out) {
  OLD(old, o);
  if (count < 0 || bl < 0 || !out) return MPI_ERR_ARG;
  Build b = {0};
  for (int64_t i = 0; i < count; ++i)
    for (int64_t j = 0; j < bl; ++j) push_type(&b, o, (i * stride + j) * o->extent);
  return finish(&b, out);
}
int MPI_Type_vector(int count, int bl, int stride, MPI_Datatype old, MPI_Datatype *out) ALIAS(MPI_Type_vector);

int PMPI_Type_contiguous(int count, MPI_Datatype old, MPI_Datatype *out) {
  return PMPI_Type_vector(count, 1, 1, old, out);
}
int MPI_Type_contiguous(int count, MPI_Datatype old, MPI_Datatype *out) ALIAS(MPI_Type_contiguous);

int PMPI_Type_create_hvector(int count, int bl, MPI_Aint stride, MPI_Datatype old, MPI_Datatype *out) {
  OLD(old, o);
  if (count < 0 || bl < 0 || !out) return MPI_ERR_ARG;
  Build b = {0};
  for (int64_t i = 0; i < count; ++i)
    for (int64_t j = 0; j < bl; ++j) push_type(&b, o, i * stride + j * o->extent);
  return finish(&b, out);
}
int MPI_Type_create_hvector(int count, int bl, MPI_Aint stride, MPI_Datatype old, MPI_Datatype *out)
    ALIAS(MPI_Type_create_hvector);

static int hindexed_impl(int count, const int *bl, int bl_const, const int64_t *disp_b, const int *disp_e,
                         MPI_Datatype old, MPI_Datatype *out) {
  OLD(old, o);
  if (count < 0 || !out) return MPI_ERR_ARG;
  Build b = {0};
  for (int64_t i = 0; i < count; ++i) {
    const int64_t n = bl ? bl[i] : bl_const;
    const int64_t d = disp_b ? disp_b[i] : (int64_t)disp_e[i] * o->extent;
    for (int64_t j = 0; j < n; ++j) push_type(&b, o, d + j * o->extent);
  }
  return finish(&b, out);
}

int PMPI_Type_indexed(int count, const int bl[], const int disp[], MPI_Datatype old, MPI_Datatype *out) {
  return hindexed_impl(count, bl, 0, NULL, disp, old, out);
}
int MPI_Type_indexed(int count, const int bl[], const int disp[], MPI_Datatype old, MPI_Datatype *out)
    ALIAS(MPI_Type_indexed);

int PMPI_Type_create_hindexed(int count, const int bl[], const MPI_Aint disp[], MPI_Datatype old,
                              MPI_Datatype *out) {
  return hindexed_impl(count, bl, 0, disp, NULL, old, out);
}
int MPI_Type_create_hindexed(int count, const int bl[], const MPI_Aint disp[], MPI_Datatype old, MPI_Datatype *out)
    ALIAS(MPI_Type_create_hindexed);

int PMPI_Type_create_indexed_block(int count, int bl, const int disp[], MPI_Datatype old, MPI_Datatype *out) {
  return hindexed_impl(count, NULL, bl, NULL, disp, old, out);
}
int MPI_Type_create_indexed_block(int count, int bl, const int disp[], MPI_Datatype old, MPI_Datatype *out)
    ALIAS(MPI_Type_create_indexed_block);

int PMPI_Type_create_hindexed_block(int count, int bl, const MPI_Aint disp[], MPI_Datatype old,
                                    MPI_Datatype *out) {
  return hindexed_impl(count, NULL, bl, disp, NULL, old, out);
}
int MPI_Type_create_hindexed_block(int count, int bl, const MPI_Aint disp[], MPI_Datatype old, MPI_Datatype *out)
    ALIAS(MPI_Type_create_hindexed_block);

int PMPI_Type_create_struct(int count, const int bl[], const MPI_Aint disp[], const MPI_Datatype types[],
                            MPI_Datatype *out) {
  if (count < 0 || !out) return MPI_ERR_ARG;
  Build b = {0};
  for (int64_t i = 0; i < count; ++i) {
    OLD(types[i], o);
    for (int64_t j = 0; j < bl[i]; ++j) push_type(&b, o, disp[i] + j * o->extent);
  }
  return finish(&b, out);
}
int MPI_Type_create_struct(int count, const int bl[], const MPI_Aint disp[], const MPI_Datatype types[],
                           MPI_Datatype *out) ALIAS(MPI_Type_create_struct);

int PMPI_Type_create_resized(MPI_Datatype old, MPI_Aint lb, MPI_Aint extent, MPI_Datatype *out) {
  OLD(old, o);
  if (!out) return MPI_ERR_ARG;
  Build b = {0};
  push_type(&b, o, 0);
  b.lb = lb;
  b.ub = lb + extent;
  return finish(&b, out);
}
int MPI_Type_create_resized(MPI_Datatype old, MPI_Aint lb, MPI_Aint extent, MPI_Datatype *out)
    ALIAS(MPI_Type_create_resized);

/* MPI-3.1 4.1.3: the typemap of the subarray, resized to [0, full array) */
int PMPI_Type_create_subarray(int nd, const int sizes[], const int subs[], const int starts[], int order,
                              MPI_Datatype old, MPI_Datatype *out) {
  OLD(old, o);
  if (nd < 1 || nd > 16 || !out || (order != MPI_ORDER_C && order != MPI_ORDER_FORTRAN)) return MPI_ERR_ARG;
  int64_t stride[16], idx[16] = {0}, full = o->extent, n = 1;
  /* dims listed fastest-last (C) or fastest-first (Fortran) */
  for (int k = 0; k < nd; ++k) {
    const int d = order == MPI_ORDER_C ? nd - 1 - k : k;
    if (subs[d] < 0 || starts[d] < 0 || starts[d] + subs[d] > sizes[d]) return MPI_ERR_ARG;
    stride[d] = full;
    full *= sizes[d];
    n *= subs[d];
  }
  Build b = {0};
  for (int64_t e = 0; e < n; ++e) {
    int64_t d0 = 0;
    for (int d = 0; d < nd; ++d) d0 += (starts[d] + idx[d]) * stride[d];
    push_type(&b, o, d0);
    for (int k = 0; k < nd; ++k) { /* odometer, fastest dimension first */
      const int d = order == MPI_ORDER_C ? nd - 1 - k : k;
      if (++idx[d] < subs[d]) break;
      idx[d] = 0;
    }
  }
  b.any = 1;
  b.lb = 0;
  b.ub = full;
  return finish(&b, out);
}
int MPI_Type_create_subarray(int nd, const int sizes[], const int subs[], const int starts[], int order,
                             MPI_Datatype old, MPI_Datatype *out) ALIAS(MPI_Type_create_subarray);

int PMPI_Type_commit(MPI_Datatype *dt) {
  Type *t = dt ? type_of(*dt) : NULL;
  if (!t) return MPI_ERR_TYPE;
  t->committed = 1;
  return MPI_SUCCESS;
}
int MPI_Type_commit(MPI_Datatype *dt) ALIAS(MPI_Type_commit);

int PMPI_Type_free(MPI_Datatype *dt) {
  Type *t = dt ? type_of(*dt) : NULL;
  if (!t || *dt <= MPI_UNSIGNED_CHAR) return MPI_ERR_TYPE;
  /* the run arrays are kept: a pending receive may still hold the type */
  t->used = 0;
  *dt = MPI_DATATYPE_NULL;
  return MPI_SUCCESS;
}
int MPI_Type_free(MPI_Datatype *dt) ALIAS(MPI_Type_free);

int PMPI_Type_size(MPI_Datatype dt, int *size) {
  OLD(dt, t);
  *size = (int)t->size;
  return MPI_SUCCESS;
}
int MPI_Type_size(MPI_Datatype dt, int *size) ALIAS(MPI_Type_size);

int PMPI_Type_get_extent(MPI_Datatype dt, MPI_Aint *lb, MPI_Aint *extent) {
  OLD(dt, t);
  *lb = t->lb;
  *extent = t->extent;
  return MPI_SUCCESS;
}
int MPI_Type_get_extent(MPI_Datatype dt, MPI_Aint *lb, MPI_Aint *extent) ALIAS(MPI_Type_get_extent);

/* ------------------------------------------------------------ packing */
int PMPI_Pack(const void *in, int incount, MPI_Datatype dt, void *out, int outsize, int *position, MPI_Comm comm) {
  OLD(dt, t);
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (!position || incount < 0) return MPI_ERR_ARG;
  if (!t->committed) return MPI_ERR_TYPE;
  if (*position + (int64_t)incount * t->size > outsize) return MPI_ERR_TRUNCATE;
  gather(t, in, incount, (uint8_t *)out + *position);
  *position += (int)(incount * t->size);
  return MPI_SUCCESS;
}
int MPI_Pack(const void *in, int incount, MPI_Datatype dt, void *out, int outsize, int *position, MPI_Comm comm)
    ALIAS(MPI_Pack);

int PMPI_Unpack(const void *in, int insize, int *position, void *out, int outcount, MPI_Datatype dt,
                MPI_Comm comm) {
  OLD(dt, t);
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (!position || outcount < 0) return MPI_ERR_ARG;
  if (!t->committed) return MPI_ERR_TYPE;
  if (*position + (int64_t)outcount * t->size > insize) return MPI_ERR_TRUNCATE;
  scatter(t, (const uint8_t *)in + *position, outcount, out);
  *position += (int)(outcount * t->size);
  return MPI_SUCCESS;
}
int MPI_Unpack(const void *in, int insize, int *position, void *out, int outcount, MPI_Datatype dt, MPI_Comm comm)
    ALIAS(MPI_Unpack);

int PMPI_Pack_size(int incount, MPI_Datatype dt, MPI_Comm comm, int *size) {
  OLD(dt, t);
  if (!comm_of(comm)) return MPI_ERR_COMM;
  *size = (int)(incount * t->size);
  return MPI_SUCCESS;
}
int MPI_Pack_size(int incount, MPI_Datatype dt, MPI_Comm comm, int *size) ALIAS(MPI_Pack_size);

/* ------------------------------------------------------------ point to point */
static int send_typed(const void *buf, int count, const Type *t, int wdest, int tag, int ctx) {
  const int64_t bytes = (int64_t)count * t->size;
  uint8_t *tmp = malloc(bytes ? (size_t)bytes : 1);
  gather(t, buf, count, tmp);
  const int rc = post(wdest, tag, ctx, tmp, bytes);
  free(tmp);
  return rc;
}

static int recv_typed(void *buf, int count, const Type *t, int wsrc, int tag, int ctx, MPI_Status *st) {
  Msg *m = fetch(wsrc, tag, ctx);
  int rc = MPI_SUCCESS;
  const int64_t cap = (int64_t)count * t->size;
  if (m->bytes > cap) {
    rc = MPI_ERR_TRUNCATE;
  } else if (t->size) {
    /* whole objects received, then the bytes of a partial last one */
    const int64_t whole = m->bytes / t->size;
    scatter(t, m->data, whole, buf);
    if (m->bytes % t->size) rc = MPI_ERR_TRUNCATE;
  }
  if (st) {
    st->MPI_SOURCE = m->src;
    st->MPI_TAG = m->tag;
    st->MPI_ERROR = rc;
    st->method = -1;
    st->bytes = m->bytes;
  }
  free(m->data);
  free(m);
  return rc;
}

int PMPI_Send(const void *buf, int count, MPI_Datatype dt, int dest, int tag, MPI_Comm comm) {
  OLD(dt, t);
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (dest == MPI_PROC_NULL) return MPI_SUCCESS;
  if (dest < 0 || dest >= (comm == MPI_COMM_SELF ? 1 : G.size)) return MPI_ERR_RANK;
  if (tag < 0) return MPI_ERR_TAG;
  if (count < 0) return MPI_ERR_COUNT;
  return send_typed(buf, count, t, world_rank(comm, dest), tag, ctx_of(comm));
}
int MPI_Send(const void *buf, int count, MPI_Datatype dt, int dest, int tag, MPI_Comm comm) ALIAS(MPI_Send);

int PMPI_Recv(void *buf, int count, MPI_Datatype dt, int source, int tag, MPI_Comm comm, MPI_Status *st) {
  OLD(dt, t);
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (source == MPI_PROC_NULL) {
    if (st) *st = (MPI_Status){MPI_PROC_NULL, MPI_ANY_TAG, MPI_SUCCESS, -1, 0};
    return MPI_SUCCESS;
  }
  if (count < 0) return MPI_ERR_COUNT;
  const int w = source == MPI_ANY_SOURCE ? MPI_ANY_SOURCE : world_rank(comm, source);
  return recv_typed(buf, count, t, w, tag, ctx_of(comm), st);
}
int MPI_Recv(void *buf, int count, MPI_Datatype dt, int source, int tag, MPI_Comm comm, MPI_Status *st)
    ALIAS(MPI_Recv);

/* requests: sends complete at once (eager); receives are matched at
 * MPI_Wait/MPI_Test */
typedef struct {
  int used, is_recv, count, src, tag, ctx;
  Type ty; /* a copy: the datatype may be freed while the receive is pending */
  void *buf;
  /* persistent requests (MPI_Send_init / MPI_Recv_init): recorded, started
   * by MPI_Start, inactive again once complete */
  int persistent, active;
  void *coll; /* a persistent neighbour collective (MPI-4): its arguments */
} Req;
static Req g_reqs[4096];

static int new_req(MPI_Request *r) {
  for (int i = 1; i < 4096; ++i)
    if (!g_reqs[i].used) {
      memset(&g_reqs[i], 0, sizeof(Req));
      g_reqs[i].used = 1;
      *r = i;
      return MPI_SUCCESS;
    }
  return MPI_ERR_OTHER;
}

int PMPI_Isend(const void *buf, int count, MPI_Datatype dt, int dest, int tag, MPI_Comm comm, MPI_Request *r) {
  if (!r) return MPI_ERR_ARG;
  *r = MPI_REQUEST_NULL;
  const int rc = PMPI_Send(buf, count, dt, dest, tag, comm);
  if (rc != MPI_SUCCESS || dest == MPI_PROC_NULL) return rc;
  return new_req(r);
}
int MPI_Isend(const void *buf, int count, MPI_Datatype dt, int dest, int tag, MPI_Comm comm, MPI_Request *r)
    ALIAS(MPI_Isend);

int PMPI_Irecv(void *buf, int count, MPI_Datatype dt, int source, int tag, MPI_Comm comm, MPI_Request *r) {
  if (!r) return MPI_ERR_ARG;
  *r = MPI_REQUEST_NULL;
  if (!type_of(dt)) return MPI_ERR_TYPE;
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (source == MPI_PROC_NULL) return MPI_SUCCESS;
  if (count < 0) return MPI_ERR_COUNT;
  const int rc = new_req(r);
  if (rc != MPI_SUCCESS) return rc;
  Req *q = &g_reqs[*r];
  q->is_recv = 1;
  q->count = count;
  q->src = source == MPI_ANY_SOURCE ? MPI_ANY_SOURCE : world_rank(comm, source);
  q->tag = tag;
  q->ctx = ctx_of(comm);
  q->ty = *type_of(dt);
  q->buf = buf;
  return MPI_SUCCESS;
}
int MPI_Irecv(void *buf, int count, MPI_Datatype dt, int source, int tag, MPI_Comm comm, MPI_Request *r)
    ALIAS(MPI_Irecv);

static int complete(MPI_Request *r, MPI_Status *st, int block, int *flag) {
  if (!r) return MPI_ERR_ARG;
  if (flag) *flag = 1;
  if (*r == MPI_REQUEST_NULL) {
    if (st) *st = (MPI_Status){MPI_ANY_SOURCE, MPI_ANY_TAG, MPI_SUCCESS, -1, 0};
    return MPI_SUCCESS;
  }
  if (*r < 0 || *r >= 4096 || !g_reqs[*r].used) return MPI_ERR_ARG;
  Req *q = &g_reqs[*r];
  int rc = MPI_SUCCESS;
  if (q->persistent && !q->active) { /* inactive: complete, empty status */
    if (st) *st = (MPI_Status){MPI_ANY_SOURCE, MPI_ANY_TAG, MPI_SUCCESS, -1, 0};
    return MPI_SUCCESS;
  }
  if (q->is_recv) {
    if (!block) {
      pthread_mutex_lock(&g_mu);
      const int ready = match_locked(q->src, q->tag, q->ctx, 0) != NULL;
      pthread_mutex_unlock(&g_mu);
      if (!ready) {
        if (flag) *flag = 0;
        return MPI_SUCCESS;
      }
    }
    rc = recv_typed(q->buf, q->count, &q->ty, q->src, q->tag, q->ctx, st);
  } else if (st) {
    *st = (MPI_Status){MPI_ANY_SOURCE, MPI_ANY_TAG, MPI_SUCCESS, -1, 0};
  }
  if (q->persistent) {
    q->active = 0;
  } else {
    q->used = 0;
    *r = MPI_REQUEST_NULL;
  }
  return rc;
}

int PMPI_Wait(MPI_Request *r, MPI_Status *st) { return complete(r, st, 1, NULL); }
int MPI_Wait(MPI_Request *r, MPI_Status *st) ALIAS(MPI_Wait);

int PMPI_Test(MPI_Request *r, int *flag, MPI_Status *st) { return complete(r, st, 0, flag); }
int MPI_Test(MPI_Request *r, int *flag, MPI_Status *st) ALIAS(MPI_Test);

int PMPI_Waitall(int n, MPI_Request rs[], MPI_Status sts[]) {
  int first = MPI_SUCCESS;
  for (int i = 0; i < n; ++i) {
    const int rc = complete(&rs[i], sts ? &sts[i] : NULL, 1, NULL);
    if (rc != MPI_SUCCESS && first == MPI_SUCCESS) first = rc;
  }
  return first;
}
int MPI_Waitall(int n, MPI_Request rs[], MPI_Status sts[]) ALIAS(MPI_Waitall);

static int inactive(MPI_Request r) {
  return r == MPI_REQUEST_NULL || (g_reqs[r].persistent && !g_reqs[r].active);
}

static int all_null(int n, const MPI_Request r[]) {
  for (int i = 0; i < n; ++i)
    if (!inactive(r[i])) return 0;
  return 1;
}

int PMPI_Testany(int n, MPI_Request rs[], int *index, int *flag, MPI_Status *st) {
  *index = MPI_UNDEFINED;
  *flag = 0;
  if (all_null(n, rs)) {
    *flag = 1;
    if (st) *st = (MPI_Status){MPI_ANY_SOURCE, MPI_ANY_TAG, MPI_SUCCESS, -1, 0};
    return MPI_SUCCESS;
  }
  for (int i = 0; i < n; ++i) {
    if (inactive(rs[i])) continue;
    int done = 0;
    const int rc = complete(&rs[i], st, 0, &done);
    if (rc != MPI_SUCCESS || done) {
      *index = i;
      *flag = 1;
      return rc;
    }
  }
  return MPI_SUCCESS;
}
int MPI_Testany(int n, MPI_Request rs[], int *index, int *flag, MPI_Status *st) ALIAS(MPI_Testany);

int PMPI_Waitany(int n, MPI_Request rs[], int *index, MPI_Status *st) {
  for (;;) {
    int flag = 0;
    const int rc = PMPI_Testany(n, rs, index, &flag, st);
    if (rc != MPI_SUCCESS || flag) return rc;
    pthread_mutex_lock(&g_mu); /* wait for the next arrival rather than spin */
    struct timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    ts.tv_nsec += 1000000;
    if (ts.tv_nsec >= 1000000000) {
      ts.tv_sec += 1;
      ts.tv_nsec -= 1000000000;
    }
    pthread_cond_timedwait(&g_cv, &g_mu, &ts);
    pthread_mutex_unlock(&g_mu);
  }
}
int MPI_Waitany(int n, MPI_Request rs[], int *index, MPI_Status *st) ALIAS(MPI_Waitany);

int PMPI_Testall(int n, MPI_Request rs[], int *flag, MPI_Status sts[]) {
  /* all or nothing (MPI-3.1 3.7.5): complete only when every one can */
  for (int i = 0; i < n; ++i) {
    if (inactive(rs[i]) || !g_reqs[rs[i]].is_recv) continue;
    const Req *q = &g_reqs[rs[i]];
    pthread_mutex_lock(&g_mu);
    const int ready = match_locked(q->src, q->tag, q->ctx, 0) != NULL;
    pthread_mutex_unlock(&g_mu);
    if (!ready) {
      *flag = 0;
      return MPI_SUCCESS;
    }
  }
  *flag = 1;
  return PMPI_Waitall(n, rs, sts);
}
int MPI_Testall(int n, MPI_Request rs[], int *flag, MPI_Status sts[]) ALIAS(MPI_Testall);

int PMPI_Waitsome(int n, MPI_Request rs[], int *outcount, int indices[], MPI_Status sts[]) {
  if (all_null(n, rs)) {
    *outcount = MPI_UNDEFINED;
    return MPI_SUCCESS;
  }
  int index = 0;
  const int rc = PMPI_Waitany(n, rs, &index, sts ? &sts[0] : NULL);
  indices[0] = index;
  *outcount = 1;
  return rc;
}
int MPI_Waitsome(int n, MPI_Request rs[], int *outcount, int indices[], MPI_Status sts[]) ALIAS(MPI_Waitsome);

int PMPI_Request_free(MPI_Request *r) {
  if (!r || *r == MPI_REQUEST_NULL) return MPI_ERR_ARG;
  const int rc = complete(r, NULL, 1, NULL);
  if (*r != MPI_REQUEST_NULL) { /* persistent: released here */
    free(g_reqs[*r].coll);
    g_reqs[*r].coll = NULL;
    g_reqs[*r].used = 0;
    *r = MPI_REQUEST_NULL;
  }
  return rc;
}

/* persistent requests: a send starts eagerly (like MPI_Isend), a receive is
 * matched at completion */
static int persist(int is_recv, void *buf, int count, MPI_Datatype dt, int peer, int tag, MPI_Comm comm,
                   MPI_Request *r) {
  if (!r || !type_of(dt)) return MPI_ERR_ARG;
  if (!comm_of(comm)) return MPI_ERR_COMM;
  const int rc = new_req(r);
  if (rc != MPI_SUCCESS) return rc;
  Req *q = &g_reqs[*r];
  q->persistent = 1;
  q->is_recv = is_recv;
  q->count = count;
  q->src = peer == MPI_ANY_SOURCE || peer == MPI_PROC_NULL ? peer : world_rank(comm, peer);
  q->tag = tag;
  q->ctx = ctx_of(comm);
  q->ty = *type_of(dt);
  q->buf = buf;
  return MPI_SUCCESS;
}

int PMPI_Send_init(const void *buf, int count, MPI_Datatype dt, int dest, int tag, MPI_Comm comm, MPI_Request *r) {
  return persist(0, (void *)buf, count, dt, dest, tag, comm, r);
}
int MPI_Send_init(const void *buf, int count, MPI_Datatype dt, int dest, int tag, MPI_Comm comm, MPI_Request *r)
    ALIAS(MPI_Send_init);

int PMPI_Recv_init(void *buf, int count, MPI_Datatype dt, int source, int tag, MPI_Comm comm, MPI_Request *r) {
  return persist(1, buf, count, dt, source, tag, comm, r);
}
int MPI_Recv_init(void *buf, int count, MPI_Datatype dt, int source, int tag, MPI_Comm comm, MPI_Request *r)
    ALIAS(MPI_Recv_init);

static int coll_start(void *coll);

int PMPI_Start(MPI_Request *r) {
  if (!r || *r <= 0 || *r >= 4096 || !g_reqs[*r].used || !g_reqs[*r].persistent || g_reqs[*r].active)
    return MPI_ERR_ARG;
  Req *q = &g_reqs[*r];
  if (q->coll) { /* a persistent collective runs at its start (blocking) */
    const int rc = coll_start(q->coll);
    if (rc == MPI_SUCCESS) q->active = 1;
    return rc;
  }
  if (q->src == MPI_PROC_NULL) return MPI_SUCCESS;
  if (!q->is_recv) {
    const int rc = send_typed(q->buf, q->count, &q->ty, q->src, q->tag, q->ctx);
    if (rc != MPI_SUCCESS) return rc;
  }
  q->active = 1;
  return MPI_SUCCESS;
}
int MPI_Start(MPI_Request *r) ALIAS(MPI_Start);

int PMPI_Startall(int n, MPI_Request rs[]) {
  for (int i = 0; i < n; ++i) {
    const int rc = PMPI_Start(&rs[i]);
    if (rc != MPI_SUCCESS) return rc;
  }
  return MPI_SUCCESS;
}
int MPI_Startall(int n, MPI_Request rs[]) ALIAS(MPI_Startall);
int MPI_Request_free(MPI_Request *r) ALIAS(MPI_Request_free);

int PMPI_Sendrecv(const void *sbuf, int scount, MPI_Datatype stype, int dest, int stag, void *rbuf, int rcount,
                  MPI_Datatype rtype, int source, int rtag, MPI_Comm comm, MPI_Status *st) {
  const int rc = PMPI_Send(sbuf, scount, stype, dest, stag, comm);
  if (rc != MPI_SUCCESS) return rc;
  return PMPI_Recv(rbuf, rcount, rtype, source, rtag, comm, st);
}
int MPI_Sendrecv(const void *sbuf, int scount, MPI_Datatype stype, int dest, int stag, void *rbuf, int rcount,
                 MPI_Datatype rtype, int source, int rtag, MPI_Comm comm, MPI_Status *st) ALIAS(MPI_Sendrecv);

/* ------------------------------------------------------------ topologies */
static int new_comm(Comm *c, MPI_Comm *out) {
  if (G.ncomms == 256) return MPI_ERR_OTHER;
  c->used = 1;
  G.comms[G.ncomms] = *c;
  *out = 100 + G.ncomms++;
  return MPI_SUCCESS;
}

static int *dup_ints(const int *a, int n) {
  int *p = malloc(sizeof(int) * (n ? n : 1));
  if (n) memcpy(p, a, sizeof(int) * n);
  return p;
}

int PMPI_Dist_graph_create_adjacent(MPI_Comm old, int indeg, const int sources[], const int *sw, int outdeg,
                                    const int dests[], const int *dw, MPI_Info info, int reorder, MPI_Comm *out) {
  (void)sw;
  (void)dw;
  (void)info;
  (void)reorder;
  if (!comm_of(old) || !out || indeg < 0 || outdeg < 0) return MPI_ERR_ARG;
  for (int i = 0; i < indeg; ++i)
    if ((sources[i] < 0 || sources[i] >= G.size) && sources[i] != MPI_PROC_NULL) return MPI_ERR_RANK;
  for (int i = 0; i < outdeg; ++i)
    if ((dests[i] < 0 || dests[i] >= G.size) && dests[i] != MPI_PROC_NULL) return MPI_ERR_RANK;
  Comm c = {0};
  c.kind = 1;
  c.nsrc = indeg;
  c.ndst = outdeg;
  c.src = dup_ints(sources, indeg);
  c.dst = dup_ints(dests, outdeg);
  return new_comm(&c, out);
}
int MPI_Dist_graph_create_adjacent(MPI_Comm old, int indeg, const int sources[], const int *sw, int outdeg,
                                   const int dests[], const int *dw, MPI_Info info, int reorder, MPI_Comm *out)
    ALIAS(MPI_Dist_graph_create_adjacent);

int PMPI_Dist_graph_neighbors_count(MPI_Comm comm, int *indeg, int *outdeg, int *weighted) {
  const Comm *c = comm_of(comm);
  if (!c) return MPI_ERR_COMM;
  *indeg = c->nsrc;
  *outdeg = c->ndst;
  if (weighted) *weighted = 0;
  return MPI_SUCCESS;
}
int MPI_Dist_graph_neighbors_count(MPI_Comm comm, int *indeg, int *outdeg, int *weighted)
    ALIAS(MPI_Dist_graph_neighbors_count);

int PMPI_Dist_graph_neighbors(MPI_Comm comm, int maxin, int sources[], int *sw, int maxout, int dests[], int *dw) {
  (void)sw;
  (void)dw;
  const Comm *c = comm_of(comm);
  if (!c) return MPI_ERR_COMM;
  for (int i = 0; i < maxin && i < c->nsrc; ++i) sources[i] = c->src[i];
  for (int i = 0; i < maxout && i < c->ndst; ++i) dests[i] = c->dst[i];
  return MPI_SUCCESS;
}
int MPI_Dist_graph_neighbors(MPI_Comm comm, int maxin, int sources[], int *sw, int maxout, int dests[], int *dw)
    ALIAS(MPI_Dist_graph_neighbors);

static int cart_rank(const Comm *c, const int *co) {
  int r = 0;
  for (int d = 0; d < c->ndims; ++d) {
    int x = co[d];
    if (c->periods[d]) x = ((x % c->dims[d]) + c->dims[d]) % c->dims[d];
    else if (x < 0 || x >= c->dims[d]) return MPI_PROC_NULL;
    r = r * c->dims[d] + x;
  }
  return r;
}

static void cart_coords(const Comm *c, int rank, int *co) {
  for (int d = c->ndims - 1; d >= 0; --d) {
    co[d] = rank % c->dims[d];
    rank /= c->dims[d];
  }
}

int PMPI_Cart_create(MPI_Comm old, int nd, const int dims[], const int periods[], int reorder, MPI_Comm *out) {
  (void)reorder;
  if (!comm_of(old) || !out || nd < 1 || nd > 16) return MPI_ERR_ARG;
  int n = 1;
  for (int d = 0; d < nd; ++d) n *= dims[d];
  if (n != G.size) return MPI_ERR_ARG;
  Comm c = {0};
  c.kind = 2;
  c.ndims = nd;
  c.dims = dup_ints(dims, nd);
  c.periods = dup_ints(periods, nd);
  /* neighbour order: per dimension, the -1 then the +1 neighbour */
  c.nsrc = c.ndst = 2 * nd;
  c.src = malloc(sizeof(int) * 2 * nd);
  c.dst = malloc(sizeof(int) * 2 * nd);
  int co[16];
  for (int d = 0; d < nd; ++d)
    for (int s = 0; s < 2; ++s) {
      cart_coords(&c, G.rank, co);
      co[d] += s ? 1 : -1;
      c.src[2 * d + s] = c.dst[2 * d + s] = cart_rank(&c, co);
    }
  return new_comm(&c, out);
}
int MPI_Cart_create(MPI_Comm old, int nd, const int dims[], const int periods[], int reorder, MPI_Comm *out)
    ALIAS(MPI_Cart_create);

int PMPI_Cart_coords(MPI_Comm comm, int rank, int maxdims, int coords[]) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind != 2 || maxdims < c->ndims) return MPI_ERR_COMM;
  cart_coords(c, rank, coords);
  return MPI_SUCCESS;
}
int MPI_Cart_coords(MPI_Comm comm, int rank, int maxdims, int coords[]) ALIAS(MPI_Cart_coords);

int PMPI_Cart_rank(MPI_Comm comm, const int coords[], int *rank) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind != 2) return MPI_ERR_COMM;
  *rank = cart_rank(c, coords);
  return MPI_SUCCESS;
}
int MPI_Cart_rank(MPI_Comm comm, const int coords[], int *rank) ALIAS(MPI_Cart_rank);

int PMPI_Cart_shift(MPI_Comm comm, int dir, int disp, int *src, int *dst) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind != 2 || dir < 0 || dir >= c->ndims) return MPI_ERR_COMM;
  int co[16];
  cart_coords(c, G.rank, co);
  co[dir] -= disp;
  *src = cart_rank(c, co);
  co[dir] += 2 * disp;
  *dst = cart_rank(c, co);
  return MPI_SUCCESS;
}
int MPI_Cart_shift(MPI_Comm comm, int dir, int disp, int *src, int *dst) ALIAS(MPI_Cart_shift);

int PMPI_Comm_free(MPI_Comm *comm) {
  Comm *c = comm ? comm_of(*comm) : NULL;
  if (!c || *comm < 100) return MPI_ERR_COMM;
  free(c->src);
  free(c->dst);
  free(c->dims);
  free(c->periods);
  c->used = 0;
  *comm = MPI_COMM_NULL;
  return MPI_SUCCESS;
}
int MPI_Comm_free(MPI_Comm *comm) ALIAS(MPI_Comm_free);

/* ------------------------------------------------------------ neighbourhood collectives */
/* the k-th edge to (from) a given peer carries tag k */
static int occurrence(const int *ranks, int i) {
  int k = 0;
  for (int j = 0; j < i; ++j) k += ranks[j] == ranks[i];
  return k;
}

static int nbr_exchange(const void *sbuf, const int scounts[], const int64_t sdisp_b[], const MPI_Datatype stypes[],
                        void *rbuf, const int rcounts[], const int64_t rdisp_b[], const MPI_Datatype rtypes[],
                        MPI_Comm comm) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind == 0) return MPI_ERR_COMM;
  const int ctx = ctx_of(comm) + 1;
  for (int i = 0; i < c->ndst; ++i) {
    if (c->dst[i] == MPI_PROC_NULL) continue;
    const Type *t = type_of(stypes[i]);
    if (!t) return MPI_ERR_TYPE;
    const int rc = send_typed((const uint8_t *)sbuf + sdisp_b[i], scounts[i], t, c->dst[i],
                              occurrence(c->dst, i), ctx);
    if (rc != MPI_SUCCESS) return rc;
  }
  for (int j = 0; j < c->nsrc; ++j) {
    if (c->src[j] == MPI_PROC_NULL) continue;
    const Type *t = type_of(rtypes[j]);
    if (!t) return MPI_ERR_TYPE;
    const int rc = recv_typed((uint8_t *)rbuf + rdisp_b[j], rcounts[j], t, c->src[j], occurrence(c->src, j),
                              ctx, NULL);
    if (rc != MPI_SUCCESS) return rc;
  }
  return MPI_SUCCESS;
}

int PMPI_Neighbor_alltoallv(const void *sbuf, const int scounts[], const int sdispls[], MPI_Datatype stype,
                            void *rbuf, const int rcounts[], const int rdispls[], MPI_Datatype rtype,
                            MPI_Comm comm) {
  const Comm *c = comm_of(comm);
  const Type *st = type_of(stype), *rt = type_of(rtype);
  if (!c) return MPI_ERR_COMM;
  if (!st || !rt) return MPI_ERR_TYPE;
  const int n = c->ndst > c->nsrc ? c->ndst : c->nsrc;
  int64_t *sd = malloc(sizeof(int64_t) * (n + 1)), *rd = malloc(sizeof(int64_t) * (n + 1));
  MPI_Datatype *sts = malloc(sizeof(MPI_Datatype) * (n + 1)), *rts = malloc(sizeof(MPI_Datatype) * (n + 1));
  for (int i = 0; i < c->ndst; ++i) {
    sd[i] = (int64_t)sdispls[i] * st->extent;
    sts[i] = stype;
  }
  for (int j = 0; j < c->nsrc; ++j) {
    rd[j] = (int64_t)rdispls[j] * rt->extent;
    rts[j] = rtype;
  }
  const int rc = nbr_exchange(sbuf, scounts, sd, sts, rbuf, rcounts, rd, rts, comm);
  free(sd);
  free(rd);
  free(sts);
  free(rts);
  return rc;
}
int MPI_Neighbor_alltoallv(const void *sbuf, const int scounts[], const int sdispls[], MPI_Datatype stype,
                           void *rbuf, const int rcounts[], const int rdispls[], MPI_Datatype rtype, MPI_Comm comm)
    ALIAS(MPI_Neighbor_alltoallv);

int PMPI_Neighbor_alltoallw(const void *sbuf, const int scounts[], const MPI_Aint sdispls[],
                            const MPI_Datatype stypes[], void *rbuf, const int rcounts[], const MPI_Aint rdispls[],
                            const MPI_Datatype rtypes[], MPI_Comm comm) {
  return nbr_exchange(sbuf, scounts, sdispls, stypes, rbuf, rcounts, rdispls, rtypes, comm);
}
int MPI_Neighbor_alltoallw(const void *sbuf, const int scounts[], const MPI_Aint sdispls[],
                           const MPI_Datatype stypes[], void *rbuf, const int rcounts[], const MPI_Aint rdispls[],
                           const MPI_Datatype rtypes[], MPI_Comm comm) ALIAS(MPI_Neighbor_alltoallw);

/* ------------------------------------------------------------ all-to-all (MPI-3.1 5.8) */
#define A2A_TAG (1 << 30) /* apart from the neighbour collectives' occurrence tags */

static int a2a(const void *sbuf, const int scounts[], const int64_t sdisp_b[], const MPI_Datatype stypes[],
               void *rbuf, const int rcounts[], const int64_t rdisp_b[], const MPI_Datatype rtypes[], MPI_Comm comm) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  const int n = comm == MPI_COMM_SELF ? 1 : G.size, ctx = ctx_of(comm) + 1;
  for (int i = 0; i < n; ++i) {
    const Type *t = type_of(stypes[i]);
    if (!t) return MPI_ERR_TYPE;
    const int rc = send_typed((const uint8_t *)sbuf + sdisp_b[i], scounts[i], t, world_rank(comm, i), A2A_TAG, ctx);
    if (rc != MPI_SUCCESS) return rc;
  }
  for (int j = 0; j < n; ++j) {
    const Type *t = type_of(rtypes[j]);
    if (!t) return MPI_ERR_TYPE;
    const int rc = recv_typed((uint8_t *)rbuf + rdisp_b[j], rcounts[j], t, world_rank(comm, j), A2A_TAG, ctx, NULL);
    if (rc != MPI_SUCCESS) return rc;
  }
  return MPI_SUCCESS;
}

int PMPI_Alltoallv(const void *sbuf, const int scounts[], const int sdispls[], MPI_Datatype stype, void *rbuf,
                   const int rcounts[], const int rdispls[], MPI_Datatype rtype, MPI_Comm comm) {
  const Type *st = type_of(stype), *rt = type_of(rtype);
  if (!st || !rt) return MPI_ERR_TYPE;
  const int n = comm == MPI_COMM_SELF ? 1 : G.size;
  int64_t *sd = malloc(sizeof(int64_t) * n), *rd = malloc(sizeof(int64_t) * n);
  MPI_Datatype *sts = malloc(sizeof(MPI_Datatype) * n), *rts = malloc(sizeof(MPI_Datatype) * n);
  for (int i = 0; i < n; ++i) {
    sd[i] = (int64_t)sdispls[i] * st->extent;
    rd[i] = (int64_t)rdispls[i] * rt->extent;
    sts[i] = stype;
    rts[i] = rtype;
  }
  const int rc = a2a(sbuf, scounts, sd, sts, rbuf, rcounts, rd, rts, comm);
  free(sd);
  free(rd);
  free(sts);
  free(rts);
  return rc;
}
int MPI_Alltoallv(const void *sbuf, const int scounts[], const int sdispls[], MPI_Datatype stype, void *rbuf,
                  const int rcounts[], const int rdispls[], MPI_Datatype rtype, MPI_Comm comm) ALIAS(MPI_Alltoallv);

int PMPI_Alltoallw(const void *sbuf, const int scounts[], const int sdispls[], const MPI_Datatype stypes[],
                   void *rbuf, const int rcounts[], const int rdispls[], const MPI_Datatype rtypes[], MPI_Comm comm) {
  const int n = comm == MPI_COMM_SELF ? 1 : G.size;
  int64_t *sd = malloc(sizeof(int64_t) * n), *rd = malloc(sizeof(int64_t) * n);
  for (int i = 0; i < n; ++i) {
    sd[i] = sdispls[i];
    rd[i] = rdispls[i];
  }
  const int rc = a2a(sbuf, scounts, sd, stypes, rbuf, rcounts, rd, rtypes, comm);
  free(sd);
  free(rd);
  return rc;
}
int MPI_Alltoallw(const void *sbuf, const int scounts[], const int sdispls[], const MPI_Datatype stypes[],
                  void *rbuf, const int rcounts[], const int rdispls[], const MPI_Datatype rtypes[], MPI_Comm comm)
    ALIAS(MPI_Alltoallw);

/* ------------------------------------------------------------ persistent neighbour collective (MPI-4.0 7.10.2) */
typedef struct {
  const void *sbuf;
  void *rbuf;
  MPI_Comm comm;
  int n_out, n_in;
  int *scounts, *rcounts;
  int64_t *sd, *rd;
  MPI_Datatype *st, *rt;
} Coll;

static int coll_start(void *p) {
  Coll *c = p;
  return nbr_exchange(c->sbuf, c->scounts, c->sd, c->st, c->rbuf, c->rcounts, c->rd, c->rt, c->comm);
}

int PMPI_Neighbor_alltoallw_init(const void *sbuf, const int scounts[], const MPI_Aint sdispls[],
                                 const MPI_Datatype stypes[], void *rbuf, const int rcounts[],
                                 const MPI_Aint rdispls[], const MPI_Datatype rtypes[], MPI_Comm comm, MPI_Info info,
                                 MPI_Request *r) {
  (void)info;
  const Comm *cm = comm_of(comm);
  if (!cm || cm->kind == 0) return MPI_ERR_COMM;
  if (!r) return MPI_ERR_ARG;
  const int no = cm->ndst, ni = cm->nsrc;
  /* one allocation: the struct, then its arrays */
  const size_t bytes = sizeof(Coll) + (size_t)(no + ni) * (sizeof(int) + sizeof(int64_t) + sizeof(MPI_Datatype));
  Coll *c = calloc(1, bytes);
  uint8_t *at = (uint8_t *)(c + 1);
  c->sd = (int64_t *)at;
  c->rd = c->sd + no;
  c->scounts = (int *)(c->rd + ni);
  c->rcounts = c->scounts + no;
  c->st = (MPI_Datatype *)(c->rcounts + ni);
  c->rt = c->st + no;
  c->sbuf = sbuf;
  c->rbuf = rbuf;
  c->comm = comm;
  c->n_out = no;
  c->n_in = ni;
  for (int i = 0; i < no; ++i) {
    c->sd[i] = sdispls[i];
    c->scounts[i] = scounts[i];
    c->st[i] = stypes[i];
  }
  for (int j = 0; j < ni; ++j) {
    c->rd[j] = rdispls[j];
    c->rcounts[j] = rcounts[j];
    c->rt[j] = rtypes[j];
  }
  const int rc = new_req(r);
  if (rc != MPI_SUCCESS) {
    free(c);
    return rc;
  }
  g_reqs[*r].persistent = 1;
  g_reqs[*r].coll = c;
  return MPI_SUCCESS;
}
int MPI_Neighbor_alltoallw_init(const void *sbuf, const int scounts[], const MPI_Aint sdispls[],
                                const MPI_Datatype stypes[], void *rbuf, const int rcounts[], const MPI_Aint rdispls[],
                                const MPI_Datatype rtypes[], MPI_Comm comm, MPI_Info info, MPI_Request *r)
    ALIAS(MPI_Neighbor_alltoallw_init);

int PMPI_Neighbor_alltoallv_init(const void *sbuf, const int scounts[], const int sdispls[], MPI_Datatype stype,
                                 void *rbuf, const int rcounts[], const int rdispls[], MPI_Datatype rtype,
                                 MPI_Comm comm, MPI_Info info, MPI_Request *r) {
  const Comm *cm = comm_of(comm);
  const Type *st = type_of(stype), *rt = type_of(rtype);
  if (!cm || cm->kind == 0) return MPI_ERR_COMM;
  if (!st || !rt) return MPI_ERR_TYPE;
  const int no = cm->ndst, ni = cm->nsrc;
  MPI_Aint *sd = malloc(sizeof(MPI_Aint) * (no + 1)), *rd = malloc(sizeof(MPI_Aint) * (ni + 1));
  MPI_Datatype *sts = malloc(sizeof(MPI_Datatype) * (no + 1)), *rts = malloc(sizeof(MPI_Datatype) * (ni + 1));
  for (int i = 0; i < no; ++i) {
    sd[i] = (MPI_Aint)sdispls[i] * st->extent;
    sts[i] = stype;
  }
  for (int j = 0; j < ni; ++j) {
    rd[j] = (MPI_Aint)rdispls[j] * rt->extent;
    rts[j] = rtype;
  }
  const int rc = PMPI_Neighbor_alltoallw_init(sbuf, scounts, sd, sts, rbuf, rcounts, rd, rts, comm, info, r);
  free(sd);
  free(rd);
  free(sts);
  free(rts);
  return rc;
}
int MPI_Neighbor_alltoallv_init(const void *sbuf, const int scounts[], const int sdispls[], MPI_Datatype stype,
                                void *rbuf, const int rcounts[], const int rdispls[], MPI_Datatype rtype, MPI_Comm comm,
                                MPI_Info info, MPI_Request *r) ALIAS(MPI_Neighbor_alltoallv_init);
