// tempi.cpp -- the MPI surface (libtempi_b200.so), include/mpi.h.
//
// TEMPI's interposer exports MPI_* and forwards what it does not accelerate
// to the system MPI through PMPI_* (PAPER.md:781-796). Here MPI_* is the
// accelerated layer (datatypes canonicalised at MPI_Type_commit, sm_100a
// pack/unpack kernels, model-selected transfers, fused pack-to-peer
// neighbour exchange) and PMPI_* the base layer over the node-local runtime
// (rt.cpp), since the image ships no MPI library.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "mpi.h"
#include "stridepack_b200.h"

namespace {

struct Comm {
  int kind = 0; // 0 world/self, 1 dist graph, 2 cartesian
  std::vector<int> sources, dests;
  std::vector<int> dims, periods;
};

struct State {
  bool initialized = false, finalized = false;
  int rank = 0, size = 1, device = -1;
  std::unordered_map<int, sp_type> types; // MPI handle -> engine handle
  int next_type = 100;
  std::unordered_map<int, Comm> comms;
  int next_comm = 100;
  int forced_method = -1;
  // MPI_Request -> engine request, and its outcome once the engine reported
  // it complete but the MPI handle has not been released yet (MPI_Testall
  // must leave every request untouched until all are done)
  struct Pending {
    sp_request r = 0;
    bool done = false;
    sp_status rc = SP_OK;
    int64_t st[4] = {0, 0, 0, 0};
    // persistent requests (MPI_Send_init / MPI_Recv_init, MPI-3.1 3.9): the
    // operation's arguments, and whether a started one is in flight
    bool persistent = false, active = false, is_send = false;
    const void *buf = nullptr;
    int count = 0, peer = 0, tag = 0;
    MPI_Datatype dt = 0;
    MPI_Comm comm = 0;
    // persistent neighbour collective (MPI-4 MPI_Neighbor_alltoallw_init):
    // the engine's compiled plan, or -- types it cannot compile -- the call
    // itself, re-run by every start
    sp_nbr_plan plan = nullptr;
    std::shared_ptr<std::function<sp_status()>> rerun;
  };
  std::unordered_map<int, Pending> requests;
  int next_request = 1;
  sp_profile profile = nullptr;
  cudaStream_t stream = nullptr;
  std::mutex mu;
};

State &S() {
  static State s;
  return s;
}

int to_mpi(sp_status st) {
  switch (st) {
  case SP_OK: return MPI_SUCCESS;
  case SP_ERR_INVALID_ARGUMENT: return MPI_ERR_ARG;
  case SP_ERR_UNSUPPORTED_ORDER: return MPI_ERR_ARG;
  case SP_ERR_INVALID_LAYOUT: return MPI_ERR_TYPE;
  case SP_ERR_BUFFER_TOO_SMALL: return MPI_ERR_TRUNCATE;
  case SP_ERR_OVERLAPPING_LAYOUT: return MPI_ERR_TYPE;
  case SP_ERR_UNSUPPORTED: return MPI_ERR_UNSUPPORTED_OPERATION;
  case SP_ERR_INVALID_HANDLE: return MPI_ERR_TYPE;
  case SP_ERR_TIMEOUT: return MPI_ERR_OTHER;
  default: return MPI_ERR_INTERN;
  }
}

#define TRY(expr)                                                                                                \
  do {                                                                                                           \
    const sp_status _st = (expr);                                                                                \
    if (_st != SP_OK) {                                                                                          \
      if (std::getenv("TEMPI_VERBOSE")) std::fprintf(stderr, "tempi: %s: %s\n", #expr, sp_last_error());        \
      return to_mpi(_st);                                                                                        \
    }                                                                                                            \
  } while (0)

int env_int(const char *a, const char *b, const char *c, int dflt) {
  for (const char *k : {a, b, c}) {
    if (!k) continue;
    if (const char *v = std::getenv(k)) return std::atoi(v);
  }
  return dflt;
}

// engine handle of an MPI datatype
bool lookup(MPI_Datatype t, sp_type *out) {
  auto it = S().types.find(t);
  if (it == S().types.end()) return false;
  *out = it->second;
  return true;
}

#define TYPE(t, var)                                                                                             \
  sp_type var;                                                                                                   \
  if (!lookup((t), &var)) return MPI_ERR_TYPE

int new_type(sp_type h, MPI_Datatype *out) {
  if (!out) return MPI_ERR_ARG;
  std::lock_guard<std::mutex> lk(S().mu);
  const int id = S().next_type++;
  S().types[id] = h;
  *out = id;
  return MPI_SUCCESS;
}

const Comm *comm_of(MPI_Comm c) {
  if (c == MPI_COMM_WORLD || c == MPI_COMM_SELF) {
    static Comm world;
    return &world;
  }
  auto it = S().comms.find(c);
  return it == S().comms.end() ? nullptr : &it->second;
}

std::string default_profile_path() {
  Dl_info info{};
  if (dladdr(reinterpret_cast<void *>(&default_profile_path), &info) && info.dli_fname) {
    std::string p(info.dli_fname);
    const auto slash = p.rfind('/');
    if (slash != std::string::npos) return p.substr(0, slash) + "/../profiles/b200.profile";
  }
  return "";
}

} // namespace

extern "C" {

// ============================================================ runtime
int PMPI_Init(int *, char ***) {
  State &s = S();
  if (s.initialized) return MPI_ERR_OTHER;
  s.rank = env_int("TEMPI_RANK", "RANK", "OMPI_COMM_WORLD_RANK", 0);
  s.size = env_int("TEMPI_SIZE", "WORLD_SIZE", "OMPI_COMM_WORLD_SIZE", 1);
  const int local = env_int("TEMPI_LOCAL_RANK", "LOCAL_RANK", "OMPI_COMM_WORLD_LOCAL_RANK", s.rank);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
    cudaGetLastError();
    ndev = 0;
  }
  s.device = ndev > 0 ? env_int("TEMPI_DEVICE", nullptr, nullptr, local % ndev) : -1;
  std::string job;
  if (const char *j = std::getenv("TEMPI_JOB")) {
    job = j;
  } else if (const char *j2 = std::getenv("TORCHELASTIC_RUN_ID")) {
    job = std::string(j2) + "_" + (std::getenv("MASTER_PORT") ? std::getenv("MASTER_PORT") : "0");
  } else if (const char *p = std::getenv("MASTER_PORT")) {
    job = std::string("port") + p;
  } else {
    job = "single" + std::to_string(getpid());
  }
  const int64_t window = static_cast<int64_t>(env_int("TEMPI_WINDOW_MB", nullptr, nullptr, 256)) << 20;
  const int64_t host = static_cast<int64_t>(env_int("TEMPI_HOST_MB", nullptr, nullptr, 256)) << 20;
  TRY(sp_rt_init(s.rank, s.size, job.c_str(), s.device, window, host));
  // predefined types
  const std::pair<int, int> named[] = {{MPI_BYTE, SP_BYTE},   {MPI_CHAR, SP_BYTE},  {MPI_INT, SP_INT},
                                       {MPI_FLOAT, SP_FLOAT}, {MPI_DOUBLE, SP_DOUBLE},
                                       {MPI_PACKED, SP_BYTE}, {MPI_UNSIGNED_CHAR, SP_BYTE}};
  for (auto [m, k] : named) {
    sp_type h = 0;
    TRY(sp_type_named(k, &h));
    TRY(sp_type_commit(h));
    s.types[m] = h;
  }
  if (s.device >= 0) {
    cudaSetDevice(s.device);
    cudaStreamCreate(&s.stream); // blocking: ordered after the application's legacy-stream work
  }
  std::string prof = std::getenv("TEMPI_PROFILE") ? std::getenv("TEMPI_PROFILE") : default_profile_path();
  if (!prof.empty() && sp_profile_load(prof.c_str(), &s.profile) == SP_OK) sp_rt_set_profile(s.profile);
  if (const char *m = std::getenv("TEMPI_METHOD")) s.forced_method = std::atoi(m);
  s.initialized = true;
  return MPI_SUCCESS;
}

int MPI_Init(int *argc, char ***argv) { return PMPI_Init(argc, argv); }

int MPI_Init_thread(int *argc, char ***argv, int, int *provided) {
  if (provided) *provided = MPI_THREAD_SERIALIZED;
  return PMPI_Init(argc, argv);
}

int MPI_Initialized(int *flag) {
  if (flag) *flag = S().initialized;
  return MPI_SUCCESS;
}

int PMPI_Finalize(void) {
  State &s = S();
  if (!s.initialized || s.finalized) return MPI_ERR_OTHER;
  TRY(sp_rt_finalize());
  if (s.stream) cudaStreamDestroy(s.stream);
  if (s.profile) sp_profile_free(s.profile);
  s.finalized = true;
  return MPI_SUCCESS;
}

int MPI_Finalize(void) { return PMPI_Finalize(); }

int MPI_Finalized(int *flag) {
  if (flag) *flag = S().finalized;
  return MPI_SUCCESS;
}

int PMPI_Comm_rank(MPI_Comm comm, int *rank) {
  if (!comm_of(comm) || !rank) return MPI_ERR_COMM;
  *rank = comm == MPI_COMM_SELF ? 0 : S().rank;
  return MPI_SUCCESS;
}
int MPI_Comm_rank(MPI_Comm comm, int *rank) { return PMPI_Comm_rank(comm, rank); }

int PMPI_Comm_size(MPI_Comm comm, int *size) {
  if (!comm_of(comm) || !size) return MPI_ERR_COMM;
  *size = comm == MPI_COMM_SELF ? 1 : S().size;
  return MPI_SUCCESS;
}
int MPI_Comm_size(MPI_Comm comm, int *size) { return PMPI_Comm_size(comm, size); }

int PMPI_Barrier(MPI_Comm comm) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (comm == MPI_COMM_SELF) return MPI_SUCCESS;
  TRY(sp_rt_barrier());
  return MPI_SUCCESS;
}
int MPI_Barrier(MPI_Comm comm) { return PMPI_Barrier(comm); }

int MPI_Abort(MPI_Comm, int errorcode) {
  std::fprintf(stderr, "MPI_Abort(%d) on rank %d\n", errorcode, S().rank);
  std::_Exit(errorcode ? errorcode : 1);
}

double MPI_Wtime(void) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int MPI_Error_string(int code, char *string, int *len) {
  if (!string || !len) return MPI_ERR_ARG;
  const char *m = code == MPI_SUCCESS ? "success" : code == MPI_ERR_TRUNCATE ? "message truncated"
                  : code == MPI_ERR_TYPE ? "invalid datatype" : code == MPI_ERR_ARG ? "invalid argument"
                  : code == MPI_ERR_UNSUPPORTED_OPERATION ? "unsupported operation" : "error";
  std::snprintf(string, MPI_MAX_ERROR_STRING, "%s", m);
  *len = static_cast<int>(std::strlen(string));
  return MPI_SUCCESS;
}

int MPI_Get_count(const MPI_Status *status, MPI_Datatype datatype, int *count) {
  TYPE(datatype, h);
  int64_t size = 0;
  TRY(sp_type_size(h, &size));
  if (!status || !count) return MPI_ERR_ARG;
  *count = size ? (status->bytes % size ? MPI_UNDEFINED : static_cast<int>(status->bytes / size)) : 0;
  return MPI_SUCCESS;
}

// ============================================================ datatypes
int MPI_Type_contiguous(int count, MPI_Datatype oldtype, MPI_Datatype *newtype) {
  TYPE(oldtype, in);
  sp_type h;
  TRY(sp_type_contiguous(count, in, &h));
  return new_type(h, newtype);
}

int MPI_Type_vector(int count, int blocklength, int stride, MPI_Datatype oldtype, MPI_Datatype *newtype) {
  TYPE(oldtype, in);
  sp_type h;
  TRY(sp_type_vector(count, blocklength, stride, in, &h));
  return new_type(h, newtype);
}

int MPI_Type_create_hvector(int count, int blocklength, MPI_Aint stride, MPI_Datatype oldtype,
                            MPI_Datatype *newtype) {
  TYPE(oldtype, in);
  sp_type h;
  TRY(sp_type_hvector(count, blocklength, stride, in, &h));
  return new_type(h, newtype);
}

// MPI_ORDER_C lists the slowest dimension first; the engine (like the
// reference, type_def.hpp:75) keeps dimension 0 innermost, so C order is
// reversed and Fortran order passed through.
int MPI_Type_create_subarray(int ndims, const int sizes[], const int subsizes[], const int starts[], int order,
                             MPI_Datatype oldtype, MPI_Datatype *newtype) {
  TYPE(oldtype, in);
  if (ndims < 1 || !sizes || !subsizes || !starts) return MPI_ERR_ARG;
  if (order != MPI_ORDER_C && order != MPI_ORDER_FORTRAN) return MPI_ERR_ARG;
  std::vector<int64_t> sz(ndims), sub(ndims), off(ndims);
  for (int i = 0; i < ndims; ++i) {
    const int j = order == MPI_ORDER_C ? ndims - 1 - i : i;
    sz[i] = sizes[j];
    sub[i] = subsizes[j];
    off[i] = starts[j];
    if (off[i] + sub[i] > sz[i]) return MPI_ERR_ARG; // MPI forbids the oversized case
  }
  sp_type h;
  TRY(sp_type_subarray(ndims, sz.data(), sub.data(), off.data(), in, SP_ORDER_C, &h));
  return new_type(h, newtype);
}

// ---- beyond the reference (MPI-3.1 4.1.4-4.1.7): regular patterns are
// canonicalised like the types above, irregular ones run on the device
// run-table kernel
int MPI_Type_indexed(int count, const int blocklengths[], const int displacements[], MPI_Datatype oldtype,
                     MPI_Datatype *newtype) {
  TYPE(oldtype, in);
  if (count < 0 || (count > 0 && (!blocklengths || !displacements))) return MPI_ERR_ARG;
  std::vector<int64_t> bl(blocklengths, blocklengths + count), d(displacements, displacements + count);
  sp_type h;
  TRY(sp_type_indexed(count, bl.data(), d.data(), in, &h));
  return new_type(h, newtype);
}

int MPI_Type_create_hindexed(int count, const int blocklengths[], const MPI_Aint displacements[],
                             MPI_Datatype oldtype, MPI_Datatype *newtype) {
  TYPE(oldtype, in);
  if (count < 0 || (count > 0 && (!blocklengths || !displacements))) return MPI_ERR_ARG;
  std::vector<int64_t> bl(blocklengths, blocklengths + count), d(displacements, displacements + count);
  sp_type h;
  TRY(sp_type_hindexed(count, bl.data(), d.data(), in, &h));
  return new_type(h, newtype);
}

int MPI_Type_create_indexed_block(int count, int blocklength, const int displacements[], MPI_Datatype oldtype,
                                  MPI_Datatype *newtype) {
  TYPE(oldtype, in);
  if (count < 0 || (count > 0 && !displacements)) return MPI_ERR_ARG;
  std::vector<int64_t> d(displacements, displacements + count);
  sp_type h;
  TRY(sp_type_indexed_block(count, blocklength, d.data(), in, &h));
  return new_type(h, newtype);
}

int MPI_Type_create_hindexed_block(int count, int blocklength, const MPI_Aint displacements[],
                                   MPI_Datatype oldtype, MPI_Datatype *newtype) {
  TYPE(oldtype, in);
  if (count < 0 || (count > 0 && !displacements)) return MPI_ERR_ARG;
  std::vector<int64_t> d(displacements, displacements + count);
  sp_type h;
  TRY(sp_type_hindexed_block(count, blocklength, d.data(), in, &h));
  return new_type(h, newtype);
}

int MPI_Type_create_struct(int count, const int blocklengths[], const MPI_Aint displacements[],
                           const MPI_Datatype types[], MPI_Datatype *newtype) {
  if (count < 0 || (count > 0 && (!blocklengths || !displacements || !types))) return MPI_ERR_ARG;
  std::vector<int64_t> bl(blocklengths, blocklengths + count), d(displacements, displacements + count);
  std::vector<sp_type> ts;
  for (int i = 0; i < count; ++i) {
    TYPE(types[i], t);
    ts.push_back(t);
  }
  sp_type h;
  TRY(sp_type_struct(count, bl.data(), d.data(), ts.data(), &h));
  return new_type(h, newtype);
}

int MPI_Type_create_resized(MPI_Datatype oldtype, MPI_Aint lb, MPI_Aint extent, MPI_Datatype *newtype) {
  TYPE(oldtype, in);
  sp_type h;
  TRY(sp_type_resized(in, lb, extent, &h));
  return new_type(h, newtype);
}

int PMPI_Type_commit(MPI_Datatype *datatype) {
  if (!datatype) return MPI_ERR_ARG;
  TYPE(*datatype, h);
  TRY(sp_type_commit(h));
  return MPI_SUCCESS;
}
int MPI_Type_commit(MPI_Datatype *datatype) { return PMPI_Type_commit(datatype); }

int MPI_Type_free(MPI_Datatype *datatype) {
  if (!datatype || *datatype < 100) return MPI_ERR_TYPE;
  TYPE(*datatype, h);
  TRY(sp_type_free(h));
  std::lock_guard<std::mutex> lk(S().mu);
  S().types.erase(*datatype);
  *datatype = MPI_DATATYPE_NULL;
  return MPI_SUCCESS;
}

int MPI_Type_size(MPI_Datatype datatype, int *size) {
  TYPE(datatype, h);
  if (!size) return MPI_ERR_ARG;
  int64_t s = 0;
  TRY(sp_type_size(h, &s));
  *size = static_cast<int>(s);
  return MPI_SUCCESS;
}

int MPI_Type_get_extent(MPI_Datatype datatype, MPI_Aint *lb, MPI_Aint *extent) {
  TYPE(datatype, h);
  if (!lb || !extent) return MPI_ERR_ARG;
  int64_t e = 0, l = 0;
  TRY(sp_type_extent(h, &e));
  TRY(sp_type_lb(h, &l));
  *lb = l;
  *extent = e;
  return MPI_SUCCESS;
}

// ============================================================ packing
int PMPI_Pack(const void *inbuf, int incount, MPI_Datatype datatype, void *outbuf, int outsize, int *position,
              MPI_Comm comm) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (!position || outsize < 0) return MPI_ERR_ARG;
  if (incount < 0) return MPI_ERR_COUNT;
  if (incount == 0) return MPI_SUCCESS; // MPI allows it; the engine (like pack.hpp:102) does not
  TYPE(datatype, h);
  int64_t pos = *position;
  TRY(sp_pack(inbuf, UINT64_MAX, h, incount, outbuf, static_cast<uint64_t>(outsize), &pos, S().stream));
  if (S().stream && cudaStreamSynchronize(S().stream) != cudaSuccess) return MPI_ERR_INTERN;
  *position = static_cast<int>(pos);
  return MPI_SUCCESS;
}
int MPI_Pack(const void *inbuf, int incount, MPI_Datatype datatype, void *outbuf, int outsize, int *position,
             MPI_Comm comm) {
  return PMPI_Pack(inbuf, incount, datatype, outbuf, outsize, position, comm);
}

int PMPI_Unpack(const void *inbuf, int insize, int *position, void *outbuf, int outcount, MPI_Datatype datatype,
                MPI_Comm comm) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (!position || insize < 0) return MPI_ERR_ARG;
  if (outcount < 0) return MPI_ERR_COUNT;
  if (outcount == 0) return MPI_SUCCESS;
  TYPE(datatype, h);
  int64_t pos = *position;
  TRY(sp_unpack(inbuf, static_cast<uint64_t>(insize), &pos, h, outcount, outbuf, UINT64_MAX, S().stream));
  if (S().stream && cudaStreamSynchronize(S().stream) != cudaSuccess) return MPI_ERR_INTERN;
  *position = static_cast<int>(pos);
  return MPI_SUCCESS;
}
int MPI_Unpack(const void *inbuf, int insize, int *position, void *outbuf, int outcount, MPI_Datatype datatype,
               MPI_Comm comm) {
  return PMPI_Unpack(inbuf, insize, position, outbuf, outcount, datatype, comm);
}

int MPI_Pack_size(int incount, MPI_Datatype datatype, MPI_Comm comm, int *size) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  TYPE(datatype, h);
  if (!size || incount < 0) return MPI_ERR_ARG;
  int64_t s = 0;
  TRY(sp_type_size(h, &s));
  *size = static_cast<int>(s * incount);
  return MPI_SUCCESS;
}

// ============================================================ point to point
static int send_impl(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
                     int method) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (dest == MPI_PROC_NULL) return MPI_SUCCESS;
  if (dest < 0 || dest >= S().size) return MPI_ERR_RANK;
  if (tag < 0) return MPI_ERR_TAG;
  if (count < 0) return MPI_ERR_COUNT;
  TYPE(datatype, h);
  TRY(sp_rt_send(buf, UINT64_MAX, count, h, dest, tag, method, nullptr));
  return MPI_SUCCESS;
}

int PMPI_Send(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm) {
  return send_impl(buf, count, datatype, dest, tag, comm, SP_METHOD_DEVICE);
}

// the interposed send: the model picks device / one-shot / staged per
// message unless TEMPI_METHOD forces one
int MPI_Send(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm) {
  return send_impl(buf, count, datatype, dest, tag, comm, S().forced_method);
}

int PMPI_Recv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
              MPI_Status *status) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (source == MPI_PROC_NULL) {
    if (status) *status = MPI_Status{MPI_PROC_NULL, MPI_ANY_TAG, MPI_SUCCESS, 0, 0};
    return MPI_SUCCESS;
  }
  if (count < 0) return MPI_ERR_COUNT;
  TYPE(datatype, h);
  int64_t st[4] = {0, 0, 0, 0};
  TRY(sp_rt_recv(buf, UINT64_MAX, count, h, source, tag, st));
  if (status) *status = MPI_Status{static_cast<int>(st[0]), static_cast<int>(st[1]), MPI_SUCCESS,
                                   static_cast<int>(st[3]), st[2]};
  return MPI_SUCCESS;
}
int MPI_Recv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm, MPI_Status *status) {
  return PMPI_Recv(buf, count, datatype, source, tag, comm, status);
}

// ------------------------------------------------------------ non-blocking
static int isend_impl(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
                      int method, MPI_Request *request) {
  if (!request) return MPI_ERR_ARG;
  *request = MPI_REQUEST_NULL;
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (dest == MPI_PROC_NULL) return MPI_SUCCESS;
  if (dest < 0 || dest >= S().size) return MPI_ERR_RANK;
  if (tag < 0) return MPI_ERR_TAG;
  if (count < 0) return MPI_ERR_COUNT;
  TYPE(datatype, h);
  sp_request r = 0;
  TRY(sp_rt_isend(buf, UINT64_MAX, count, h, dest, tag, method, &r));
  std::lock_guard<std::mutex> lk(S().mu);
  const int id = S().next_request++;
  S().requests[id].r = r;
  *request = id;
  return MPI_SUCCESS;
}

int PMPI_Isend(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
               MPI_Request *request) {
  return isend_impl(buf, count, datatype, dest, tag, comm, SP_METHOD_DEVICE, request);
}

int MPI_Isend(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
              MPI_Request *request) {
  return isend_impl(buf, count, datatype, dest, tag, comm, S().forced_method, request);
}

int PMPI_Irecv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
               MPI_Request *request) {
  if (!request) return MPI_ERR_ARG;
  *request = MPI_REQUEST_NULL;
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (source == MPI_PROC_NULL) return MPI_SUCCESS;
  if (count < 0) return MPI_ERR_COUNT;
  TYPE(datatype, h);
  sp_request r = 0;
  TRY(sp_rt_irecv(buf, UINT64_MAX, count, h, source, tag, &r));
  std::lock_guard<std::mutex> lk(S().mu);
  const int id = S().next_request++;
  S().requests[id].r = r;
  *request = id;
  return MPI_SUCCESS;
}

int MPI_Irecv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
              MPI_Request *request) {
  return PMPI_Irecv(buf, count, datatype, source, tag, comm, request);
}

// asks the engine whether a request is done (waiting for it when `block`)
// and records the outcome on the request; the MPI handle stays valid
static int progress(MPI_Request request, bool block, bool *done) {
  State::Pending p;
  {
    std::lock_guard<std::mutex> lk(S().mu);
    auto it = S().requests.find(request);
    if (it == S().requests.end()) return MPI_ERR_ARG;
    p = it->second;
  }
  if (p.persistent && !p.active) { // an inactive persistent request is complete
    *done = true;
    return MPI_SUCCESS;
  }
  if (!p.done && p.plan) { // a started persistent neighbour collective
    int d = 1;
    p.rc = block ? sp_nbr_plan_wait(p.plan) : sp_nbr_plan_test(p.plan, &d);
    p.done = d || p.rc != SP_OK;
    std::lock_guard<std::mutex> lk(S().mu);
    S().requests[request] = p;
  }
  if (!p.done) {
    int d = 1;
    p.rc = block ? sp_rt_wait(p.r, p.st) : sp_rt_test(p.r, &d, p.st);
    p.done = d || p.rc != SP_OK;
    std::lock_guard<std::mutex> lk(S().mu);
    S().requests[request] = p;
  }
  *done = p.done;
  return MPI_SUCCESS;
}

static int complete(MPI_Request *request, MPI_Status *status, bool block, int *flag) {
  if (!request) return MPI_ERR_ARG;
  if (*request == MPI_REQUEST_NULL) { // null or PROC_NULL request: empty status
    if (status) *status = MPI_Status{MPI_ANY_SOURCE, MPI_ANY_TAG, MPI_SUCCESS, 0, 0};
    if (flag) *flag = 1;
    return MPI_SUCCESS;
  }
  bool done = false;
  const int prc = progress(*request, block, &done);
  if (prc != MPI_SUCCESS) return prc;
  if (flag) *flag = done;
  if (!done) return MPI_SUCCESS;
  State::Pending p;
  {
    std::lock_guard<std::mutex> lk(S().mu);
    State::Pending &e = S().requests[*request];
    p = e;
    if (e.persistent) { // completes, and stays allocated (inactive) for the next MPI_Start
      e.active = false;
      e.done = false;
      e.r = 0;
    } else {
      S().requests.erase(*request);
    }
  }
  if (!p.persistent) *request = MPI_REQUEST_NULL;
  if (p.persistent && !p.active) { // inactive: an empty status
    if (status) *status = MPI_Status{MPI_ANY_SOURCE, MPI_ANY_TAG, MPI_SUCCESS, 0, 0};
    return MPI_SUCCESS;
  }
  TRY(p.rc);
  if (status) *status = MPI_Status{static_cast<int>(p.st[0]), static_cast<int>(p.st[1]), MPI_SUCCESS,
                                   static_cast<int>(p.st[3]), p.st[2]};
  return MPI_SUCCESS;
}

// MPI_REQUEST_NULL or an inactive persistent request: skipped by the set
// completions (MPI-3.1 3.7.5)
static bool inactive(MPI_Request r) {
  if (r == MPI_REQUEST_NULL) return true;
  std::lock_guard<std::mutex> lk(S().mu);
  auto it = S().requests.find(r);
  return it != S().requests.end() && it->second.persistent && !it->second.active;
}

// ---- persistent requests (MPI-3.1 3.9)
static int persistent_init(bool is_send, const void *buf, int count, MPI_Datatype dt, int peer, int tag,
                           MPI_Comm comm, MPI_Request *request) {
  if (!request) return MPI_ERR_ARG;
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (count < 0) return MPI_ERR_COUNT;
  if (is_send && tag < 0) return MPI_ERR_TAG;
  if (peer != MPI_PROC_NULL && (is_send || peer != MPI_ANY_SOURCE) && (peer < 0 || peer >= S().size))
    return MPI_ERR_RANK;
  TYPE(dt, h);
  (void)h;
  std::lock_guard<std::mutex> lk(S().mu);
  const int id = S().next_request++;
  State::Pending &e = S().requests[id];
  e.persistent = true;
  e.is_send = is_send;
  e.buf = buf;
  e.count = count;
  e.dt = dt;
  e.peer = peer;
  e.tag = tag;
  e.comm = comm;
  *request = id;
  return MPI_SUCCESS;
}

int MPI_Send_init(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
                  MPI_Request *request) {
  return persistent_init(true, buf, count, datatype, dest, tag, comm, request);
}

int MPI_Recv_init(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
                  MPI_Request *request) {
  return persistent_init(false, buf, count, datatype, source, tag, comm, request);
}

int MPI_Start(MPI_Request *request) {
  if (!request || *request == MPI_REQUEST_NULL) return MPI_ERR_ARG;
  State::Pending p;
  {
    std::lock_guard<std::mutex> lk(S().mu);
    auto it = S().requests.find(*request);
    if (it == S().requests.end() || !it->second.persistent || it->second.active) return MPI_ERR_ARG;
    p = it->second;
  }
  if (p.plan || p.rerun) { // a persistent neighbour collective
    const sp_status rc = p.plan ? sp_nbr_plan_start(p.plan) : (*p.rerun)();
    std::lock_guard<std::mutex> lk(S().mu);
    State::Pending &e = S().requests[*request];
    e.active = true;
    e.done = !p.plan || rc != SP_OK; // the re-run call has completed already
    e.rc = rc;
    for (auto &v : e.st) v = 0;
    return MPI_SUCCESS;
  }
  if (p.peer == MPI_PROC_NULL) return MPI_SUCCESS; // completes at once
  TYPE(p.dt, h);
  sp_request r = 0;
  if (p.is_send) {
    TRY(sp_rt_isend(p.buf, UINT64_MAX, p.count, h, p.peer, p.tag, S().forced_method, &r));
  } else {
    TRY(sp_rt_irecv(const_cast<void *>(p.buf), UINT64_MAX, p.count, h, p.peer, p.tag, &r));
  }
  std::lock_guard<std::mutex> lk(S().mu);
  State::Pending &e = S().requests[*request];
  e.r = r;
  e.active = true;
  e.done = false;
  e.rc = SP_OK;
  return MPI_SUCCESS;
}

int MPI_Startall(int count, MPI_Request requests[]) {
  if (count < 0 || (count && !requests)) return MPI_ERR_ARG;
  for (int i = 0; i < count; ++i) {
    const int rc = MPI_Start(&requests[i]);
    if (rc != MPI_SUCCESS) return rc;
  }
  return MPI_SUCCESS;
}

int PMPI_Wait(MPI_Request *request, MPI_Status *status) { return complete(request, status, true, nullptr); }
int MPI_Wait(MPI_Request *request, MPI_Status *status) { return PMPI_Wait(request, status); }

int MPI_Test(MPI_Request *request, int *flag, MPI_Status *status) {
  if (!flag) return MPI_ERR_ARG;
  return complete(request, status, false, flag);
}

int MPI_Waitall(int count, MPI_Request requests[], MPI_Status statuses[]) {
  if (count < 0 || (count && !requests)) return MPI_ERR_ARG;
  int first_err = MPI_SUCCESS;
  for (int i = 0; i < count; ++i) {
    const int rc = complete(&requests[i], statuses ? &statuses[i] : nullptr, true, nullptr);
    if (rc != MPI_SUCCESS && first_err == MPI_SUCCESS) first_err = rc;
  }
  return first_err;
}

// MPI-3.1 3.7.5: the set forms poll every active request with MPI_Test
// (which progresses the runtime) until their condition holds
static bool all_null(int n, const MPI_Request r[]) {
  for (int i = 0; i < n; ++i)
    if (!inactive(r[i])) return false;
  return true;
}

int MPI_Testany(int count, MPI_Request requests[], int *index, int *flag, MPI_Status *status) {
  if (count < 0 || (count && !requests) || !index || !flag) return MPI_ERR_ARG;
  *index = MPI_UNDEFINED;
  *flag = 0;
  if (all_null(count, requests)) { // no active request: flag true, index undefined
    *flag = 1;
    if (status) *status = MPI_Status{MPI_ANY_SOURCE, MPI_ANY_TAG, MPI_SUCCESS, 0, 0};
    return MPI_SUCCESS;
  }
  for (int i = 0; i < count; ++i) {
    if (inactive(requests[i])) continue;
    int done = 0;
    const int rc = complete(&requests[i], status, false, &done);
    if (rc != MPI_SUCCESS || done) {
      *index = i;
      *flag = 1;
      return rc;
    }
  }
  return MPI_SUCCESS;
}

int MPI_Waitany(int count, MPI_Request requests[], int *index, MPI_Status *status) {
  int flag = 0;
  for (;;) {
    const int rc = MPI_Testany(count, requests, index, &flag, status);
    if (rc != MPI_SUCCESS || flag) return rc;
  }
}

int MPI_Testall(int count, MPI_Request requests[], int *flag, MPI_Status statuses[]) {
  if (count < 0 || (count && !requests) || !flag) return MPI_ERR_ARG;
  // all or nothing: no handle changes until every request is done
  for (int i = 0; i < count; ++i) {
    if (requests[i] == MPI_REQUEST_NULL) continue;
    bool done = false;
    const int rc = progress(requests[i], false, &done);
    if (rc != MPI_SUCCESS) return rc;
    if (!done) {
      *flag = 0;
      return MPI_SUCCESS;
    }
  }
  *flag = 1;
  return MPI_Waitall(count, requests, statuses); // every one is done: releases them
}

int MPI_Waitsome(int incount, MPI_Request requests[], int *outcount, int indices[], MPI_Status statuses[]) {
  if (incount < 0 || (incount && !requests) || !outcount || (incount && !indices)) return MPI_ERR_ARG;
  if (all_null(incount, requests)) {
    *outcount = MPI_UNDEFINED;
    return MPI_SUCCESS;
  }
  for (;;) {
    int n = 0, first = MPI_SUCCESS;
    for (int i = 0; i < incount; ++i) {
      if (inactive(requests[i])) continue;
      int done = 0;
      const int rc = complete(&requests[i], statuses ? &statuses[n] : nullptr, false, &done);
      if (rc != MPI_SUCCESS && first == MPI_SUCCESS) first = rc;
      if (done || rc != MPI_SUCCESS) indices[n++] = i;
    }
    if (n) {
      *outcount = n;
      return first;
    }
  }
}

int MPI_Request_free(MPI_Request *request) {
  if (!request) return MPI_ERR_ARG;
  if (*request == MPI_REQUEST_NULL) return MPI_ERR_ARG;
  const int rc = complete(request, nullptr, true, nullptr); // completes it, then the handle is released
  if (*request != MPI_REQUEST_NULL) { // persistent: released here
    sp_nbr_plan plan = nullptr;
    {
      std::lock_guard<std::mutex> lk(S().mu);
      plan = S().requests[*request].plan;
      S().requests.erase(*request);
    }
    if (plan) sp_nbr_plan_free(plan);
    *request = MPI_REQUEST_NULL;
  }
  return rc;
}

int MPI_Sendrecv(const void *sendbuf, int sendcount, MPI_Datatype sendtype, int dest, int sendtag, void *recvbuf,
                 int recvcount, MPI_Datatype recvtype, int source, int recvtag, MPI_Comm comm,
                 MPI_Status *status) {
  MPI_Request r[2] = {MPI_REQUEST_NULL, MPI_REQUEST_NULL};
  int rc = MPI_Irecv(recvbuf, recvcount, recvtype, source, recvtag, comm, &r[0]);
  if (rc != MPI_SUCCESS) return rc;
  rc = MPI_Isend(sendbuf, sendcount, sendtype, dest, sendtag, comm, &r[1]);
  if (rc != MPI_SUCCESS) {
    MPI_Wait(&r[0], MPI_STATUS_IGNORE);
    return rc;
  }
  const int rc1 = MPI_Wait(&r[1], MPI_STATUS_IGNORE);
  const int rc0 = MPI_Wait(&r[0], status);
  return rc0 != MPI_SUCCESS ? rc0 : rc1;
}

// ============================================================ topologies
int MPI_Dist_graph_create_adjacent(MPI_Comm comm_old, int indegree, const int sources[], const int *,
                                   int outdegree, const int destinations[], const int *, MPI_Info, int,
                                   MPI_Comm *comm_dist_graph) {
  if (!comm_of(comm_old) || !comm_dist_graph) return MPI_ERR_COMM;
  if (indegree < 0 || outdegree < 0) return MPI_ERR_ARG;
  Comm c;
  c.kind = 1;
  c.sources.assign(sources, sources + indegree);
  c.dests.assign(destinations, destinations + outdegree);
  for (int r : c.sources)
    if ((r < 0 || r >= S().size) && r != MPI_PROC_NULL) return MPI_ERR_RANK;
  for (int r : c.dests)
    if ((r < 0 || r >= S().size) && r != MPI_PROC_NULL) return MPI_ERR_RANK;
  std::lock_guard<std::mutex> lk(S().mu);
  const int id = S().next_comm++;
  S().comms[id] = std::move(c);
  *comm_dist_graph = id;
  return MPI_SUCCESS;
}

int MPI_Dist_graph_neighbors_count(MPI_Comm comm, int *indegree, int *outdegree, int *weighted) {
  const Comm *c = comm_of(comm);
  if (!c || !indegree || !outdegree) return MPI_ERR_COMM;
  *indegree = static_cast<int>(c->sources.size());
  *outdegree = static_cast<int>(c->dests.size());
  if (weighted) *weighted = 0;
  return MPI_SUCCESS;
}

int MPI_Dist_graph_neighbors(MPI_Comm comm, int maxin, int sources[], int *, int maxout, int destinations[],
                             int *) {
  const Comm *c = comm_of(comm);
  if (!c) return MPI_ERR_COMM;
  for (int i = 0; i < maxin && i < static_cast<int>(c->sources.size()); ++i) sources[i] = c->sources[i];
  for (int i = 0; i < maxout && i < static_cast<int>(c->dests.size()); ++i) destinations[i] = c->dests[i];
  return MPI_SUCCESS;
}

int MPI_Cart_create(MPI_Comm comm_old, int ndims, const int dims[], const int periods[], int, MPI_Comm *comm_cart) {
  if (!comm_of(comm_old) || !comm_cart) return MPI_ERR_COMM;
  int n = 1;
  for (int i = 0; i < ndims; ++i) n *= dims[i];
  if (n != S().size) return MPI_ERR_ARG;
  Comm c;
  c.kind = 2;
  c.dims.assign(dims, dims + ndims);
  c.periods.assign(periods, periods + ndims);
  std::lock_guard<std::mutex> lk(S().mu);
  const int id = S().next_comm++;
  S().comms[id] = c;
  *comm_cart = id;
  // neighbour order of a Cartesian topology: per dimension, -1 then +1
  auto &cc = S().comms[id];
  for (int d = 0; d < ndims; ++d) {
    int src = 0, dst = 0;
    MPI_Cart_shift(id, d, 1, &src, &dst);
    cc.sources.push_back(src);
    cc.sources.push_back(dst);
    cc.dests.push_back(src);
    cc.dests.push_back(dst);
  }
  return MPI_SUCCESS;
}

int MPI_Cart_coords(MPI_Comm comm, int rank, int maxdims, int coords[]) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind != 2) return MPI_ERR_COMM;
  const int nd = static_cast<int>(c->dims.size());
  for (int d = nd - 1; d >= 0; --d) { // row-major: last dimension fastest
    if (d < maxdims) coords[d] = rank % c->dims[d];
    rank /= c->dims[d];
  }
  return MPI_SUCCESS;
}

int MPI_Cart_rank(MPI_Comm comm, const int coords[], int *rank) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind != 2 || !rank) return MPI_ERR_COMM;
  int r = 0;
  for (size_t d = 0; d < c->dims.size(); ++d) {
    int x = coords[d];
    if (c->periods[d]) {
      x = ((x % c->dims[d]) + c->dims[d]) % c->dims[d];
    } else if (x < 0 || x >= c->dims[d]) {
      *rank = MPI_PROC_NULL;
      return MPI_SUCCESS;
    }
    r = r * c->dims[d] + x;
  }
  *rank = r;
  return MPI_SUCCESS;
}

int MPI_Cart_shift(MPI_Comm comm, int direction, int disp, int *rank_source, int *rank_dest) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind != 2 || direction < 0 || direction >= static_cast<int>(c->dims.size())) return MPI_ERR_COMM;
  std::vector<int> co(c->dims.size());
  MPI_Cart_coords(comm, S().rank, static_cast<int>(co.size()), co.data());
  co[direction] -= disp;
  MPI_Cart_rank(comm, co.data(), rank_source);
  co[direction] += 2 * disp;
  MPI_Cart_rank(comm, co.data(), rank_dest);
  return MPI_SUCCESS;
}

int MPI_Comm_free(MPI_Comm *comm) {
  if (!comm || *comm < 100) return MPI_ERR_COMM;
  std::lock_guard<std::mutex> lk(S().mu);
  S().comms.erase(*comm);
  *comm = MPI_COMM_NULL;
  return MPI_SUCCESS;
}

// ============================================================ neighbour exchange
// contiguous bytes: the packed-segment receive of the neighbour alltoallv path
static bool dense_type(sp_type h) {
  sp_type_info info{};
  return sp_type_query(h, &info, nullptr, nullptr, 0) == SP_OK &&
         (info.form == SP_FORM_EMPTY ||
          (info.form == SP_FORM_STRIDED && info.ndims == 1 && info.start == 0 && info.extent == info.size));
}

int PMPI_Neighbor_alltoallv(const void *sendbuf, const int sendcounts[], const int sdispls[], MPI_Datatype sendtype,
                            void *recvbuf, const int recvcounts[], const int rdispls[], MPI_Datatype recvtype,
                            MPI_Comm comm) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind == 0) return MPI_ERR_COMM;
  TYPE(sendtype, hs);
  TYPE(recvtype, hr);
  // drop MPI_PROC_NULL edges (non-periodic Cartesian borders)
  std::vector<int> src, dst;
  std::vector<int64_t> scount, sdisp, rcount, rdisp;
  for (size_t i = 0; i < c->dests.size(); ++i)
    if (c->dests[i] != MPI_PROC_NULL) {
      dst.push_back(c->dests[i]);
      scount.push_back(sendcounts[i]);
      sdisp.push_back(sdispls[i]);
    }
  for (size_t j = 0; j < c->sources.size(); ++j)
    if (c->sources[j] != MPI_PROC_NULL) {
      src.push_back(c->sources[j]);
      rcount.push_back(recvcounts[j]);
      rdisp.push_back(rdispls[j]);
    }
  if (!dense_type(hr)) {
    // a strided receive type: every block is a typed copy to its strided
    // place (the alltoallw path, byte displacements)
    int64_t se = 0, re = 0;
    TRY(sp_type_extent(hs, &se));
    TRY(sp_type_extent(hr, &re));
    for (auto &d : sdisp) d *= se;
    for (auto &d : rdisp) d *= re;
    const std::vector<sp_type> st(dst.size(), hs), rt(src.size(), hr);
    TRY(sp_rt_neighbor_alltoallw(sendbuf, scount.data(), sdisp.data(), st.data(), static_cast<int64_t>(dst.size()),
                                 dst.data(), recvbuf, rcount.data(), rdisp.data(), rt.data(),
                                 static_cast<int64_t>(src.size()), src.data()));
    return MPI_SUCCESS;
  }
  TRY(sp_rt_neighbor_alltoallv(sendbuf, scount.data(), sdisp.data(), static_cast<int64_t>(dst.size()), dst.data(),
                               hs, recvbuf, rcount.data(), rdisp.data(), static_cast<int64_t>(src.size()),
                               src.data(), hr));
  return MPI_SUCCESS;
}

int MPI_Neighbor_alltoallv(const void *sendbuf, const int sendcounts[], const int sdispls[], MPI_Datatype sendtype,
                           void *recvbuf, const int recvcounts[], const int rdispls[], MPI_Datatype recvtype,
                           MPI_Comm comm) {
  return PMPI_Neighbor_alltoallv(sendbuf, sendcounts, sdispls, sendtype, recvbuf, recvcounts, rdispls, recvtype,
                                 comm);
}

int PMPI_Neighbor_alltoallw(const void *sendbuf, const int sendcounts[], const MPI_Aint sdispls[],
                            const MPI_Datatype sendtypes[], void *recvbuf, const int recvcounts[],
                            const MPI_Aint rdispls[], const MPI_Datatype recvtypes[], MPI_Comm comm) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind == 0) return MPI_ERR_COMM;
  std::vector<int> src, dst;
  std::vector<int64_t> scount, sdisp, rcount, rdisp;
  std::vector<sp_type> st, rt;
  for (size_t i = 0; i < c->dests.size(); ++i)
    if (c->dests[i] != MPI_PROC_NULL) {
      TYPE(sendtypes[i], h);
      dst.push_back(c->dests[i]);
      scount.push_back(sendcounts[i]);
      sdisp.push_back(sdispls[i]);
      st.push_back(h);
    }
  for (size_t j = 0; j < c->sources.size(); ++j)
    if (c->sources[j] != MPI_PROC_NULL) {
      TYPE(recvtypes[j], h);
      src.push_back(c->sources[j]);
      rcount.push_back(recvcounts[j]);
      rdisp.push_back(rdispls[j]);
      rt.push_back(h);
    }
  TRY(sp_rt_neighbor_alltoallw(sendbuf, scount.data(), sdisp.data(), st.data(), static_cast<int64_t>(dst.size()),
                               dst.data(), recvbuf, rcount.data(), rdisp.data(), rt.data(),
                               static_cast<int64_t>(src.size()), src.data()));
  return MPI_SUCCESS;
}

int MPI_Neighbor_alltoallw(const void *sendbuf, const int sendcounts[], const MPI_Aint sdispls[],
                           const MPI_Datatype sendtypes[], void *recvbuf, const int recvcounts[],
                           const MPI_Aint rdispls[], const MPI_Datatype recvtypes[], MPI_Comm comm) {
  return PMPI_Neighbor_alltoallw(sendbuf, sendcounts, sdispls, sendtypes, recvbuf, recvcounts, rdispls, recvtypes,
                                 comm);
}

// ---- persistent neighbour collectives (MPI-4.0 7.10.2): compiled once
// into one signalled typed-copy launch per start, capturable into CUDA
// graphs; types the engine cannot compile re-run the call at every start
static int nbr_init(const void *sendbuf, const int sendcounts[], const std::vector<int64_t> &sdisp_b,
                    const std::vector<MPI_Datatype> &stypes, void *recvbuf, const int recvcounts[],
                    const std::vector<int64_t> &rdisp_b, const std::vector<MPI_Datatype> &rtypes, MPI_Comm comm,
                    MPI_Request *request) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind == 0) return MPI_ERR_COMM;
  if (!request) return MPI_ERR_ARG;
  std::vector<int> src, dst;
  std::vector<int64_t> scount, sdisp, rcount, rdisp;
  std::vector<sp_type> st, rt;
  for (size_t i = 0; i < c->dests.size(); ++i)
    if (c->dests[i] != MPI_PROC_NULL) {
      TYPE(stypes[i], h);
      dst.push_back(c->dests[i]);
      scount.push_back(sendcounts[i]);
      sdisp.push_back(sdisp_b[i]);
      st.push_back(h);
    }
  for (size_t j = 0; j < c->sources.size(); ++j)
    if (c->sources[j] != MPI_PROC_NULL) {
      TYPE(rtypes[j], h);
      src.push_back(c->sources[j]);
      rcount.push_back(recvcounts[j]);
      rdisp.push_back(rdisp_b[j]);
      rt.push_back(h);
    }
  sp_nbr_plan plan = nullptr;
  const sp_status rc = sp_rt_neighbor_alltoallw_init(sendbuf, scount.data(), sdisp.data(), st.data(),
                                                     static_cast<int64_t>(dst.size()), dst.data(), recvbuf,
                                                     rcount.data(), rdisp.data(), rt.data(),
                                                     static_cast<int64_t>(src.size()), src.data(), &plan);
  if (rc != SP_OK && rc != SP_ERR_UNSUPPORTED) TRY(rc);
  std::lock_guard<std::mutex> lk(S().mu);
  const int id = S().next_request++;
  State::Pending &e = S().requests[id];
  e.persistent = true;
  e.plan = plan;
  if (!plan) // every rank agreed the types cannot be compiled: re-run the call
    e.rerun = std::make_shared<std::function<sp_status()>>([=] {
      return sp_rt_neighbor_alltoallw(sendbuf, scount.data(), sdisp.data(), st.data(),
                                      static_cast<int64_t>(dst.size()), dst.data(), recvbuf, rcount.data(),
                                      rdisp.data(), rt.data(), static_cast<int64_t>(src.size()), src.data());
    });
  *request = id;
  return MPI_SUCCESS;
}

int MPI_Neighbor_alltoallw_init(const void *sendbuf, const int sendcounts[], const MPI_Aint sdispls[],
                                const MPI_Datatype sendtypes[], void *recvbuf, const int recvcounts[],
                                const MPI_Aint rdispls[], const MPI_Datatype recvtypes[], MPI_Comm comm, MPI_Info,
                                MPI_Request *request) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind == 0) return MPI_ERR_COMM;
  std::vector<int64_t> sd(sdispls, sdispls + c->dests.size()), rd(rdispls, rdispls + c->sources.size());
  std::vector<MPI_Datatype> st(sendtypes, sendtypes + c->dests.size()), rt(recvtypes, recvtypes + c->sources.size());
  return nbr_init(sendbuf, sendcounts, sd, st, recvbuf, recvcounts, rd, rt, comm, request);
}

int MPI_Neighbor_alltoallv_init(const void *sendbuf, const int sendcounts[], const int sdispls[],
                                MPI_Datatype sendtype, void *recvbuf, const int recvcounts[], const int rdispls[],
                                MPI_Datatype recvtype, MPI_Comm comm, MPI_Info, MPI_Request *request) {
  const Comm *c = comm_of(comm);
  if (!c || c->kind == 0) return MPI_ERR_COMM;
  TYPE(sendtype, hs);
  TYPE(recvtype, hr);
  int64_t se = 0, re = 0;
  TRY(sp_type_extent(hs, &se));
  TRY(sp_type_extent(hr, &re));
  std::vector<int64_t> sd, rd;
  for (size_t i = 0; i < c->dests.size(); ++i) sd.push_back(static_cast<int64_t>(sdispls[i]) * se);
  for (size_t j = 0; j < c->sources.size(); ++j) rd.push_back(static_cast<int64_t>(rdispls[j]) * re);
  return nbr_init(sendbuf, sendcounts, sd, std::vector<MPI_Datatype>(c->dests.size(), sendtype), recvbuf, recvcounts,
                  rd, std::vector<MPI_Datatype>(c->sources.size(), recvtype), comm, request);
}

// ============================================================ all-to-all
// MPI_Alltoallv / MPI_Alltoallw (MPI-3.1 5.8) over the communicator's
// complete graph: the neighbour alltoallw path (one typed-copy launch per
// rank, blocks stored at their strided place in the receivers' buffers).
static int alltoall_impl(const void *sendbuf, const int sendcounts[], const std::vector<int64_t> &sdisp_b,
                         const std::vector<sp_type> &stypes, void *recvbuf, const int recvcounts[],
                         const std::vector<int64_t> &rdisp_b, const std::vector<sp_type> &rtypes, MPI_Comm comm) {
  std::vector<int> ranks;
  if (comm == MPI_COMM_SELF) {
    ranks.push_back(S().rank);
  } else {
    for (int r = 0; r < S().size; ++r) ranks.push_back(r);
  }
  const int64_t n = static_cast<int64_t>(ranks.size());
  if (n > 64) return MPI_ERR_UNSUPPORTED_OPERATION; // the typed-copy path's edge limit
  std::vector<int64_t> sc(sendcounts, sendcounts + n), rc(recvcounts, recvcounts + n);
  TRY(sp_rt_neighbor_alltoallw(sendbuf, sc.data(), sdisp_b.data(), stypes.data(), n, ranks.data(), recvbuf,
                               rc.data(), rdisp_b.data(), rtypes.data(), n, ranks.data()));
  return MPI_SUCCESS;
}

int PMPI_Alltoallv(const void *sendbuf, const int sendcounts[], const int sdispls[], MPI_Datatype sendtype,
                   void *recvbuf, const int recvcounts[], const int rdispls[], MPI_Datatype recvtype, MPI_Comm comm) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (!sendcounts || !sdispls || !recvcounts || !rdispls) return MPI_ERR_ARG;
  TYPE(sendtype, hs);
  TYPE(recvtype, hr);
  int64_t se = 0, re = 0;
  TRY(sp_type_extent(hs, &se));
  TRY(sp_type_extent(hr, &re));
  const int n = comm == MPI_COMM_SELF ? 1 : S().size;
  std::vector<int64_t> sd(n), rd(n);
  for (int i = 0; i < n; ++i) {
    sd[i] = static_cast<int64_t>(sdispls[i]) * se;
    rd[i] = static_cast<int64_t>(rdispls[i]) * re;
  }
  return alltoall_impl(sendbuf, sendcounts, sd, std::vector<sp_type>(n, hs), recvbuf, recvcounts, rd,
                       std::vector<sp_type>(n, hr), comm);
}
int MPI_Alltoallv(const void *sendbuf, const int sendcounts[], const int sdispls[], MPI_Datatype sendtype,
                  void *recvbuf, const int recvcounts[], const int rdispls[], MPI_Datatype recvtype, MPI_Comm comm) {
  return PMPI_Alltoallv(sendbuf, sendcounts, sdispls, sendtype, recvbuf, recvcounts, rdispls, recvtype, comm);
}

int PMPI_Alltoallw(const void *sendbuf, const int sendcounts[], const int sdispls[], const MPI_Datatype sendtypes[],
                   void *recvbuf, const int recvcounts[], const int rdispls[], const MPI_Datatype recvtypes[],
                   MPI_Comm comm) {
  if (!comm_of(comm)) return MPI_ERR_COMM;
  if (!sendcounts || !sdispls || !sendtypes || !recvcounts || !rdispls || !recvtypes) return MPI_ERR_ARG;
  const int n = comm == MPI_COMM_SELF ? 1 : S().size;
  std::vector<int64_t> sd(sdispls, sdispls + n), rd(rdispls, rdispls + n);
  std::vector<sp_type> st, rt;
  for (int i = 0; i < n; ++i) {
    TYPE(sendtypes[i], h);
    st.push_back(h);
  }
  for (int j = 0; j < n; ++j) {
    TYPE(recvtypes[j], h);
    rt.push_back(h);
  }
  return alltoall_impl(sendbuf, sendcounts, sd, st, recvbuf, recvcounts, rd, rt, comm);
}
int MPI_Alltoallw(const void *sendbuf, const int sendcounts[], const int sdispls[], const MPI_Datatype sendtypes[],
                  void *recvbuf, const int recvcounts[], const int rdispls[], const MPI_Datatype recvtypes[],
                  MPI_Comm comm) {
  return PMPI_Alltoallw(sendbuf, sendcounts, sdispls, sendtypes, recvbuf, recvcounts, rdispls, recvtypes, comm);
}

// ============================================================ TEMPI controls
int TEMPI_Set_method(int method) {
  if (method < -1 || method > 3) return MPI_ERR_ARG;
  S().forced_method = method;
  return MPI_SUCCESS;
}

int TEMPI_Load_profile(const char *path) {
  sp_profile p = nullptr;
  TRY(sp_profile_load(path, &p));
  TRY(sp_rt_set_profile(p));
  if (S().profile) sp_profile_free(S().profile);
  S().profile = p;
  return MPI_SUCCESS;
}

} // extern "C"
