// NCCL communicator in the C ABI ("an NCCL communicator handle init/teardown").
//
// The reference's data-parallel split (sobench/backend.py:178-204) is a thread pool inside
// one process; here the split is one process per GPU, and a host that is not Python (the
// reference's CLI driving the library through ctypes, a C++ runner) needs the collective
// without torch.distributed.  libnccl is resolved at run time: the copy torch already
// loaded (RTLD_NOLOAD) when there is one, else libnccl.so.2 from the loader path -- so the
// library has no link-time NCCL dependency and never mixes two NCCL versions in one
// process.  The few NCCL entry points used are declared here with NCCL's stable C ABI
// (ncclUniqueId = 128 bytes, enum values of nccl.h 2.x).
#include <dlfcn.h>
#include <string.h>

#include <mutex>

#include "common.cuh"

namespace {

typedef struct {
  char internal[128];
} NcclUniqueId;
typedef void* NcclComm;
typedef int NcclResult;
constexpr int kNcclUint8 = 1, kNcclFloat64 = 8, kNcclSum = 0, kNcclMin = 3;

struct Nccl {
  NcclResult (*get_unique_id)(NcclUniqueId*) = nullptr;
  NcclResult (*comm_init_rank)(NcclComm*, int, NcclUniqueId, int) = nullptr;
  NcclResult (*comm_destroy)(NcclComm) = nullptr;
  NcclResult (*all_reduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  NcclResult (*all_gather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
  NcclResult (*broadcast)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  const char* (*error_string)(NcclResult) = nullptr;
  NcclResult (*get_version)(int*) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](const char* s) { return dlsym(h, s); };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
    n.broadcast = reinterpret_cast<decltype(n.broadcast)>(sym("ncclBroadcast"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    n.get_version = reinterpret_cast<decltype(n.get_version)>(sym("ncclGetVersion"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_reduce && n.all_gather &&
           n.broadcast && n.error_string;
  });
  return n;
}

int nccl_status(NcclResult r, const char* what) {
  if (r == 0) return SIMOPT_OK;
  simopt_set_error("%s: %s", what, nccl().error_string ? nccl().error_string(r) : "NCCL error");
  return SIMOPT_E_CUDA;
}

#define NCCL_REQUIRE()                                                                            \
  SIMOPT_REQUIRE(nccl().ok, SIMOPT_E_CUDA, "libnccl.so.2 not found (load torch first or put NCCL " \
                 "on the loader path)")

}  // namespace

extern "C" int simopt_comm_version(int* version) {
  NCCL_REQUIRE();
  *version = 0;
  if (nccl().get_version) return nccl_status(nccl().get_version(version), "ncclGetVersion");
  return SIMOPT_OK;
}

extern "C" int simopt_comm_unique_id(uint8_t* id128) {
  NCCL_REQUIRE();
  NcclUniqueId id;
  if (int rc = nccl_status(nccl().get_unique_id(&id), "ncclGetUniqueId")) return rc;
  memcpy(id128, id.internal, 128);
  return SIMOPT_OK;
}

extern "C" int simopt_comm_init(const uint8_t* id128, int world, int rank, void** comm) {
  NCCL_REQUIRE();
  SIMOPT_REQUIRE(world >= 1 && rank >= 0 && rank < world, SIMOPT_E_CONFIG, "bad rank %d of %d", rank,
                 world);
  NcclUniqueId id;
  memcpy(id.internal, id128, 128);
  NcclComm c = nullptr;
  if (int rc = nccl_status(nccl().comm_init_rank(&c, world, id, rank), "ncclCommInitRank")) return rc;
  *comm = c;
  return SIMOPT_OK;
}

extern "C" int simopt_comm_destroy(void* comm) {
  NCCL_REQUIRE();
  if (!comm) return SIMOPT_OK;
  return nccl_status(nccl().comm_destroy(comm), "ncclCommDestroy");
}

// In-place or out-of-place fp64 sum over ranks, on `stream` (the gradient, HVP and C5
// Hessian exchanges of the sample-sharded solvers).
extern "C" int simopt_comm_allreduce_f64(void* comm, void* stream, const double* send, double* recv,
                                         int64_t n) {
  NCCL_REQUIRE();
  if (n == 0) return SIMOPT_OK;
  return nccl_status(nccl().all_reduce(send, recv, (size_t)n, kNcclFloat64, kNcclSum, comm,
                                       as_stream(stream)),
                     "ncclAllReduce");
}

// fp64 minimum over ranks (the newsvendor LMO fallback's agreement check).
extern "C" int simopt_comm_allreduce_min_f64(void* comm, void* stream, const double* send, double* recv,
                                             int64_t n) {
  NCCL_REQUIRE();
  if (n == 0) return SIMOPT_OK;
  return nccl_status(nccl().all_reduce(send, recv, (size_t)n, kNcclFloat64, kNcclMin, comm,
                                       as_stream(stream)),
                     "ncclAllReduce");
}

// Concatenation of every rank's `bytes` bytes in rank order (chunk partials of the
// deterministic-mode reductions, LMO candidates).
extern "C" int simopt_comm_allgather(void* comm, void* stream, const void* send, void* recv,
                                     int64_t bytes) {
  NCCL_REQUIRE();
  if (bytes == 0) return SIMOPT_OK;
  return nccl_status(nccl().all_gather(send, recv, (size_t)bytes, kNcclUint8, comm, as_stream(stream)),
                     "ncclAllGather");
}

extern "C" int simopt_comm_broadcast(void* comm, void* stream, const void* send, void* recv,
                                     int64_t bytes, int root) {
  NCCL_REQUIRE();
  if (bytes == 0) return SIMOPT_OK;
  return nccl_status(nccl().broadcast(send, recv, (size_t)bytes, kNcclUint8, root, comm,
                                      as_stream(stream)),
                     "ncclBroadcast");
}
