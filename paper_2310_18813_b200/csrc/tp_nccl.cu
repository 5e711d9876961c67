// NCCL backend of sb_collectives_t (tensor-parallel exchange of the sharded
// target, BASELINE config 4).  libnccl is opened at run time (the copy torch
// already loaded into the process, or the system one), so the library has no
// link-time NCCL dependency; NCCL calls are stream-ordered and CUDA-graph
// capturable, so a TP forward captures into the per-(b,k) iteration graph.
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace {

typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclFloat32 = 7, kNcclBfloat16 = 9, kNcclSum = 0 };

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
    a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
    a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce && a.all_gather;
  });
  return a;
}

int nccl_dtype(int32_t dt) { return dt == SB_BF16 ? kNcclBfloat16 : kNcclFloat32; }

// NCCL failures are reported as SB_EUNSUPPORTED + 1000 + ncclResult (>= 2000, distinct from cudaError_t)
int nccl_rc(ncclResult_t r) { return r == 0 ? 0 : 2000 + r; }

int cb_all_reduce(void* ctx, void* buf, size_t count, int32_t dtype, void* stream) {
  return nccl_rc(api().all_reduce(buf, buf, count, nccl_dtype(dtype), kNcclSum, (ncclComm_t)ctx, (cudaStream_t)stream));
}
int cb_all_gather(void* ctx, const void* send, void* recv, size_t count, int32_t dtype, void* stream) {
  return nccl_rc(api().all_gather(send, recv, count, nccl_dtype(dtype), (ncclComm_t)ctx, (cudaStream_t)stream));
}

}  // namespace

extern "C" {

int sb_nccl_unique_id(void* id_out) {
  if (!id_out) return SB_EINVAL;
  if (!api().ok) return SB_EUNSUPPORTED;
  ncclUniqueId id;
  int rc = nccl_rc(api().get_unique_id(&id));
  if (rc) return rc;
  memcpy(id_out, &id, sizeof(id));
  return 0;
}

int sb_nccl_collectives_init(const void* id, int32_t world, int32_t rank, sb_collectives_t* out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return SB_EINVAL;
  if (!api().ok) return SB_EUNSUPPORTED;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  int rc = nccl_rc(api().comm_init_rank(&comm, world, uid, rank));
  if (rc) return rc;
  out->ctx = comm;
  out->all_reduce_sum = cb_all_reduce;
  out->all_gather = cb_all_gather;
  out->world = world;
  out->rank = rank;
  return 0;
}

int sb_nccl_collectives_destroy(sb_collectives_t* c) {
  if (!c || !c->ctx) return SB_EINVAL;
  int rc = nccl_rc(api().comm_destroy((ncclComm_t)c->ctx));
  c->ctx = nullptr;
  return rc;
}

}  // extern "C"
