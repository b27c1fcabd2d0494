// Data-parallel gradient exchange: a minimal NCCL binding behind the C ABI.
//
// "NCCL communicator init from a torch-store-shared
// ncclUniqueId; bucketed allreduce enqueue".  The reference trains single
// process and consumes already-reduced gradients (F/engine.py:4-7); the
// exchange step is the one LightSeq2 delegates to PyTorch's all-reduce.
//
// libnccl is resolved at run time (dlopen) rather than linked: the process
// normally already holds the NCCL that torch.distributed loaded, and binding
// that same copy (RTLD_NOLOAD first) keeps one NCCL per process.  Collectives
// are plain stream-ordered enqueues, so they can be captured into the step's
// CUDA graph next to the kernels that produce and consume the buckets.
#include <dlfcn.h>

#include <mutex>

#include "common.cuh"

namespace {

struct NcclUid {
  char internal[128];
};
using ncclComm_t = void*;
using ncclResult_t = int;

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(NcclUid*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, NcclUid, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, int, int, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

// NCCL's ncclDataType_t / ncclRedOp_t values (stable across NCCL 2.x)
constexpr int kNcclInt32 = 2, kNcclFloat16 = 6, kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclBfloat16 = 9;
constexpr int kNcclSum = 0;

int nccl_dtype(int dtype) {
  switch (dtype) {
    case LS2_F16: return kNcclFloat16;
    case LS2_BF16: return kNcclBfloat16;
    case LS2_F32: return kNcclFloat32;
    case LS2_F64: return kNcclFloat64;
    case LS2_I32: return kNcclInt32;
    default: return -1;
  }
}

int load_nccl(const char* path) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.handle) return LS2_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h && path && *path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return ls2::fail(LS2_ERR_CUDA, std::string("cannot load libnccl.so.2: ") + dlerror());
  NcclApi api;
  api.handle = h;
  api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
  api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
  api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
  api.reduce_scatter = (decltype(api.reduce_scatter))dlsym(h, "ncclReduceScatter");
  api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
  api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
  api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
  api.get_version = (decltype(api.get_version))dlsym(h, "ncclGetVersion");
  if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.reduce_scatter ||
      !api.all_gather || !api.comm_destroy)
    return ls2::fail(LS2_ERR_CUDA, "libnccl.so.2 lacks the required entry points");
  g_nccl = api;
  return LS2_OK;
}

int nccl_fail(const char* what, ncclResult_t r) {
  const char* s = g_nccl.error_string ? g_nccl.error_string(r) : "?";
  return ls2::fail(LS2_ERR_CUDA, std::string(what) + ": " + s);
}

}  // namespace

extern "C" {

int ls2_comm_load(const char* path) { return load_nccl(path); }

int ls2_comm_version(int* out) {
  if (int rc = load_nccl(nullptr)) return rc;
  *out = 0;
  if (g_nccl.get_version) g_nccl.get_version(out);
  return LS2_OK;
}

int ls2_comm_unique_id(uint8_t* out128) {
  if (int rc = load_nccl(nullptr)) return rc;
  NcclUid uid;
  if (ncclResult_t r = g_nccl.get_unique_id(&uid)) return nccl_fail("ncclGetUniqueId", r);
  memcpy(out128, uid.internal, 128);
  return LS2_OK;
}

int ls2_comm_init(void** comm_out, int nranks, int rank, const uint8_t* id128, int device) {
  if (int rc = load_nccl(nullptr)) return rc;
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return ls2::fail(LS2_ERR_SHAPE, "comm_init: rank out of range");
  if (cudaSetDevice(device) != cudaSuccess) return ls2::fail(LS2_ERR_CUDA, "comm_init: bad device");
  NcclUid uid;
  memcpy(uid.internal, id128, 128);
  ncclComm_t c = nullptr;
  if (ncclResult_t r = g_nccl.comm_init_rank(&c, nranks, uid, rank))
    return nccl_fail("ncclCommInitRank", r);
  *comm_out = c;
  return LS2_OK;
}

// Sum-allreduce of `count` elements; in place when send == recv.  Enqueue only.
int ls2_comm_allreduce(void* comm, const void* send, void* recv, int64_t count, int dtype,
                       void* stream) {
  if (count <= 0) return LS2_OK;
  if (!comm || !g_nccl.all_reduce) return ls2::fail(LS2_ERR_CUDA, "allreduce: no communicator");
  int dt = nccl_dtype(dtype);
  if (dt < 0) return ls2::fail(LS2_ERR_DTYPE, "allreduce: unsupported dtype");
  if (ncclResult_t r = g_nccl.all_reduce(send, recv, (size_t)count, dt, kNcclSum, comm,
                                         ls2::as_stream(stream)))
    return nccl_fail("ncclAllReduce", r);
  return LS2_OK;
}

// Sum-reduce-scatter: rank r receives elements [r*count, (r+1)*count) of the sum of
// every rank's `send` (N*count elements).  In place when recv == send + rank*count:
// the sharded-optimizer exchange reduces each fp32 gradient bucket this way.
int ls2_comm_reduce_scatter(void* comm, const void* send, void* recv, int64_t count, int dtype,
                            void* stream) {
  if (count <= 0) return LS2_OK;
  if (!comm || !g_nccl.reduce_scatter)
    return ls2::fail(LS2_ERR_CUDA, "reduce_scatter: no communicator");
  int dt = nccl_dtype(dtype);
  if (dt < 0) return ls2::fail(LS2_ERR_DTYPE, "reduce_scatter: unsupported dtype");
  if (ncclResult_t r = g_nccl.reduce_scatter(send, recv, (size_t)count, dt, kNcclSum, comm,
                                             ls2::as_stream(stream)))
    return nccl_fail("ncclReduceScatter", r);
  return LS2_OK;
}

// All-gather: every rank's `count` elements land at recv + r*count on all ranks.  In
// place when send == recv + rank*count (the updated params16 shard of a bucket).
int ls2_comm_all_gather(void* comm, const void* send, void* recv, int64_t count, int dtype,
                        void* stream) {
  if (count <= 0) return LS2_OK;
  if (!comm || !g_nccl.all_gather) return ls2::fail(LS2_ERR_CUDA, "all_gather: no communicator");
  int dt = nccl_dtype(dtype);
  if (dt < 0) return ls2::fail(LS2_ERR_DTYPE, "all_gather: unsupported dtype");
  if (ncclResult_t r = g_nccl.all_gather(send, recv, (size_t)count, dt, comm,
                                         ls2::as_stream(stream)))
    return nccl_fail("ncclAllGather", r);
  return LS2_OK;
}

int ls2_comm_destroy(void* comm) {
  if (!comm || !g_nccl.comm_destroy) return LS2_OK;
  if (ncclResult_t r = g_nccl.comm_destroy(comm)) return nccl_fail("ncclCommDestroy", r);
  return LS2_OK;
}

}  // extern "C"
