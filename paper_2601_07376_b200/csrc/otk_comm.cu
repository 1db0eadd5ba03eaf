// otk_comm.cu — batch sharding over NCCL (include/otk.h "Batch sharding"; SURVEY.md §8(e) BATCH): the ctx's
// communicator and the three exchanges of a batch-sharded step (global token count, group statistics over the
// union of the shards, loss statistics). Host code only; NCCL is bound at run time (dlopen), so libotk.so has
// no link-time NCCL dependency and, inside a PyTorch process, uses the NCCL copy torch already loaded.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types and enum values only (the functions come from dlsym)

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "otk_internal.h"

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi load_nccl() {
  NcclApi a;
  const char* env = std::getenv("OTK_NCCL_LIB");
  void* h = nullptr;
  if (env && *env) {
    h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
  } else {
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // already in the process (e.g. torch's)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
  }
  if (!h) {
    const char* e = dlerror();
    a.why = std::string("cannot load NCCL: ") + (e ? e : "libnccl.so.2 not found");
    return a;
  }
  auto sym = [&](const char* name) -> void* {
    void* f = dlsym(h, name);
    if (!f && a.why.empty()) a.why = std::string("NCCL symbol missing: ") + name;
    return f;
  };
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
  a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
  a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
  a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
  a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
  a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  a.ok = a.why.empty();
  return a;
}

const NcclApi& nccl() {
  static NcclApi api = load_nccl();   // thread-safe one-time binding
  return api;
}

otk_status nccl_fail(const char* where, ncclResult_t r) {
  const std::string msg = std::string(where) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
  return otk::host_fail(OTK_ERR_NCCL, msg.c_str());
}

#define OTK_REQ(cond, code, msg)                      \
  do {                                                \
    if (!(cond)) return otk::host_fail(code, msg);    \
  } while (0)
#define OTK_NCCL(call, where)                         \
  do {                                                \
    const ncclResult_t r_ = (call);                   \
    if (r_ != ncclSuccess) return nccl_fail(where, r_); \
  } while (0)

otk_status need_nccl() {
  if (!nccl().ok) return otk::host_fail(OTK_ERR_NCCL, nccl().why.c_str());
  return OTK_OK;
}

otk_status need_comm(const otk_ctx* ctx) {
  OTK_REQ(ctx, OTK_ERR_INVALID_ARG, "ctx is NULL");
  OTK_REQ(ctx->comm, OTK_ERR_NO_COMM, "no communicator on this ctx (otk_comm_init)");
  return OTK_OK;
}

ncclComm_t comm_of(const otk_ctx* ctx) { return reinterpret_cast<ncclComm_t>(ctx->comm); }

}  // namespace

void otk::comm_release(otk_ctx* ctx) {
  if (ctx && ctx->comm && nccl().ok) nccl().CommDestroy(comm_of(ctx));
  if (ctx) {
    ctx->comm = nullptr;
    ctx->comm_nranks = 0;
    ctx->comm_rank = 0;
  }
}

extern "C" {

otk_status otk_comm_unique_id(unsigned char id[OTK_COMM_ID_BYTES]) {
  OTK_REQ(id, OTK_ERR_INVALID_ARG, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == OTK_COMM_ID_BYTES, "NCCL unique id size");
  if (otk_status s = need_nccl()) return s;
  ncclUniqueId u;
  OTK_NCCL(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
  return OTK_OK;
}

otk_status otk_comm_init(otk_ctx* ctx, const unsigned char id[OTK_COMM_ID_BYTES], int32_t nranks, int32_t rank) {
  OTK_REQ(ctx && id, OTK_ERR_INVALID_ARG, "ctx / id is NULL");
  OTK_REQ(nranks >= 1 && rank >= 0 && rank < nranks, OTK_ERR_SHAPE, "need nranks >= 1 and 0 <= rank < nranks");
  OTK_REQ(!ctx->comm, OTK_ERR_INVALID_ARG, "ctx already has a communicator (otk_comm_destroy first)");
  if (otk_status s = need_nccl()) return s;
  const cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return otk::host_fail(OTK_ERR_CUDA, cudaGetErrorString(e));
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  OTK_NCCL(nccl().CommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
  ctx->comm = c;
  ctx->comm_nranks = nranks;
  ctx->comm_rank = rank;
  return OTK_OK;
}

otk_status otk_comm_destroy(otk_ctx* ctx) {
  OTK_REQ(ctx, OTK_ERR_INVALID_ARG, "ctx is NULL");
  otk::comm_release(ctx);
  return OTK_OK;
}

otk_status otk_comm_size(const otk_ctx* ctx, int32_t* nranks, int32_t* rank) {
  OTK_REQ(nranks && rank, OTK_ERR_INVALID_ARG, "nranks / rank is NULL");
  if (otk_status s = need_comm(ctx)) return s;
  *nranks = ctx->comm_nranks;
  *rank = ctx->comm_rank;
  return OTK_OK;
}

otk_status otk_batch_allreduce_i64(otk_ctx* ctx, int64_t* buf, int64_t n, otk_stream_t stream) {
  if (otk_status s = need_comm(ctx)) return s;
  OTK_REQ(n >= 0 && (n == 0 || buf), OTK_ERR_INVALID_ARG, "need n >= 0 and buf");
  if (n == 0) return OTK_OK;
  OTK_NCCL(nccl().AllReduce(buf, buf, size_t(n), ncclInt64, ncclSum, comm_of(ctx),
                            reinterpret_cast<cudaStream_t>(stream)),
           "ncclAllReduce(int64)");
  return OTK_OK;
}

otk_status otk_batch_allreduce_f64(otk_ctx* ctx, double* buf, int64_t n, otk_stream_t stream) {
  if (otk_status s = need_comm(ctx)) return s;
  OTK_REQ(n >= 0 && (n == 0 || buf), OTK_ERR_INVALID_ARG, "need n >= 0 and buf");
  if (n == 0) return OTK_OK;
  OTK_NCCL(nccl().AllReduce(buf, buf, size_t(n), ncclFloat64, ncclSum, comm_of(ctx),
                            reinterpret_cast<cudaStream_t>(stream)),
           "ncclAllReduce(float64)");
  return OTK_OK;
}

otk_status otk_batch_group_advantages(otk_ctx* ctx, int32_t num_traj_local, const int32_t* group_id,
                                      const double* returns, const int32_t* counts, int32_t num_groups,
                                      uint32_t flags, double std_floor, int32_t* gid_all, double* ret_all,
                                      double* adv_all, double* group_mean, double* group_std, int32_t* group_size,
                                      otk_stream_t stream) {
  if (otk_status s = need_comm(ctx)) return s;
  OTK_REQ(counts && gid_all && ret_all && adv_all, OTK_ERR_INVALID_ARG, "counts / gid_all / ret_all / adv_all is NULL");
  const int P = ctx->comm_nranks, me = ctx->comm_rank;
  OTK_REQ(counts[me] == num_traj_local, OTK_ERR_SHAPE, "counts[rank] != num_traj_local");
  OTK_REQ(num_traj_local == 0 || (group_id && returns), OTK_ERR_INVALID_ARG, "group_id / returns is NULL");
  int64_t total = 0;
  for (int r = 0; r < P; ++r) {
    OTK_REQ(counts[r] >= 0, OTK_ERR_SHAPE, "counts[r] < 0");
    total += counts[r];
  }
  OTK_REQ(total >= 1, OTK_ERR_EMPTY_GROUP, "no trajectory on any rank (EmptyGroup)");
  OTK_REQ(total <= (int64_t(1) << 30), OTK_ERR_SHAPE, "global batch too large");
  const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // the union of the shards in rank order: one broadcast per rank and array, fused in one NCCL group
  OTK_NCCL(nccl().GroupStart(), "ncclGroupStart");
  int64_t off = 0;
  ncclResult_t r = ncclSuccess;
  for (int q = 0; q < P && r == ncclSuccess; ++q) {
    if (counts[q] > 0) {
      r = nccl().Broadcast(q == me ? static_cast<const void*>(group_id) : nullptr, gid_all + off, size_t(counts[q]),
                           ncclInt32, q, comm_of(ctx), st);
      if (r == ncclSuccess)
        r = nccl().Broadcast(q == me ? static_cast<const void*>(returns) : nullptr, ret_all + off, size_t(counts[q]),
                             ncclFloat64, q, comm_of(ctx), st);
    }
    off += counts[q];
  }
  const ncclResult_t r2 = nccl().GroupEnd();
  if (r != ncclSuccess) return nccl_fail("ncclBroadcast", r);
  if (r2 != ncclSuccess) return nccl_fail("ncclGroupEnd", r2);
  // step (2) on the whole batch: the same statistics, in the same trajectory order, on every rank
  return otk_group_advantages(ctx, int32_t(total), gid_all, num_groups, ret_all, nullptr, nullptr, flags, std_floor,
                              adv_all, nullptr, group_mean, group_std, group_size, stream);
}

}  // extern "C"
