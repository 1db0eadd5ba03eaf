// Test infrastructure only: an in-process stand-in for libnccl.so.2 so that the library's batch-sharded exchanges
// (paper_2601_07376_b200/csrc/otk_comm.cu, bound through $OTK_NCCL_LIB) run with SEVERAL ranks on a one-GPU box —
// real NCCL refuses two ranks on one device. Ranks are threads of one process sharing the device; every collective
// is a blocking rendezvous: each rank synchronises its stream, posts its buffers, waits for all ranks, then reads
// the others' device buffers with cudaMemcpy and writes its own result, with a second barrier so an in-place
// buffer is not overwritten while a peer still reads it. Only the calls otk_comm.cu uses exist. Not NCCL: no
// overlap, no graphs, no inter-process ranks.
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <vector>

extern "C" {
typedef enum { ncclSuccess = 0, ncclUnhandledCudaError = 1, ncclSystemError = 2, ncclInternalError = 3,
               ncclInvalidArgument = 4, ncclInvalidUsage = 5 } ncclResult_t;
typedef enum { ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclUint32 = 3, ncclInt64 = 4, ncclUint64 = 5,
               ncclFloat16 = 6, ncclFloat32 = 7, ncclFloat64 = 8 } ncclDataType_t;
typedef enum { ncclSum = 0 } ncclRedOp_t;
typedef struct { char internal[128]; } ncclUniqueId;
}

namespace {
struct Group {            // one communicator: nranks threads
  int nranks = 0, joined = 0;
  std::mutex mu;
  std::condition_variable cv;
  int gen = 0, arrived = 0;                     // generation barrier
  std::vector<const void*> send;
  std::vector<cudaStream_t> stream;
};
struct Comm {
  Group* g;
  int rank;
};
std::mutex g_mu;
std::map<std::string, Group*> g_groups;

bool barrier(Group* g) {   // all ranks; false on a 60 s timeout (a rank that never arrived)
  std::unique_lock<std::mutex> lk(g->mu);
  const int my = g->gen;
  if (++g->arrived == g->nranks) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
    return true;
  }
  return g->cv.wait_for(lk, std::chrono::seconds(60), [&] { return g->gen != my; });
}
size_t elem_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}
}  // namespace

extern "C" {
const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "success" : "fake NCCL error"; }

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static int counter = 0;
  std::lock_guard<std::mutex> lk(g_mu);
  std::memset(id, 0, sizeof(*id));
  std::snprintf(id->internal, sizeof(id->internal), "fake-nccl-%d", ++counter);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(void** comm, int nranks, ncclUniqueId id, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  Group* g;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& slot = g_groups[std::string(id.internal, strnlen(id.internal, sizeof(id.internal)))];
    if (!slot) {
      slot = new Group;
      slot->nranks = nranks;
      slot->send.assign(nranks, nullptr);
      slot->stream.assign(nranks, nullptr);
    }
    g = slot;
  }
  if (g->nranks != nranks) return ncclInvalidUsage;
  *comm = new Comm{g, rank};
  return barrier(g) ? ncclSuccess : ncclSystemError;   // blocks until every rank joined, like NCCL
}

ncclResult_t ncclCommDestroy(void* comm) {
  delete static_cast<Comm*>(comm);
  return ncclSuccess;
}
ncclResult_t ncclGroupStart() { return ncclSuccess; }
ncclResult_t ncclGroupEnd() { return ncclSuccess; }

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t type, ncclRedOp_t op,
                           void* comm, cudaStream_t stream) {
  Comm* c = static_cast<Comm*>(comm);
  Group* g = c->g;
  if (op != ncclSum || (type != ncclInt64 && type != ncclFloat64)) return ncclInvalidArgument;
  if (cudaStreamSynchronize(stream) != cudaSuccess) return ncclUnhandledCudaError;
  g->send[c->rank] = send;
  if (!barrier(g)) return ncclSystemError;
  std::vector<char> acc(count * 8, 0), tmp(count * 8);
  for (int r = 0; r < g->nranks; ++r) {   // rank order: the same sum on every rank
    if (cudaMemcpy(tmp.data(), g->send[r], count * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return ncclUnhandledCudaError;
    for (size_t i = 0; i < count; ++i) {
      if (type == ncclInt64) reinterpret_cast<int64_t*>(acc.data())[i] += reinterpret_cast<int64_t*>(tmp.data())[i];
      else reinterpret_cast<double*>(acc.data())[i] += reinterpret_cast<double*>(tmp.data())[i];
    }
  }
  if (!barrier(g)) return ncclSystemError;   // every rank has read every send buffer
  if (cudaMemcpy(recv, acc.data(), count * 8, cudaMemcpyHostToDevice) != cudaSuccess) return ncclUnhandledCudaError;
  return barrier(g) ? ncclSuccess : ncclSystemError;
}

ncclResult_t ncclBroadcast(const void* send, void* recv, size_t count, ncclDataType_t type, int root, void* comm,
                           cudaStream_t stream) {
  Comm* c = static_cast<Comm*>(comm);
  Group* g = c->g;
  if (root < 0 || root >= g->nranks) return ncclInvalidArgument;
  if (cudaStreamSynchronize(stream) != cudaSuccess) return ncclUnhandledCudaError;
  if (c->rank == root) g->send[root] = send;
  if (!barrier(g)) return ncclSystemError;
  const size_t bytes = count * elem_size(type);
  if (bytes && cudaMemcpy(recv, g->send[root], bytes, cudaMemcpyDeviceToDevice) != cudaSuccess)
    return ncclUnhandledCudaError;
  return barrier(g) ? ncclSuccess : ncclSystemError;
}
}  // extern "C"
