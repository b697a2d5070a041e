// comm.cu — NCCL loading, communicator lifetime and the collectives the data-parallel and sharded
// scoring paths use: one process per GPU (moses_comm_init_rank, torchrun-style) or
// one process driving n GPUs (moses_comm_init_all, ncclCommInitAll).
#include <dlfcn.h>

#include <mutex>
#include <string>

#include "comm.cuh"

namespace moses {

const NcclApi& nccl() {
  static NcclApi api{};
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) -> void* {
      void* p = dlsym(h, name);
      if (p == nullptr && err.empty()) err = std::string("libnccl.so.2 lacks ") + name;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
  });
  if (!err.empty()) fail(MOSES_ERR_CUDA, err);
  return api;
}

void comm_allreduce_f32(moses_comm* c, float* buf, long long n, bool average, cudaStream_t st) {
  if (c == nullptr || n <= 0) return;
  MOSES_NCCL(nccl().AllReduce(buf, buf, size_t(n), ncclFloat32, average ? ncclAvg : ncclSum, c->comm, st));
}
void comm_allreduce_f64(moses_comm* c, double* buf, long long n, cudaStream_t st) {
  if (c == nullptr || n <= 0) return;
  MOSES_NCCL(nccl().AllReduce(buf, buf, size_t(n), ncclFloat64, ncclSum, c->comm, st));
}
void comm_allgather_f32(moses_comm* c, const float* send, float* recv, long long n, cudaStream_t st) {
  if (c == nullptr || n <= 0) return;
  MOSES_NCCL(nccl().AllGather(send, recv, size_t(n), ncclFloat32, c->comm, st));
}
void comm_allgather_bytes(moses_comm* c, const void* send, void* recv, long long bytes, cudaStream_t st) {
  if (c == nullptr || bytes <= 0) return;
  MOSES_NCCL(nccl().AllGather(send, recv, size_t(bytes), ncclUint8, c->comm, st));
}

}  // namespace moses
