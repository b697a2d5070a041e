// comm.cuh — NCCL communicators behind the C ABI.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"): inside a PyTorch process that is the
// library torch already loaded (one NCCL per process), elsewhere the system one. The product library
// therefore has no link-time NCCL dependency; the moses_comm_* entry points fail loudly
// (MOSES_ERR_CUDA + message) when NCCL cannot be loaded.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include "common.cuh"

struct moses_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

namespace moses {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GetVersion)(int*);
};
const NcclApi& nccl();  // loads on first use; fails (Status) when libnccl.so.2 is unavailable

#define MOSES_NCCL(expr)                                                                              \
  do {                                                                                                \
    const ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess)                                                                            \
      ::moses::fail(MOSES_ERR_CUDA, std::string(#expr) + ": " + ::moses::nccl().GetErrorString(_r)); \
  } while (0)

// in-place collectives on `st` (graph-capturable)
void comm_allreduce_f32(moses_comm* c, float* buf, long long n, bool average, cudaStream_t st);
void comm_allreduce_f64(moses_comm* c, double* buf, long long n, cudaStream_t st);
// recv[r*n .. (r+1)*n) = rank r's send; send may alias recv + rank*n (in place)
void comm_allgather_f32(moses_comm* c, const float* send, float* recv, long long n, cudaStream_t st);
void comm_allgather_bytes(moses_comm* c, const void* send, void* recv, long long bytes, cudaStream_t st);

}  // namespace moses
