// common.cuh — shared declarations for the Moses B200 library.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/moses_gpu.h"

namespace moses {

// Thrown inside the library, converted to a status code at the C-ABI.
struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Status(code, msg); }

#define MOSES_CUDA(expr)                                                                        \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess)                                                                      \
      ::moses::fail(MOSES_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));       \
  } while (0)

inline int ceil_div(long long a, long long b) { return int((a + b - 1) / b); }
inline long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

// ---------------------------------------------------------------- GEMM launcher (gemm.cu)
struct Operand {
  const void* ptr;
  long long ld;   // row stride in elements of the stored matrix
  bool mn_major;  // true: element (mn, k) at ptr[k*ld + mn]; false: at ptr[mn*ld + k]
  const void* lo = nullptr;  // 3xTF32: low halves, same layout (nullptr: single operand)
};
struct GemmEpilogue;  // fwd decl (gemm.cuh GemmArgs is the device-side form)

enum class EpiKind : int { Fwd = 0, Dgrad = 1, StoreF32 = 2 };

struct GemmCall {
  int M, N, K;
  Operand A, B;
  EpiKind epi;
  void* out;
  long long ldo;
  const float* bias = nullptr;
  int relu = 0;
  const float* head_w = nullptr;
  const float* head_u = nullptr;
  float* head_part = nullptr;
  float* head_part2 = nullptr;
  long long head_ld = 0;
  const void* mask = nullptr;
  long long ldm = 0;
  int bn = 0;  // 0 = auto
  int round_out = 1;  // fp32 outputs: round to tf32 (operand of the next kind::tf32 GEMM)
  void* out_lo = nullptr;  // 3xTF32: low halves of the output
};

// ---------------------------------------------------------------- device-time profiler (capi.cu)
// Optional per-category CUDA-event brackets around launches (off by default; a separate
// profiling pass of bench.py turns it on to attribute step time to kernel classes).
enum ProfCat : int {
  P_GEMM_FWD = 0, P_GEMM_DGRAD, P_GEMM_WGRAD, P_RANK, P_HEAD, P_UPDATE, P_SELECT, P_TOPK, P_OTHER, P_NCAT
};
struct ProfScope {
  int cat;
  cudaStream_t st;
  int idx = -1;
  ProfScope(int c, cudaStream_t s);
  ~ProfScope();
};

// elem = 2 (bf16, kind::f16) or 4 (fp32 operands, kind::tf32). Returns the N tile used.
int launch_gemm(int elem, const GemmCall& c, cudaStream_t s);
int gemm_pick_bn(int M, int N);

}  // namespace moses
