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
  int kperm = 0;  // split-bf16 scoring layer fed by a hidden layer: the chain's K-block order
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

// Whole hidden-layer chain of 128-row blocks in one clustered kernel (mlp_chain.cuh; bf16,
// hidden width 512). fwd: relu(A W + b) per layer with head partials at the last layer
// (4 partial tiles); !fwd: dZ chain (dz W^T) * [act > 0].
struct ChainCall {
  bool fwd = true;
  int M = 0, n_layers = 0;
  const void* in = nullptr;  // layer-0 A operand [M][K0] bf16
  long long ld_in = 0;
  int K[8] = {};
  const void* w[8] = {};     // fwd: [K][512]; dgrad: [512][512]
  const float* bias[8] = {};
  void* out[8] = {};
  long long ldo[8] = {};
  const void* mask[8] = {};
  long long ldm[8] = {};
  const float* head_w = nullptr;
  const float* head_u = nullptr;
  float* head_part = nullptr;
  float* head_part2 = nullptr;
  long long head_ld = 0;
  unsigned long long* trace = nullptr;
  // split-bf16 operands (mlp_chain_split.cuh): lo planes of the input, the weights and the outputs
  bool split = false;
  const void* in_lo = nullptr;
  const void* w_lo[8] = {};
  void* out_lo[8] = {};
};
void launch_chain(const ChainCall& c, cudaStream_t s);

// Every level's weight-gradient GEMM in one launch (gemm_group.cuh; bf16), optionally with the
// momentum-SGD update of the produced parameters fused into the epilogue.
struct WgradGroupCall {
  int n = 0, K = 0;
  const void* a[8] = {};
  long long lda[8] = {};
  const void* b[8] = {};
  long long ldb[8] = {};
  int M[8] = {}, N[8] = {};
  float* g[8] = {};
  float* w[8] = {};
  float* mom[8] = {};
  void* shadow[8] = {};
  // split-bf16 operands (MOSES_PREC_BF16X3): lo planes of a / b and the lo half of the shadow
  bool split = false;
  const void* a_lo[8] = {};
  const void* b_lo[8] = {};
  void* shadow_lo[8] = {};
  float lr = 0.f, mu = 0.f;
  bool update = false;
  long long* counter = nullptr;
  const double* loss_src = nullptr;
  double* loss_acc = nullptr;
  double* loss_copy = nullptr;
  float* sk_ws = nullptr;  // split-bf16: L2 workspace of the split-K reduction (wgrad_sk_ws_bytes())
  int max_ctas = 0;        // split-bf16: CTA budget of the launch (0: every SM), e.g. beside a running chain
  int max_split = 8;       // split-bf16: widest cluster (beside a chain only pairs fit the leftover SMs)
};
size_t wgrad_sk_ws_bytes();
void launch_wgrad_group(const WgradGroupCall& c, cudaStream_t s);
extern int g_group;
extern int g_wgrad_sk;
extern int g_wgrad_sk_splits;
extern int g_wgrad_sk_kc;
extern int g_wgrad_early;
extern int g_chain_pair;
extern int g_num_sms;
extern unsigned long long* g_wgrad_sk_trace;
extern int g_rank_fused;  // rank_step (one launch) instead of rank_pairs + rank_finalize
extern int g_chain;  // fused chain enabled (moses_debug_set_chain)

// elem = 2 (bf16, kind::f16) or 4 (fp32 operands, kind::tf32). Returns the N tile used.
int launch_gemm(int elem, const GemmCall& c, cudaStream_t s);
int gemm_pick_bn(int M, int N);

}  // namespace moses
