// capi.cu — the C ABI (include/moses_gpu.h): device model / adversary handles
// and the reference-facing operations, each composed from the sm_100a kernels.
//
// Device data layout:
//   params / grads / momentum / xi : fp32, the reference flat order (lottery.hpp:13-14)
//   weight operand                 : bf16 shadow of params (BF16 mode) or params itself (TF32 mode);
//                                    level l's block [in][out] is the GEMM B operand, MN-major for the
//                                    forward pass and K-major for the data-gradient pass.
//   activations act[l]             : rows x ld[l], column dims[l] == 1.0 (bias row of the wgrad GEMM),
//                                    row block [0, m) = adversary replay rows, [m, m+n) = batch rows.
//   dZ[l]                          : rows x lddz[l]
#include <algorithm>
#include <atomic>
#include <bit>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_set>
#include <thread>
#include <vector>

#include "comm.cuh"
#include "common.cuh"
#include "kernels.cuh"
#include "pipeline.cuh"

namespace moses {

std::atomic<long long> g_launches{0};
void note_launch(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---- profiler
struct Profiler {
  std::mutex mu;
  bool on = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> rec;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
};
static Profiler& prof() {
  static Profiler p;
  return p;
}
ProfScope::ProfScope(int c, cudaStream_t s) : cat(c), st(s) {
  Profiler& p = prof();
  if (!p.on) return;
  std::lock_guard<std::mutex> lk(p.mu);
  std::pair<cudaEvent_t, cudaEvent_t> ev;
  if (!p.pool.empty()) {
    ev = p.pool.back();
    p.pool.pop_back();
  } else {
    cudaEventCreate(&ev.first);
    cudaEventCreate(&ev.second);
  }
  idx = int(p.rec.size());
  p.rec.push_back({c, ev});
  cudaEventRecord(ev.first, s);
}
ProfScope::~ProfScope() {
  if (idx < 0) return;
  Profiler& p = prof();
  std::lock_guard<std::mutex> lk(p.mu);
  cudaEventRecord(p.rec[idx].second.second, st);
}

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MOSES_OK;
  } catch (const Status& s) {
    g_err = s.what();
    return s.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MOSES_ERR_INVALID_ARG;
  }
}

template <typename T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  MOSES_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return static_cast<T*>(p);
}
void dfree(void* p) {
  if (p) cudaFree(p);
}

// ---- reference-side validation helpers (model.cpp:20-37)
void check_dims(const int32_t* dims, int nd, bool strict) {
  if (dims == nullptr || (strict ? nd != 4 : nd < 3))
    fail(MOSES_ERR_BAD_DIMS, "expected 4 levels, got " + std::to_string(nd));
  for (int i = 0; i < nd; ++i)
    if (dims[i] <= 0) fail(MOSES_ERR_BAD_DIMS, "non-positive level width");
  if (dims[nd - 1] != 1) fail(MOSES_ERR_BAD_DIMS, "output width must be 1");
}
long long level_off(const std::vector<int>& d, int l) {
  long long o = 0;
  for (int k = 0; k < l; ++k) o += (long long)d[k] * d[k + 1] + d[k + 1];
  return o;
}

// ---- keyed SplitMix64 (rng.hpp:16-80) for host-side init
struct KeyBuilder {
  uint64_t h = 0xcbf29ce484222325ull;
  void step(unsigned char b) { h ^= b; h *= 0x100000001b3ull; }
  KeyBuilder& add(uint64_t v) {
    for (int i = 0; i < 8; ++i) step((unsigned char)(v >> (8 * i)));
    return *this;
  }
  KeyBuilder& add(const char* s) {
    for (; *s; ++s) step((unsigned char)*s);
    step(0);
    return *this;
  }
};
struct Rng {
  uint64_t s;
  uint64_t next() {
    s += 0x9e3779b97f4a7c15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double u01() { return double(next() >> 11) * 0x1.0p-53; }
};

// Scratch context for the handle-less entry points (ranking loss, top-k, pooling, MMD, ...).
struct Scratch {
  std::mutex mu;
  cudaStream_t st = nullptr;
  void* buf = nullptr;
  size_t cap = 0;
  long long* host = nullptr;      // pinned, mapped: the top-k result (conclusive flag + indices)
  long long* host_dev = nullptr;  // its device address (the kernel writes it directly)
  long long* pinned() {
    if (!host) {
      MOSES_CUDA(cudaHostAlloc(&host, sizeof(long long) * (kTopkMax + 1), cudaHostAllocPortable | cudaHostAllocMapped));
      MOSES_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&host_dev), host, 0));
    }
    return host;
  }
  void* ensure(size_t bytes) {
    if (!st) MOSES_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    if (bytes > cap) {
      dfree(buf);
      buf = nullptr;
      cap = 0;
      MOSES_CUDA(cudaMalloc(&buf, bytes));
      cap = bytes;
    }
    return buf;
  }
};
// one scratch context per device (a process may drive several GPUs: moses_comm_init_all)
Scratch& scratch() {
  constexpr int kMaxDev = 64;
  static Scratch s[kMaxDev];
  int dev = 0;
  MOSES_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) fail(MOSES_ERR_NO_DEVICE, "device ordinal out of range");
  return s[dev];
}

struct Carver {
  uint8_t* p;
  template <typename T>
  T* take(size_t count) {
    T* r = reinterpret_cast<T*>(p);
    p += round_up(count * sizeof(T) + 1, 256);
    return r;
  }
};

}  // namespace
}  // namespace moses

using namespace moses;

struct moses_adversary {
  int D = 0, W = 0;
  long long m = 0;
  float* replay = nullptr;  // m x D fp32 (device)
  float* u = nullptr;       // [W] + c at u[W]... kept separate:
  float* c = nullptr;       // [1]
  float eta = 0.1f;
  ~moses_adversary() {
    dfree(replay);
    dfree(u);
    dfree(c);
  }
};

struct moses_model {
  std::vector<int> dims;
  int L = 0;  // levels
  long long P = 0;
  std::vector<long long> off;
  int prec = MOSES_PREC_BF16;
  int device = 0;  // CUDA device the handle's streams and buffers live on (current device at create)
  int esz = 2;
  // split operands: every GEMM operand buffer has a low twin (hi plane, then lo plane at + cap*ld):
  // MOSES_PREC_FP32 = 3xTF32 (esz 4), MOSES_PREC_BF16X3 = split bf16 (esz 2, fused chain kernels only)
  bool split = false;
  long long cap = 0;
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;      // weight-gradient side stream
  std::vector<cudaEvent_t> evs;   // fork / dz-ready / join events of the two-stream backward
  // CUDA graph of one device-resident training step (moses_train_graph_*)
  cudaGraphExec_t train_exec = nullptr;
  long long* dcounter = nullptr;   // device batch index consumed by the graph's gather kernel
  // pooled training graphs alternate two batch buffers: graph k computes on one while a side
  // branch gathers batch k+1 into the other (moses_train_graph_create_pooled)
  cudaGraphExec_t train_exec2 = nullptr;
  int train_parity = 0;
  long long* pcounter = nullptr;   // next batch to prefetch
  cudaStream_t st3 = nullptr;
  cudaStream_t st4 = nullptr;      // head gradient / head-block update beside the early weight gradient
  double* host_sc = nullptr;       // pinned: per-call scalars read back without a blocking pageable copy
  cudaEvent_t pf_fork = nullptr, pf_join = nullptr;
  struct BatchBuf {
    void* act = nullptr;           // hi plane; split handles: lo plane at + cap * ld[0] elements
    float* labels = nullptr;
    long long* seg_off = nullptr;
    int* seg_rows = nullptr;
  } alt;
  // asynchronous host-input pooled step (moses_train_step_pooled_async): three staging slots
  struct AsyncSlot {
    double* x = nullptr;           // device float64 statement rows (cap x D)
    double* y = nullptr;           // device float64 labels (cap)
    long long* off = nullptr;      // device CSR offsets (cap + 1)
    long long* dims = nullptr;     // device {n_stmt, programs}
    long long* dims_host = nullptr;  // pinned source of dims
    cudaEvent_t ready = nullptr, free = nullptr;
    bool used = false;
    cudaGraphExec_t exec = nullptr;
    long long programs = -1;
    float lr = 0.f, mu = 0.f;
    double* box_host = nullptr;    // loss mailbox written by the slot's graph (mapped pinned)
    double* box_dev = nullptr;
    double* pending = nullptr;     // caller's loss_out for the slot's step in flight
    // the slot's packed batch (layer-0 rows [hi | lo], labels, CSR offsets, row -> program): packed on
    // the copy stream right after the upload, while the previous step still computes
    void* act = nullptr;
    float* labels = nullptr;
    long long* seg_off = nullptr;
    int* seg_rows = nullptr;
  } aslot[3];  // three slots: the host may run two steps ahead of the device
  cudaStream_t st_copy = nullptr;
  long long async_steps = 0;
  // epoch over a ranking-batch plan (moses_train_plan_device)
  struct PlanState {
    long long* rows = nullptr;     // device row indices
    long long* off = nullptr;      // device batch offsets
    long long* counter = nullptr;  // device batch index
    double* loss_sum = nullptr;    // device running sum of batch losses
    float* stage = nullptr;        // FP32 handles: gathered fp32 rows before the hi/lo split
    long long cap_rows = 0, cap_b = 0;
    cudaGraphExec_t exec = nullptr;
    const void* x = nullptr;
    const float* y = nullptr;
    long long ldx = 0, batch = 0;
    float lr = 0.f, mu = 0.f;
    long long graph_kernels = 0;
  } plan;
  float* gbias = nullptr;          // pooled head-bias gradient (device scalar)
  float* wgsk_ws = nullptr;        // split bf16: L2 workspace of the split-K weight-gradient reduction
  float* mmd_g = nullptr;          // MMD loss: d MMD^2 / dH of every row (cap x W)
  double* mmd_v = nullptr;         // MMD loss: per-row value partials (cap)
  // data parallel (moses_model_set_comm): 1 = average the gradients of every rank's own batch
  // (throughput mode), 2 = exact batch (the global batch is the rank-ordered concatenation of every
  // rank's rows; scores all-gathered, pair terms of the own rows, gradients summed)
  moses_comm* comm = nullptr;
  int comm_mode = 0;
  float* dp_s = nullptr;           // exact mode: all-gathered scores / labels of the global batch
  float* dp_y = nullptr;
  double* dp_tot = nullptr;        // exact mode: (loss sum, pair count) partials -> global
  long long dp_cap = 0;
  const void* dp_x0 = nullptr;     // exact mode: the local rows of the step in flight
  long long dp_ld0 = 0, dp_n = 0;
  void* lot_ws = nullptr;          // fused lottery-step workspace (lottery.cu)
  long long* seg_off = nullptr;    // pooled: device CSR offsets of the current batch (cap+1)
  int* seg_rows = nullptr;         // pooled: program of each statement row (cap)
  unsigned int* rank_ticket = nullptr;  // rank_step last-CTA ticket (self re-arming)
  long long rank_ws_rows = 0;           // ranking workspace sized for batches of this many rows
  std::vector<void*> retired;           // outgrown workspaces (captured graphs may still point at them)
  // parameters
  float *w = nullptr, *mom = nullptr, *g = nullptr, *xi = nullptr;
  float *m1 = nullptr, *m2 = nullptr;
  uint8_t* mask = nullptr;
  __nv_bfloat16* wbf = nullptr;  // bf16 operand shadow (BF16 mode)
  float* wtf = nullptr;          // tf32-rounded operand shadow (TF32 mode; FP32 mode: [hi P | lo P])
  bool xi_valid = false, xi_norm = false, mask_valid = false;
  // activations
  std::vector<void*> act, dz;
  std::vector<long long> ld, lddz;
  int max_tiles = 0;
  float *head_part = nullptr, *head_part2 = nullptr;
  float *scores = nullptr, *labels = nullptr, *coefA = nullptr, *coefB = nullptr;
  RankWs rank{};
  double* dscal = nullptr;  // [0] loss, [1] ce, [2..] scratch
  long long* dpairs = nullptr;
  unsigned long long* dcount = nullptr;
  void* sel_base = nullptr;
  SelectWs sel{};
  double* staging = nullptr;  // host-double staging [cap * stage_w]
  long long stage_w = 0;
  float* adv_ws = nullptr;
  int last_tiles = 0;  // N tiles of the last hidden GEMM of the most recent forward

  const void* wop(int l) const {
    return esz == 2 ? static_cast<const void*>(wbf + off[l]) : static_cast<const void*>(wtf + off[l]);
  }
  bool bsplit() const { return split && esz == 2; }  // MOSES_PREC_BF16X3
  // element type of device-resident input rows (moses_*_device, training graphs, plans): the operand
  // type, except split-bf16 handles, which take fp32 rows and split them into their hi/lo planes
  int in_esz() const { return bsplit() ? 4 : esz; }
  // shadow written by the generic update kernels; split modes refresh the hi/lo pair afterwards
  // (post_update); the fused training step writes the split-bf16 pair itself
  Shadow shadow() const { return esz == 2 ? (split ? Shadow{nullptr, 0} : Shadow{wbf, 1}) : (split ? Shadow{nullptr, 0} : Shadow{wtf, 2}); }
  Shadow shadow_full() const {
    return split ? (esz == 2 ? Shadow{wbf, 4, shadow_lo_offset(P)} : Shadow{wtf, 3}) : shadow();
  }
  const void* wop_lo(int l) const {
    if (!split) return nullptr;
    return esz == 2 ? static_cast<const void*>(wbf + shadow_lo_offset(P) + off[l])
                    : static_cast<const void*>(wtf + shadow_lo_offset(P) + off[l]);
  }
  void* act_lo(int l) const { return split ? static_cast<uint8_t*>(act[l]) + cap * ld[l] * esz : nullptr; }
  void* dz_lo(int l) const { return split ? static_cast<uint8_t*>(dz[l]) + cap * lddz[l] * esz : nullptr; }
  template <typename T>
  T* act_lo_t(int l) const { return static_cast<T*>(act_lo(l)); }
  template <typename T>
  T* dz_lo_t(int l) const { return static_cast<T*>(dz_lo(l)); }
  // lo plane of a layer-0 operand buffer (act[0] or the alternate batch buffer)
  const void* x0_lo(const void* x0) const {
    if (!split) return nullptr;
    if (x0 == act[0]) return act_lo(0);
    if (alt.act != nullptr && x0 == alt.act) return static_cast<const uint8_t*>(alt.act) + cap * ld[0] * esz;
    for (const auto& a : aslot)
      if (a.act != nullptr && x0 == a.act) return static_cast<const uint8_t*>(a.act) + cap * ld[0] * esz;
    fail(MOSES_ERR_INVALID_ARG, "split-operand handles take layer-0 rows from their own packed buffers");
  }
  void post_update() {  // FP32 mode: hi/lo operand pair of the updated parameters
    if (split) refresh_shadow(w, P, shadow_full(), st);
  }
  int width(int l) const { return dims[l]; }
  int W() const { return dims[L - 1]; }
  const float* head_w() const { return w + off[L - 1]; }
  const float* head_b() const { return w + off[L - 1] + dims[L - 1]; }
  const float* bias(int l) const { return w + off[l] + (long long)dims[l] * dims[l + 1]; }

  ~moses_model() {
    if (st) cudaStreamSynchronize(st);
    for (void* p : {(void*)w, (void*)mom, (void*)g, (void*)xi, (void*)m1, (void*)m2, (void*)mask, (void*)wbf, (void*)wtf,
                    (void*)head_part, (void*)head_part2, (void*)scores, (void*)labels, (void*)coefA, (void*)coefB,
                    (void*)rank.gs_part, (void*)rank.loss_part, (void*)rank.pairs_part, (void*)dscal, (void*)dpairs,
                    (void*)dcount, sel_base, (void*)staging, (void*)adv_ws, (void*)wgsk_ws})
      dfree(p);
    for (void* p : act) dfree(p);
    for (void* p : dz) dfree(p);
    if (train_exec) cudaGraphExecDestroy(train_exec);
    if (train_exec2) cudaGraphExecDestroy(train_exec2);
    dfree(pcounter);
    dfree(alt.act);
    dfree(alt.labels);
    dfree(alt.seg_off);
    dfree(alt.seg_rows);
    if (pf_fork) cudaEventDestroy(pf_fork);
    if (pf_join) cudaEventDestroy(pf_join);
    if (st3) cudaStreamDestroy(st3);
    if (st4) cudaStreamDestroy(st4);
    if (host_sc) cudaFreeHost(host_sc);
    for (auto& a : aslot) {
      if (a.exec) cudaGraphExecDestroy(a.exec);
      dfree(a.x);
      dfree(a.y);
      dfree(a.off);
      dfree(a.dims);
      dfree(a.act);
      dfree(a.labels);
      dfree(a.seg_off);
      dfree(a.seg_rows);
      if (a.dims_host) cudaFreeHost(a.dims_host);
      if (a.box_host) cudaFreeHost(a.box_host);
      if (a.ready) cudaEventDestroy(a.ready);
      if (a.free) cudaEventDestroy(a.free);
    }
    if (st_copy) cudaStreamDestroy(st_copy);
    if (plan.exec) cudaGraphExecDestroy(plan.exec);
    dfree(plan.rows);
    dfree(plan.off);
    dfree(plan.counter);
    dfree(plan.loss_sum);
    dfree(plan.stage);
    dfree(dcounter);
    dfree(gbias);
    dfree(mmd_g);
    dfree(mmd_v);
    dfree(dp_s);
    dfree(dp_y);
    dfree(dp_tot);
    dfree(lot_ws);
    dfree(seg_off);
    dfree(seg_rows);
    dfree(rank_ticket);
    for (void* p : retired) dfree(p);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    if (st2) cudaStreamDestroy(st2);
    if (st) cudaStreamDestroy(st);
  }
};

namespace moses {
namespace {

// ---------------------------------------------------------------- forward / backward composition
// Fused hidden-layer chain (mlp_chain.cuh): bf16, every hidden width 512, input width <= 512.
// The fused chain is a latency design (training batches, ~2.3K statement rows); scoring chunks of
// 64K rows run layer by layer on the persistent tcgen05 kernels (2x faster there, tools/gemm_sweep.py).
constexpr long long kChainMaxRows = 16384;
bool chain_ok(const moses_model* m) {
  if (!g_chain || m->esz != 2 || m->L - 1 < 1 || m->L - 1 > 8 || m->dims[0] > 512) return false;
  for (int l = 1; l < m->L; ++l)
    if (m->dims[l] != 512) return false;
  return true;
}

template <typename T>
void forward_rows(moses_model* m, const void* x0, long long ldx0, long long R, const float* head_u, bool keep_last) {
  if (m->split && x0 != m->act[0] && x0 != m->alt.act && x0 != m->aslot[0].act && x0 != m->aslot[1].act &&
      x0 != m->aslot[2].act)
    fail(MOSES_ERR_INVALID_ARG, "split-operand handles take inputs through their packed buffers");
  if (m->bsplit() && !chain_ok(m))
    fail(MOSES_ERR_INVALID_ARG, "split-bf16 handles need hidden widths of 512 and input width <= 512");
  if (chain_ok(m) && R > 0 && R <= kChainMaxRows) {
    // the fused chain: a latency design for training batches; above kChainMaxRows rows (candidate-pool
    // scoring) the layers run one by one on the throughput kernels (split bf16: umma_fwd_pair_split)
    const void* x0_lo = m->x0_lo(x0);
    for (long long r0 = 0; r0 < R; r0 += kChainMaxRows) {
      const long long Rc = std::min(kChainMaxRows, R - r0);
      const size_t es = size_t(m->esz);
      auto at = [&](const void* p, long long ld) -> void* {
        return p ? const_cast<uint8_t*>(static_cast<const uint8_t*>(p)) + size_t(r0) * size_t(ld) * es : nullptr;
      };
      ChainCall cc;
      cc.fwd = true;
      cc.M = int(Rc);
      cc.n_layers = m->L - 1;
      cc.in = at(x0, ldx0);
      cc.ld_in = ldx0;
      cc.split = m->bsplit();
      cc.in_lo = at(x0_lo, ldx0);
      for (int l = 0; l + 1 < m->L; ++l) {
        cc.K[l] = m->dims[l];
        cc.w[l] = m->wop(l);
        cc.w_lo[l] = m->wop_lo(l);
        cc.bias[l] = m->bias(l);
        const bool keep = !(l + 2 == m->L && !keep_last);
        cc.out[l] = keep ? at(m->act[l + 1], m->ld[l + 1]) : nullptr;
        cc.out_lo[l] = keep ? at(m->act_lo(l + 1), m->ld[l + 1]) : nullptr;
        cc.ldo[l] = m->ld[l + 1];
      }
      cc.head_w = m->head_w();
      cc.head_u = head_u;
      cc.head_part = m->head_part + r0;
      cc.head_part2 = head_u ? m->head_part2 + r0 : nullptr;
      cc.head_ld = m->cap;
      {
        ProfScope ps(P_GEMM_FWD, m->st);
        launch_chain(cc, m->st);
      }
      note_launch(1);
    }
    m->last_tiles = m->bsplit() ? 8 : 4;  // split chain: per-64-column head partials
    return;
  }
  for (int l = 0; l + 1 < m->L; ++l) {
    GemmCall c{};
    c.M = int(R);
    c.N = m->dims[l + 1];
    c.K = m->dims[l];
    c.A = {l == 0 ? x0 : m->act[l], l == 0 ? ldx0 : m->ld[l], false, l == 0 ? m->x0_lo(x0) : m->act_lo(l)};
    c.B = {m->wop(l), m->dims[l + 1], true, m->wop_lo(l)};
    c.epi = EpiKind::Fwd;
    const bool last = l + 2 == m->L;
    c.out = (last && !keep_last) ? nullptr : m->act[l + 1];
    c.ldo = m->ld[l + 1];
    c.bias = m->bias(l);
    c.relu = 1;
    c.round_out = !last;  // the last hidden layer is never a GEMM operand: keep it full fp32
    c.kperm = l > 0;      // split bf16: the fused chain's K-block order for layers fed by a hidden layer
    if (!last || (m->bsplit() && c.out != nullptr)) c.out_lo = m->act_lo(l + 1);  // split bf16 keeps both planes
    if (last) {
      c.head_w = m->head_w();
      c.head_u = head_u;
      c.head_part = m->head_part;
      c.head_part2 = head_u ? m->head_part2 : nullptr;
      c.head_ld = m->cap;
    }
    int bn;
    {
      ProfScope ps(P_GEMM_FWD, m->st);
      bn = launch_gemm(m->esz, c, m->st);
    }
    note_launch(1);
    if (last) m->last_tiles = ceil_div(c.N, bn);
  }
}

struct SgdFuse {  // momentum-SGD step fused into the grouped weight-gradient epilogue
  float lr, mu;
  long long* counter = nullptr;      // training graphs: batch index to advance with the step
  const double* loss_src = nullptr;  // plan epochs: loss to add into loss_acc with the step
  double* loss_acc = nullptr;
  double* loss_copy = nullptr;       // async steps: per-slot loss mailbox (mapped pinned memory)
  mutable bool folded = false;       // set when the grouped wgrad kernel took the bookkeeping
};

// Returns true when `fuse` was applied (every parameter updated) inside the backward pass.
template <typename T>
bool backward_rows(moses_model* m, const void* x0, long long ldx0, long long R, const float* u,
                   const float* gb_override = nullptr, const SgdFuse* fuse = nullptr, const float* extra = nullptr,
                   float extra_scale = 0.f) {
  // Two streams: the data-gradient chain (head backward -> dgrad(L-2) -> ... -> dgrad(1)) runs on
  // st; every weight-gradient GEMM (and the head-gradient column reduction) runs on st2 as soon
  // as its dZ is ready. At batch 512 each GEMM fills only 16-40 of the 148 SMs, so the two
  // chains overlap almost perfectly.
  const int L = m->L, W = m->W();
  T* hl = static_cast<T*>(m->act[L - 1]);
  cudaEvent_t* ev = m->evs.data();  // ev[0] fork, ev[1 + l] "dz[l] ready", ev[L + 1] join
  MOSES_CUDA(cudaEventRecord(ev[0], m->st));
  MOSES_CUDA(cudaStreamWaitEvent(m->st2, ev[0], 0));
  // split bf16 beside the dZ chain: the last hidden level's weight gradient needs only the head
  // backward's dZ, so it runs on the SMs the chain leaves free while the chain computes the others;
  // it goes first on the side stream (the head-gradient reduction and head-block update follow it)
  const bool chain_path = sizeof(T) == 2 && chain_ok(m) && L - 2 >= 1 && (R <= kChainMaxRows || m->bsplit());
  int free_sms = 0;
  bool early_ok = false;
  if (chain_path && m->bsplit() && g_group && L - 1 <= 8 && g_wgrad_sk && g_wgrad_early) {
    const int chain_ctas = 4 * int(std::min<long long>(ceil_div(R, 128), ceil_div(kChainMaxRows, 128)));
    free_sms = g_num_sms - chain_ctas;
    const int tiles = ceil_div(m->dims[L - 2], 128) * ceil_div(m->dims[L - 1], 256);
    early_ok = free_sms >= 4 * tiles;
  }
  auto head_grad = [&](cudaStream_t hs) {
    ProfScope ps(P_HEAD, hs);
    column_dot<T>(m->coefA, hl, m->ld[L - 1], R, W, m->g + m->off[L - 1], m->adv_ws, hs, gb_override,
                  m->act_lo_t<T>(L - 1));
  };
  if (!early_ok) head_grad(m->st2);
  {
    ProfScope ps(P_HEAD, m->st);
    head_backward<T>(m->coefA, m->coefB, m->head_w(), u, hl, m->ld[L - 1], R, W, static_cast<T*>(m->dz[L - 1]),
                     m->lddz[L - 1], m->st, m->dz_lo_t<T>(L - 1), extra, extra_scale);
  }
  MOSES_CUDA(cudaEventRecord(ev[1 + (L - 1)], m->st));
  note_launch(2);
  // dZ chain dz[L-2] .. dz[1] in one clustered kernel when the shape allows (mlp_chain.cuh); split-bf16
  // handles run it in row chunks of at most kChainMaxRows
  const bool chain = sizeof(T) == 2 && chain_ok(m) && L - 2 >= 1 && (R <= kChainMaxRows || m->bsplit());
  if (m->bsplit() && !(g_group && L - 1 <= 8))
    fail(MOSES_ERR_INVALID_ARG, "split-bf16 handles need the grouped weight-gradient kernel");
  if (chain) {
    for (long long r0 = 0; r0 < R; r0 += kChainMaxRows) {
      const long long Rc = std::min(kChainMaxRows, R - r0);
      auto at = [&](const void* p, long long ld) -> void* {
        return p ? const_cast<uint8_t*>(static_cast<const uint8_t*>(p)) + size_t(r0) * size_t(ld) * sizeof(T) : nullptr;
      };
      ChainCall cc;
      cc.fwd = false;
      cc.M = int(Rc);
      cc.n_layers = L - 2;
      cc.in = at(m->dz[L - 1], m->lddz[L - 1]);
      cc.ld_in = m->lddz[L - 1];
      cc.split = m->bsplit();
      cc.in_lo = at(m->dz_lo(L - 1), m->lddz[L - 1]);
      for (int j = 0; j < L - 2; ++j) {
        const int lev = L - 2 - j;
        cc.K[j] = m->dims[lev + 1];
        cc.w[j] = m->wop(lev);
        cc.w_lo[j] = m->wop_lo(lev);
        cc.out[j] = at(m->dz[lev], m->lddz[lev]);
        cc.out_lo[j] = at(m->dz_lo(lev), m->lddz[lev]);
        cc.ldo[j] = m->lddz[lev];
        cc.mask[j] = at(m->act[lev], m->ld[lev]);
        cc.ldm[j] = m->ld[lev];
      }
      {
        ProfScope ps(P_GEMM_DGRAD, m->st);
        launch_chain(cc, m->st);
      }
      note_launch(1);
    }
    MOSES_CUDA(cudaEventRecord(ev[1 + 1], m->st));  // every dz[l], l <= L-2, is ready
  }
  // bf16: all weight-gradient GEMMs in one launch once every dZ exists (gemm_group.cuh)
  const bool grouped = sizeof(T) == 2 && g_group && L - 1 <= 8;
  if (grouped) {
    for (int l = L - 2; l >= 1 && !chain; --l) {
      GemmCall dg{};
      dg.M = int(R);
      dg.N = m->dims[l];
      dg.K = m->dims[l + 1];
      dg.A = {m->dz[l + 1], m->lddz[l + 1], false};
      dg.B = {m->wop(l), m->dims[l + 1], false};
      dg.epi = EpiKind::Dgrad;
      dg.out = m->dz[l];
      dg.ldo = m->lddz[l];
      dg.mask = m->act[l];
      dg.ldm = m->ld[l];
      {
        ProfScope ps(P_GEMM_DGRAD, m->st);
        launch_gemm(m->esz, dg, m->st);
      }
      note_launch(1);
    }
    auto head_update = [&](cudaStream_t hs) {  // the head block (gradient from column_dot) once head_backward read it
      if (!fuse) return;
      MOSES_CUDA(cudaStreamWaitEvent(hs, ev[1 + (L - 1)], 0));
      const long long o = m->off[L - 1];
      ProfScope ps(P_UPDATE, hs);
      sgd_update(m->w + o, m->mom + o, m->g + o, nullptr, m->P - o, fuse->lr, fuse->mu, true,
                 m->bsplit() ? Shadow{m->wbf + o, 4, shadow_lo_offset(m->P)} : Shadow{m->wbf + o, 1}, hs);
      note_launch(1);
    };
    if (!early_ok) head_update(m->st2);
    int early = 0;
    if (early_ok) {
      const int lev = L - 2;
      {
        WgradGroupCall we;
        we.n = 1;
        we.K = int(R);
        we.split = true;
        we.sk_ws = m->wgsk_ws;
        we.max_ctas = free_sms;
        we.max_split = 4;  // 4-CTA clusters fit the SMs the chain's 4-CTA clusters leave free
        we.a[0] = m->act[lev];
        we.lda[0] = m->ld[lev];
        we.b[0] = m->dz[lev + 1];
        we.ldb[0] = m->lddz[lev + 1];
        we.M[0] = m->dims[lev] + 1;
        we.N[0] = m->dims[lev + 1];
        we.g[0] = m->g + m->off[lev];
        we.w[0] = m->w + m->off[lev];
        we.mom[0] = m->mom + m->off[lev];
        we.shadow[0] = m->wbf + m->off[lev];
        we.a_lo[0] = m->act_lo(lev);
        we.b_lo[0] = m->dz_lo(lev + 1);
        we.shadow_lo[0] = m->wbf + shadow_lo_offset(m->P) + m->off[lev];
        // gradient only: the dZ chain's first layer reads this level's weights (their operand shadow)
        // while the launch runs, so the level's update waits for the chain (below, on the fourth stream)
        MOSES_CUDA(cudaStreamWaitEvent(m->st2, ev[1 + (L - 1)], 0));
        {
          ProfScope ps(P_GEMM_WGRAD, m->st2);
          launch_wgrad_group(we, m->st2);
        }
        MOSES_CUDA(cudaEventRecord(ev[L + 3], m->st2));  // the early level's gradient exists
        note_launch(1);
        early = 1;
      }
      // the head gradient and head-block update on a fourth stream (joined before the step ends), so
      // neither the early nor the remaining weight-gradient launch queues behind them
      if (!m->st4) MOSES_CUDA(cudaStreamCreateWithFlags(&m->st4, cudaStreamNonBlocking));
      MOSES_CUDA(cudaStreamWaitEvent(m->st4, ev[0], 0));
      head_grad(m->st4);
      head_update(m->st4);
    }
    MOSES_CUDA(cudaEventRecord(ev[1], m->st));
    if (early) {
      if (fuse) {  // the early level's update once the chain has read its weights (and its gradient exists)
        const int lev = L - 2;
        const long long o = m->off[lev], cnt = m->off[lev + 1] - o;
        MOSES_CUDA(cudaStreamWaitEvent(m->st4, ev[1], 0));
        MOSES_CUDA(cudaStreamWaitEvent(m->st4, ev[L + 3], 0));
        ProfScope ps(P_UPDATE, m->st4);
        sgd_update(m->w + o, m->mom + o, m->g + o, nullptr, cnt, fuse->lr, fuse->mu, true,
                   Shadow{m->wbf + o, 4, shadow_lo_offset(m->P)}, m->st4);
        note_launch(1);
      }
      MOSES_CUDA(cudaEventRecord(ev[L + 2], m->st4));
    }
    MOSES_CUDA(cudaStreamWaitEvent(m->st2, ev[1], 0));
    WgradGroupCall wc;
    wc.n = L - 1 - early;
    wc.K = int(R);
    wc.split = m->bsplit();
    wc.sk_ws = m->wgsk_ws;
    if (fuse) {
      wc.counter = fuse->counter;
      wc.loss_src = fuse->loss_src;
      wc.loss_acc = fuse->loss_acc;
      wc.loss_copy = fuse->loss_copy;
      fuse->folded = true;
    }
    for (int l = 0; l + 1 < L - early; ++l) {
      wc.a[l] = l == 0 ? x0 : m->act[l];
      wc.lda[l] = l == 0 ? ldx0 : m->ld[l];
      wc.b[l] = m->dz[l + 1];
      wc.ldb[l] = m->lddz[l + 1];
      wc.M[l] = m->dims[l] + 1;  // + the ones column -> bias gradient row
      wc.N[l] = m->dims[l + 1];
      wc.g[l] = m->g + m->off[l];
      wc.w[l] = m->w + m->off[l];
      wc.mom[l] = m->mom + m->off[l];
      wc.shadow[l] = m->wbf + m->off[l];
      if (wc.split) {
        wc.a_lo[l] = l == 0 ? m->x0_lo(x0) : m->act_lo(l);
        wc.b_lo[l] = m->dz_lo(l + 1);
        wc.shadow_lo[l] = m->wbf + shadow_lo_offset(m->P) + m->off[l];
      }
    }
    if (fuse) {
      wc.update = true;
      wc.lr = fuse->lr;
      wc.mu = fuse->mu;
    }
    {
      ProfScope ps(P_GEMM_WGRAD, m->st2);
      launch_wgrad_group(wc, m->st2);
    }
    note_launch(1);
    MOSES_CUDA(cudaEventRecord(ev[L + 1], m->st2));
    MOSES_CUDA(cudaStreamWaitEvent(m->st, ev[L + 1], 0));
    if (early) MOSES_CUDA(cudaStreamWaitEvent(m->st, ev[L + 2], 0));
    return fuse != nullptr;
  }
  for (int l = L - 2; l >= 0; --l) {
    const void* a = l == 0 ? x0 : m->act[l];
    const long long lda = l == 0 ? ldx0 : m->ld[l];
    GemmCall wg{};
    wg.M = m->dims[l] + 1;  // + the ones column -> bias gradient row (flat layout: W block then b)
    wg.N = m->dims[l + 1];
    wg.K = int(R);
    wg.A = {a, lda, true, m->act_lo(l)};
    wg.B = {m->dz[l + 1], m->lddz[l + 1], true, m->dz_lo(l + 1)};
    wg.epi = EpiKind::StoreF32;
    wg.out = m->g + m->off[l];
    wg.ldo = m->dims[l + 1];
    MOSES_CUDA(cudaStreamWaitEvent(m->st2, ev[(chain && l + 1 < L - 1) ? 2 : 1 + (l + 1)], 0));
    {
      ProfScope ps(P_GEMM_WGRAD, m->st2);
      launch_gemm(m->esz, wg, m->st2);
    }
    note_launch(1);
    if (l > 0 && !chain) {
      GemmCall dg{};
      dg.M = int(R);
      dg.N = m->dims[l];
      dg.K = m->dims[l + 1];
      dg.A = {m->dz[l + 1], m->lddz[l + 1], false, m->dz_lo(l + 1)};
      dg.B = {m->wop(l), m->dims[l + 1], false, m->wop_lo(l)};
      dg.epi = EpiKind::Dgrad;
      dg.out = m->dz[l];
      dg.out_lo = m->dz_lo(l);
      dg.ldo = m->lddz[l];
      dg.mask = m->act[l];
      dg.ldm = m->ld[l];
      {
        ProfScope ps(P_GEMM_DGRAD, m->st);
        launch_gemm(m->esz, dg, m->st);
      }
      MOSES_CUDA(cudaEventRecord(ev[1 + l], m->st));
      note_launch(1);
    }
  }
  MOSES_CUDA(cudaEventRecord(ev[L + 1], m->st2));
  MOSES_CUDA(cudaStreamWaitEvent(m->st, ev[L + 1], 0));
  return false;
}

// apply_update is synchronous for host callers (reference value semantics); the device-resident
// DP loop (bench, moses_set_async) keeps it asynchronous on the handle's stream.
thread_local bool g_async = false;
bool sync_updates() { return !g_async; }

void require_model(moses_model* m) {
  if (!m) fail(MOSES_ERR_INVALID_ARG, "null model handle");
}

// Pack host double rows into act[0] rows [row0, row0+n).
void upload_rows(moses_model* m, const double* x, long long n, long long row0) {
  if (n <= 0) return;
  const int D = m->dims[0];
  for (long long r = 0; r < n;) {
    const long long c = std::min(n - r, m->cap * m->stage_w / std::max(D, 1));
    MOSES_CUDA(cudaMemcpyAsync(m->staging, x + r * D, sizeof(double) * c * D, cudaMemcpyHostToDevice, m->st));
    if (m->esz == 2)
      pack_rows<__nv_bfloat16>(m->staging, c, D, static_cast<__nv_bfloat16*>(m->act[0]) + (row0 + r) * m->ld[0],
                               m->ld[0], m->st,
                               m->split ? m->act_lo_t<__nv_bfloat16>(0) + (row0 + r) * m->ld[0] : nullptr);
    else
      pack_rows<float>(m->staging, c, D, static_cast<float*>(m->act[0]) + (row0 + r) * m->ld[0], m->ld[0], m->st,
                       m->split ? m->act_lo_t<float>(0) + (row0 + r) * m->ld[0] : nullptr);
    note_launch(1);
    r += c;
  }
}
void upload_replay(moses_model* m, const moses_adversary* a) {
  if (m->esz == 2)
    pack_rows_f32<__nv_bfloat16>(a->replay, a->m, a->D, a->D, static_cast<__nv_bfloat16*>(m->act[0]), m->ld[0], m->st,
                                 m->act_lo_t<__nv_bfloat16>(0));
  else
    pack_rows_f32<float>(a->replay, a->m, a->D, a->D, static_cast<float*>(m->act[0]), m->ld[0], m->st,
                         m->act_lo_t<float>(0));
  note_launch(1);
}
void upload_f32(moses_model* m, const double* src, long long n, float* dst) {
  if (n <= 0) return;
  for (long long r = 0; r < n;) {
    const long long c = std::min(n - r, m->cap * m->stage_w);
    MOSES_CUDA(cudaMemcpyAsync(m->staging, src + r, sizeof(double) * c, cudaMemcpyHostToDevice, m->st));
    f64_to_f32(m->staging, c, dst + r, m->st);
    note_launch(1);
    r += c;
  }
}
void download_f32(moses_model* m, const float* src, long long n, double* dst) {
  if (n <= 0) return;
  for (long long r = 0; r < n;) {
    const long long c = std::min(n - r, m->cap * m->stage_w);
    f32_to_f64(src + r, c, m->staging, m->st);
    note_launch(1);
    MOSES_CUDA(cudaMemcpyAsync(dst + r, m->staging, sizeof(double) * c, cudaMemcpyDeviceToHost, m->st));
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    r += c;
  }
}

// Device-resident input rows (x, ldx elements of in_esz() bytes) as the layer-0 operand: split handles
// convert rows [0, n) into the hi/lo planes of act[0]; every other handle reads them in place.
const void* stage_device_rows(moses_model* m, const void* x, long long ldx, long long n, long long* ld_out) {
  if (!m->split) {
    *ld_out = ldx;
    return x;
  }
  const int D = m->dims[0];
  if (ldx < D) fail(MOSES_ERR_INVALID_ARG, "row stride below the input width");
  if (m->esz == 2)
    pack_rows_f32<__nv_bfloat16>(static_cast<const float*>(x), n, D, ldx, static_cast<__nv_bfloat16*>(m->act[0]),
                                 m->ld[0], m->st, m->act_lo_t<__nv_bfloat16>(0));
  else
    pack_rows_f32<float>(static_cast<const float*>(x), n, D, ldx, static_cast<float*>(m->act[0]), m->ld[0], m->st,
                         m->act_lo_t<float>(0));
  note_launch(1);
  *ld_out = m->ld[0];
  return m->act[0];
}

void dispatch_forward(moses_model* m, const void* x0, long long ldx0, long long R, const float* u, bool keep_last) {
  if (m->esz == 2) forward_rows<__nv_bfloat16>(m, x0, ldx0, R, u, keep_last);
  else forward_rows<float>(m, x0, ldx0, R, u, keep_last);
}

// Segment-sum pooling of statement rows into programs (north-star (2); S == 1 is the reference).
struct Pool {
  const long long* seg_off = nullptr;  // device, programs+1 CSR offsets over statement rows
  const int* seg_of_row = nullptr;     // device, program of each statement row (-1 = padding)
  long long rows = 0;                  // statement rows incl. padding
};

// Ranking workspace (per-(split, row) partials of the two-kernel path, per-row sums of the grid
// form): rank_splits(n) * n entries, allocated for min(cap, 4096) rows and grown on the first larger
// batch. A grown-out buffer is retired, not freed: a CUDA graph captured earlier may reference it.
constexpr long long kRankWsInitRows = 4096;
void ensure_rank_ws(moses_model* m, long long n) {
  if (n <= m->rank_ws_rows) return;
  const long long ns = rank_splits(n);
  for (void* p : {(void*)m->rank.gs_part, (void*)m->rank.loss_part, (void*)m->rank.pairs_part})
    if (p) m->retired.push_back(p);
  m->rank.gs_part = dalloc<double>(ns * n);
  m->rank.loss_part = dalloc<double>(ns * n);
  m->rank.pairs_part = dalloc<long long>(ns * n);
  m->rank.nsplit = int(ns);
  m->rank_ws_rows = n;
}

// MMD^2 domain term (north-star (4)): rows [0, rows) of the step are source rows (the replay rows'
// slot), beta * MMD^2(H_src, H_batch) joins the loss and its gradient enters dH of every row.
struct MmdTerm {
  long long rows = 0;
  double beta = 0.0;
  double sigma = 1.0;
};
void ensure_mmd_ws(moses_model* m) {
  if (m->mmd_g) return;
  m->mmd_g = dalloc<float>(size_t(m->cap) * m->W());
  m->mmd_v = dalloc<double>(m->cap);
}

// gradients() core on rows already packed at act[0] (or x0): [0, mrep) replay, [mrep, mrep+n) batch;
// pooled: rows [0, pool->rows) are statements of the n programs.
// Returns true when `fuse` (momentum SGD) was applied inside the backward pass; the caller runs
// the separate update otherwise.
bool gradients_core(moses_model* m, const void* x0, long long ldx0, const float* y, long long n, moses_adversary* adv,
                    double beta, const Pool* pool = nullptr, const SgdFuse* fuse = nullptr,
                    const MmdTerm* mmd = nullptr) {
  const bool active = adv != nullptr && beta != 0.0 && n > 0 && pool == nullptr;
  const bool mmd_on = mmd != nullptr && mmd->beta != 0.0 && n > 0 && pool == nullptr && !active;
  const long long mrep = active ? adv->m : (mmd_on ? mmd->rows : 0);
  const long long R = pool ? pool->rows : mrep + n;
  ensure_rank_ws(m, n);  // before any capture-sensitive work (warm-ups reach here with the captured n)
  if (n == 0 || R == 0) {
    MOSES_CUDA(cudaMemsetAsync(m->g, 0, sizeof(float) * m->P, m->st));
    MOSES_CUDA(cudaMemsetAsync(m->dscal, 0, sizeof(double) * 2, m->st));
    m->xi_valid = false;
    return false;
  }
  const float* u = active ? adv->u : nullptr;
  dispatch_forward(m, x0, ldx0, R, u, true);
  if (!active && !mmd_on && g_rank_fused) {
    if (!m->rank_ticket) {
      m->rank_ticket = dalloc<unsigned int>(4);  // [grid-form ticket, symmetric form: count, generation, ticket]
      MOSES_CUDA(cudaMemsetAsync(m->rank_ticket, 0, 4 * sizeof(unsigned int), m->st));
    }
  }
  bool ranked = false;
  if (!active && !mmd_on && g_rank_fused && m->rank_ticket) {
    ProfScope ps(P_RANK, m->st);
    FinalizeOut fo{m->dscal, m->dpairs, m->coefA, m->coefB, m->dscal + 1};
    if (pool) fo.gb = m->gbias;
    ranked = rank_step(m->head_part, m->last_tiles, m->cap, m->head_b(), pool ? pool->seg_off : nullptr, y, n,
                       {m->rank.gs_part, m->rank.loss_part, m->rank.pairs_part, rank_splits(n)}, m->rank_ticket,
                       m->scores, pool ? pool->seg_of_row : nullptr, R, fo, m->st);
    if (ranked) note_launch(1);
  }
  if (!ranked) {
    ProfScope ps(P_RANK, m->st);
    rank_pairs_fused(m->head_part + mrep, m->last_tiles, m->cap, m->head_b(), pool ? pool->seg_off : nullptr, y, n,
                     {m->rank.gs_part, m->rank.loss_part, m->rank.pairs_part, rank_splits(n)}, m->scores, m->st);
    FinalizeOut fo{m->dscal, m->dpairs, m->coefA, m->coefB, m->dscal + 1};
    if (pool) {
      fo.seg_of_row = pool->seg_of_row;
      fo.R_rows = R;
      fo.gb = m->gbias;
    }
    rank_finalize({m->rank.gs_part, m->rank.loss_part, m->rank.pairs_part, rank_splits(n)}, n, mrep,
                  active ? m->head_part2 : nullptr, m->last_tiles, m->cap, active ? adv->c : nullptr, beta, fo, m->st);
    note_launch(2);
  }
  const float* gbo = pool ? m->gbias : nullptr;
  const float* extra = nullptr;
  if (mmd_on) {  // beta * MMD^2 between the source rows' and the batch rows' last hidden layer
    ensure_mmd_ws(m);
    const int W = m->W();
    ProfScope ps(P_OTHER, m->st);
    if (m->esz == 2)
      mmd_grad<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(m->act[m->L - 1]), m->act_lo_t<__nv_bfloat16>(m->L - 1),
                              m->ld[m->L - 1], R, mrep, W, float(mmd->sigma), m->mmd_g, m->mmd_v, m->dscal,
                              mmd->beta, true, m->st);
    else
      mmd_grad<float>(static_cast<const float*>(m->act[m->L - 1]), m->act_lo_t<float>(m->L - 1), m->ld[m->L - 1], R,
                      mrep, W, float(mmd->sigma), m->mmd_g, m->mmd_v, m->dscal, mmd->beta, true, m->st);
    note_launch(2);
    extra = m->mmd_g;
  }
  const float escale = mmd_on ? float(mmd->beta) : 0.f;
  const bool fused = m->esz == 2 ? backward_rows<__nv_bfloat16>(m, x0, ldx0, R, u, gbo, fuse, extra, escale)
                                 : backward_rows<float>(m, x0, ldx0, R, u, gbo, fuse, extra, escale);
  m->xi_valid = false;
  return fused;
}

void check_rows(moses_model* m, long long R) {
  if (R > m->cap)
    fail(MOSES_ERR_CAPACITY, "rows " + std::to_string(R) + " exceed the handle capacity " + std::to_string(m->cap));
}

// momentum SGD over every parameter (tuner.cpp:146-147) with the handle's operand shadow kept current
// (split bf16: the hi/lo pair written by the update kernel itself)
void update_momentum(moses_model* m, float lr, float mu, cudaStream_t st) {
  if (m->bsplit()) {
    sgd_update(m->w, m->mom, m->g, nullptr, m->P, lr, mu, true, m->shadow_full(), st);
  } else {
    sgd_update(m->w, m->mom, m->g, nullptr, m->P, lr, mu, true, m->shadow(), st);
    m->post_update();
  }
  note_launch(1);
}

// ---- data-parallel exact batch: the global batch of n_global = nranks * n
// rows is the rank-ordered concatenation of every rank's n local rows. Phase 1: local forward, local
// scores and labels into their slots of the global arrays. (All-gather.) Phase 2: pair terms of the
// local rows against the whole batch (model.cpp:71-106; each distinct-label pair counted once, at its
// hi row), (loss sum, pair count) partials. (All-reduce.) Phase 3: coefficients normalised by the
// global pair count, local backward -> this rank's share of the gradient. (All-reduce: the sum is the
// gradient of the global batch, up to summation order.) Unpooled rows.
void dp_reserve(moses_model* m, long long n_global) {
  if (n_global <= m->dp_cap) return;
  for (void* p : {(void*)m->dp_s, (void*)m->dp_y})
    if (p) m->retired.push_back(p);  // captured graphs may still point at them
  m->dp_s = dalloc<float>(n_global);
  m->dp_y = dalloc<float>(n_global);
  if (!m->dp_tot) m->dp_tot = dalloc<double>(2);
  m->dp_cap = n_global;
}
void dp_exact_forward(moses_model* m, const void* x0, long long ld0, const float* y, long long n, float* s_slot,
                      float* y_slot) {
  check_rows(m, n);
  dispatch_forward(m, x0, ld0, n, nullptr, true);
  head_scores(m->head_part, m->last_tiles, m->cap, m->head_b(), n, s_slot, m->st);
  note_launch(1);
  if (n > 0 && y_slot != y) MOSES_CUDA(cudaMemcpyAsync(y_slot, y, sizeof(float) * n, cudaMemcpyDeviceToDevice, m->st));
  m->dp_x0 = x0;
  m->dp_ld0 = ld0;
  m->dp_n = n;
}
void dp_exact_rank(moses_model* m, const float* s_global, const float* y_global, long long n_global, long long p0,
                   double* totals_out) {
  const long long n = m->dp_n;
  if (p0 < 0 || p0 + n > n_global) fail(MOSES_ERR_SHAPE_MISMATCH, "local rows outside the global batch");
  const long long need = rank_splits(n_global) * std::max<long long>(n, 1);
  if (need > rank_splits(m->rank_ws_rows) * m->rank_ws_rows) ensure_rank_ws(m, n_global);
  const RankWs ws{m->rank.gs_part, m->rank.loss_part, m->rank.pairs_part, rank_splits(n_global)};
  ProfScope ps(P_RANK, m->st);
  rank_pairs_rows(s_global, y_global, n_global, p0, n, ws, m->st);
  rank_local_totals(ws, n, totals_out, m->st);
  note_launch(2);
}
void dp_exact_backward(moses_model* m, long long n_global, const double* totals_global) {
  const long long n = m->dp_n;
  const RankWs ws{m->rank.gs_part, m->rank.loss_part, m->rank.pairs_part, rank_splits(n_global)};
  {
    ProfScope ps(P_RANK, m->st);
    const FinalizeOut fo{m->dscal, m->dpairs, m->coefA, m->coefB, m->dscal + 1};
    rank_finalize(ws, n, 0, nullptr, 0, 0, nullptr, 0.0, fo, m->st, totals_global);
    note_launch(1);
  }
  if (m->esz == 2) backward_rows<__nv_bfloat16>(m, m->dp_x0, m->dp_ld0, n, nullptr);
  else backward_rows<float>(m, m->dp_x0, m->dp_ld0, n, nullptr);
  m->xi_valid = false;
}
// one exact-batch step on the handle's communicator (graph-capturable): forward -> all-gather ->
// pair terms -> all-reduce of (loss, pairs) -> backward -> all-reduce of the gradients [-> update]
void dp_exact_step(moses_model* m, const void* x0, long long ld0, const float* y, long long n, bool update, float lr,
                   float mu) {
  moses_comm* c = m->comm;
  const long long ng = n * c->nranks, p0 = n * c->rank;
  dp_reserve(m, ng);
  dp_exact_forward(m, x0, ld0, y, n, m->dp_s + p0, m->dp_y + p0);
  comm_allgather_f32(c, m->dp_s + p0, m->dp_s, n, m->st);
  comm_allgather_f32(c, m->dp_y + p0, m->dp_y, n, m->st);
  dp_exact_rank(m, m->dp_s, m->dp_y, ng, p0, m->dp_tot);
  comm_allreduce_f64(c, m->dp_tot, 2, m->st);
  dp_exact_backward(m, ng, m->dp_tot);
  comm_allreduce_f32(c, m->g, m->P, false, m->st);
  if (update) update_momentum(m, lr, mu, m->st);
}

}  // namespace
}  // namespace moses

// ====================================================================== C ABI
extern "C" {

MOSES_API const char* moses_last_error(void) { return g_err.c_str(); }
MOSES_API const char* moses_version(void) { return "moses-b200 0.1 (sm_100a, tcgen05/TMA)"; }
MOSES_API int64_t moses_kernel_launches(void) { return g_launches.load(); }

MOSES_API int moses_device_check(void) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) fail(MOSES_ERR_NO_DEVICE, "no CUDA device");
    cudaDeviceProp p;
    MOSES_CUDA(cudaGetDeviceProperties(&p, 0));
    if (p.major != 10) fail(MOSES_ERR_NO_DEVICE, std::string("need sm_100 (B200), found ") + p.name);
  });
}

MOSES_API int64_t moses_param_count(const int32_t* dims, int32_t nd) {
  int64_t out = 0;
  const int rc = guarded([&] {
    check_dims(dims, nd, false);
    std::vector<int> d(dims, dims + nd);
    out = level_off(d, nd - 1);
  });
  return rc ? -rc : out;
}

MOSES_API int moses_init_random(const int32_t* dims, int32_t nd, uint64_t seed, int32_t strict, double* flat) {
  return guarded([&] {
    check_dims(dims, nd, strict != 0);
    std::vector<int> d(dims, dims + nd);
    const long long P = level_off(d, nd - 1);
    std::fill(flat, flat + P, 0.0);
    for (int l = 0; l + 1 < nd; ++l) {
      const int fi = d[l], fo = d[l + 1];
      const double bound = std::sqrt(6.0 / double(fi + fo));
      KeyBuilder k;
      k.add(seed).add("init").add(uint64_t(l));
      Rng r{k.h};
      double* w = flat + level_off(d, l);
      for (long long i = 0; i < (long long)fi * fo; ++i) w[i] = (2.0 * r.u01() - 1.0) * bound;
    }
  });
}

MOSES_API int moses_model_create(const int32_t* dims, int32_t nd, int32_t precision, int64_t max_rows,
                                 moses_model_t* out) {
  return guarded([&] {
    *out = nullptr;
    check_dims(dims, nd, false);
    if (precision != MOSES_PREC_BF16 && precision != MOSES_PREC_TF32 && precision != MOSES_PREC_FP32 &&
        precision != MOSES_PREC_BF16X3)
      fail(MOSES_ERR_INVALID_ARG, "precision");
    if (precision == MOSES_PREC_BF16X3) {  // the split-bf16 kernels are the fused 512-wide chains
      bool ok = dims[0] <= 512 && nd - 2 <= 8;
      for (int l = 1; l + 1 < nd; ++l) ok = ok && dims[l] == 512;
      if (!ok) fail(MOSES_ERR_INVALID_ARG, "split-bf16 (BF16X3) handles need hidden widths of 512, input width <= 512 "
                                           "and at most 8 hidden layers; use TF32 or FP32 for other shapes");
    }
    for (int l = 1; l + 1 < nd; ++l)
      if (dims[l] % 8) fail(MOSES_ERR_INVALID_ARG, "hidden widths must be multiples of 8 (TMA 16-byte rows)");
    if (max_rows < 1) max_rows = 1;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(MOSES_ERR_NO_DEVICE, "no CUDA device visible");
    auto m = std::make_unique<moses_model>();
    m->dims.assign(dims, dims + nd);
    m->L = nd - 1;
    m->P = level_off(m->dims, m->L);
    for (int l = 0; l <= m->L; ++l) m->off.push_back(level_off(m->dims, l));
    m->prec = precision;
    MOSES_CUDA(cudaGetDevice(&m->device));
    m->esz = (precision == MOSES_PREC_BF16 || precision == MOSES_PREC_BF16X3) ? 2 : 4;
    m->split = precision == MOSES_PREC_FP32 || precision == MOSES_PREC_BF16X3;
    const int twin = m->split ? 2 : 1;  // split modes: [hi | lo] halves of every GEMM operand buffer
    m->cap = round_up(max_rows, 128);
    keep_async_pool();  // per-call stream-ordered workspaces (encode, MMD, tune loop) stay mapped
    MOSES_CUDA(cudaStreamCreateWithFlags(&m->st, cudaStreamNonBlocking));
    MOSES_CUDA(cudaStreamCreateWithFlags(&m->st2, cudaStreamNonBlocking));
    m->evs.resize(m->L + 4);
    for (auto& e : m->evs) MOSES_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const long long P = m->P;
    m->w = dalloc<float>(P);
    m->mom = dalloc<float>(P);
    m->g = dalloc<float>(P);
    m->xi = dalloc<float>(P);
    m->mask = dalloc<uint8_t>(P);
    const long long shadow_n = twin == 2 ? 2 * shadow_lo_offset(P) : P;  // split: [hi | lo] at shadow_lo_offset
    if (m->esz == 2) m->wbf = dalloc<__nv_bfloat16>(shadow_n);
    else m->wtf = dalloc<float>(shadow_n);
    // Every initialisation goes through the handle's (non-blocking) stream: a plain cudaMemset runs on
    // the legacy stream, which does NOT order against m->st, and could land after the first upload or
    // after the ones-column fill below (an intermittent wrong bias gradient, seen in bitwise tests).
    MOSES_CUDA(cudaMemsetAsync(m->w, 0, P * 4, m->st));
    MOSES_CUDA(cudaMemsetAsync(m->mom, 0, P * 4, m->st));
    MOSES_CUDA(cudaMemsetAsync(m->g, 0, P * 4, m->st));
    if (m->wbf) MOSES_CUDA(cudaMemsetAsync(m->wbf, 0, shadow_n * 2, m->st));
    if (m->wtf) MOSES_CUDA(cudaMemsetAsync(m->wtf, 0, shadow_n * 4, m->st));
    const int vec = 16 / m->esz;
    int maxw = 0;
    for (int l = 0; l < m->L; ++l) {
      const long long ldl = round_up(m->dims[l] + 1, vec);
      m->ld.push_back(ldl);
      m->lddz.push_back(round_up(m->dims[l], vec));
      maxw = std::max(maxw, m->dims[l]);
      void* a = nullptr;
      MOSES_CUDA(cudaMalloc(&a, m->cap * ldl * m->esz * twin));
      MOSES_CUDA(cudaMemsetAsync(a, 0, m->cap * ldl * m->esz * twin, m->st));
      m->act.push_back(a);
      void* d = nullptr;
      if (l > 0) {
        MOSES_CUDA(cudaMalloc(&d, m->cap * m->lddz[l] * m->esz * twin));
        MOSES_CUDA(cudaMemsetAsync(d, 0, m->cap * m->lddz[l] * m->esz * twin, m->st));
      }
      m->dz.push_back(d);
      // ones column of every activation buffer (never overwritten by the epilogues)
      if (m->esz == 2) set_ones_column<__nv_bfloat16>(static_cast<__nv_bfloat16*>(a), m->cap, m->dims[l], ldl, m->st);
      else set_ones_column<float>(static_cast<float*>(a), m->cap, m->dims[l], ldl, m->st);
      note_launch(1);
    }
    m->max_tiles = ceil_div(m->dims[m->L - 1], 64);
    m->head_part = dalloc<float>(m->max_tiles * m->cap);
    m->head_part2 = dalloc<float>(m->max_tiles * m->cap);
    m->scores = dalloc<float>(m->cap);
    m->labels = dalloc<float>(m->cap);
    m->coefA = dalloc<float>(m->cap);
    m->coefB = dalloc<float>(m->cap);
    ensure_rank_ws(m.get(), std::min<long long>(m->cap, kRankWsInitRows));
    m->dscal = dalloc<double>(16);
    m->dpairs = dalloc<long long>(4);
    m->dcount = dalloc<unsigned long long>(4);
    const long long seln = std::max<long long>(P, m->cap);
    const size_t selb = select_ws_bytes(seln, nullptr);
    MOSES_CUDA(cudaMalloc(&m->sel_base, selb));
    select_ws_carve(m->sel_base, seln, &m->sel);
    m->stage_w = std::max<long long>(maxw, 1) + 1;
    m->staging = dalloc<double>(m->cap * m->stage_w);
    m->gbias = dalloc<float>(4);
    if (m->bsplit()) m->wgsk_ws = dalloc<float>(wgrad_sk_ws_bytes() / sizeof(float));
    m->seg_off = dalloc<long long>(m->cap + 1);
    m->seg_rows = dalloc<int>(m->cap);
    m->adv_ws = dalloc<float>(round_up(m->cap, 64) + round_up(maxw + 1, 64) + 64 + 16 +
                              column_dot_ws_floats(m->cap, maxw) + 64);
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    *out = m.release();
  });
}

MOSES_API int moses_model_destroy(moses_model_t m) {
  return guarded([&] { delete m; });
}

MOSES_API int moses_model_upload(moses_model_t m, const double* params, const double* momentum, int64_t count) {
  return guarded([&] {
    require_model(m);
    if (count != m->P) fail(MOSES_ERR_SHAPE_MISMATCH, "parameter count mismatch");
    upload_f32(m, params, count, m->w);
    if (momentum) upload_f32(m, momentum, count, m->mom);
    else MOSES_CUDA(cudaMemsetAsync(m->mom, 0, count * 4, m->st));
    refresh_shadow(m->w, count, m->shadow_full(), m->st);
    note_launch(1);
    m->xi_valid = false;
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

MOSES_API int moses_model_download(moses_model_t m, double* params, double* momentum, int64_t count) {
  return guarded([&] {
    require_model(m);
    if (count != m->P) fail(MOSES_ERR_SHAPE_MISMATCH, "parameter count mismatch");
    if (params) download_f32(m, m->w, count, params);
    if (momentum) download_f32(m, m->mom, count, momentum);
  });
}

MOSES_API int moses_model_copy(moses_model_t dst, moses_model_t src) {
  return guarded([&] {
    require_model(dst);
    require_model(src);
    if (dst->dims != src->dims) fail(MOSES_ERR_SHAPE_MISMATCH, "model dims differ");
    MOSES_CUDA(cudaStreamSynchronize(src->st));
    MOSES_CUDA(cudaMemcpyAsync(dst->w, src->w, src->P * 4, cudaMemcpyDeviceToDevice, dst->st));
    MOSES_CUDA(cudaMemcpyAsync(dst->mom, src->mom, src->P * 4, cudaMemcpyDeviceToDevice, dst->st));
    refresh_shadow(dst->w, dst->P, dst->shadow_full(), dst->st);
    note_launch(1);
    MOSES_CUDA(cudaStreamSynchronize(dst->st));
  });
}

MOSES_API int moses_model_synchronize(moses_model_t m) {
  return guarded([&] {
    require_model(m);
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    for (auto& a : m->aslot)  // asynchronous steps: deliver the losses of the completed steps
      if (a.pending) {
        *a.pending = *a.box_host;
        a.pending = nullptr;
      }
  });
}

MOSES_API int64_t moses_packed_ld(moses_model_t m) { return m ? m->ld[0] : -MOSES_ERR_INVALID_ARG; }

static void predict_impl(moses_model* m, const double* x, long long n, int D, double* out, bool penult) {
  require_model(m);
  if (D != m->dims[0])
    fail(MOSES_ERR_DIM_MISMATCH, "feature width " + std::to_string(D) + " != model input width " +
                                     std::to_string(m->dims[0]));
  const int W = m->W();
  for (long long r = 0; r < n;) {
    const long long c = std::min(n - r, m->cap);
    upload_rows(m, x + r * D, c, 0);
    dispatch_forward(m, m->act[0], m->ld[0], c, nullptr, penult);
    if (penult) {
      if (m->esz == 2)
        unpack_rows<__nv_bfloat16>(static_cast<__nv_bfloat16*>(m->act[m->L - 1]), c, W, m->ld[m->L - 1], m->staging,
                                   m->st, m->act_lo_t<__nv_bfloat16>(m->L - 1));
      else
        unpack_rows<float>(static_cast<float*>(m->act[m->L - 1]), c, W, m->ld[m->L - 1], m->staging, m->st,
                           m->act_lo_t<float>(m->L - 1));
      note_launch(1);
      for (long long q = 0; q < c;) {  // staging holds cap*stage_w doubles >= c*W
        const long long cc = c - q;
        MOSES_CUDA(cudaMemcpyAsync(out + (r + q) * W, m->staging + q * W, sizeof(double) * cc * W,
                                   cudaMemcpyDeviceToHost, m->st));
        q += cc;
      }
      MOSES_CUDA(cudaStreamSynchronize(m->st));
    } else {
      head_scores(m->head_part, m->last_tiles, m->cap, m->head_b(), c, m->scores, m->st);
      note_launch(1);
      download_f32(m, m->scores, c, out + r);
    }
    r += c;
  }
}

MOSES_API int moses_predict(moses_model_t m, const double* x, int64_t n, int32_t D, double* scores) {
  return guarded([&] { predict_impl(m, x, n, D, scores, false); });
}
MOSES_API int moses_penultimate(moses_model_t m, const double* x, int64_t n, int32_t D, double* h) {
  return guarded([&] { predict_impl(m, x, n, D, h, true); });
}

MOSES_API int moses_predict_device(moses_model_t m, const void* x_dev, int32_t dtype, int64_t ldx, int64_t n,
                                   float* scores_dev) {
  return guarded([&] {
    require_model(m);
    if ((dtype == MOSES_DTYPE_BF16) != (m->in_esz() == 2))
      fail(MOSES_ERR_INVALID_ARG, "dtype must match the handle's input type (bf16 for bf16 handles, else fp32)");
    for (long long r = 0; r < n;) {
      const long long c = std::min(n - r, m->cap);
      long long ld0 = 0;
      const void* x0 = stage_device_rows(m, static_cast<const uint8_t*>(x_dev) + r * ldx * m->in_esz(), ldx, c, &ld0);
      dispatch_forward(m, x0, ld0, c, nullptr, false);
      head_scores(m->head_part, m->last_tiles, m->cap, m->head_b(), c, scores_dev + r, m->st);
      note_launch(1);
      r += c;
    }
  });
}

MOSES_API int moses_predict_pooled(moses_model_t m, const double* x, int64_t n, int32_t D, const int64_t* offsets,
                                   int64_t programs, double* scores) {
  return guarded([&] {
    require_model(m);
    if (D != m->dims[0]) fail(MOSES_ERR_DIM_MISMATCH, "feature width != model input width");
    if (offsets[0] != 0 || offsets[programs] != n) fail(MOSES_ERR_SHAPE_MISMATCH, "offsets must span the rows");
    for (int64_t p = 0; p < programs; ++p)
      if (offsets[p + 1] < offsets[p]) fail(MOSES_ERR_SHAPE_MISMATCH, "offsets must be non-decreasing");
    // per-statement head dots (bias excluded), then segment sum + bias on the device
    float* stmt = nullptr;
    long long* doff = nullptr;
    float* pout = nullptr;
    stmt = dalloc<float>(n);
    doff = dalloc<long long>(programs + 1);
    pout = dalloc<float>(programs);
    float zero_b = 0.f;
    float* dzero = dalloc<float>(1);
    MOSES_CUDA(cudaMemcpyAsync(dzero, &zero_b, 4, cudaMemcpyHostToDevice, m->st));
    MOSES_CUDA(cudaMemcpyAsync(doff, offsets, sizeof(long long) * (programs + 1), cudaMemcpyHostToDevice, m->st));
    for (long long r = 0; r < n;) {
      const long long c = std::min(n - r, m->cap);
      upload_rows(m, x + r * D, c, 0);
      dispatch_forward(m, m->act[0], m->ld[0], c, nullptr, false);
      head_scores(m->head_part, m->last_tiles, m->cap, dzero, c, stmt + r, m->st);
      note_launch(1);
      r += c;
    }
    float hb = 0.f;
    MOSES_CUDA(cudaMemcpyAsync(&hb, m->head_b(), 4, cudaMemcpyDeviceToHost, m->st));
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    segment_sum_scalar(stmt, doff, programs, hb, pout, m->st);
    note_launch(1);
    download_f32(m, pout, programs, scores);
    dfree(stmt);
    dfree(doff);
    dfree(pout);
    dfree(dzero);
  });
}

static void gradients_host(moses_model* m, const double* x, const double* y, long long n, int D, moses_adversary* adv,
                           double beta) {
  require_model(m);
  if (D != m->dims[0])
    fail(MOSES_ERR_DIM_MISMATCH, "batch feature width " + std::to_string(D) + " != model input width " +
                                     std::to_string(m->dims[0]));
  const bool active = adv != nullptr && beta != 0.0 && n > 0;
  if (active) {  // model.cpp:130-137
    if (adv->W != m->W()) fail(MOSES_ERR_DIM_MISMATCH, "discriminator width != penultimate width");
    if (adv->m == 0) fail(MOSES_ERR_ADVERSARY_DISABLED, "adversary has an empty replay buffer");
    if (adv->D != m->dims[0]) fail(MOSES_ERR_DIM_MISMATCH, "replay feature width != model input width");
  }
  const long long mrep = active ? adv->m : 0;
  check_rows(m, mrep + n);
  if (active) upload_replay(m, adv);
  upload_rows(m, x, n, mrep);
  upload_f32(m, y, n, m->labels);
  gradients_core(m, m->act[0], m->ld[0], m->labels, n, active ? adv : nullptr, beta);
}

MOSES_API int moses_gradients(moses_model_t m, const double* x, const double* y, int64_t n, int32_t D,
                              moses_adversary_t adv, double beta, double* loss_out) {
  return guarded([&] {
    gradients_host(m, x, y, n, D, adv, beta);
    if (loss_out) {
      MOSES_CUDA(cudaMemcpyAsync(loss_out, m->dscal, sizeof(double), cudaMemcpyDeviceToHost, m->st));
      MOSES_CUDA(cudaStreamSynchronize(m->st));
    }
  });
}

MOSES_API int moses_objective(moses_model_t m, const double* x, const double* y, int64_t n, int32_t D,
                              moses_adversary_t adv, double beta, double* out) {
  // objective = the loss gradients() reports (model.cpp:246-261 vs :237); the gradient buffer is
  // preserved so the call stays read-only on the handle's visible state.
  return guarded([&] {
    require_model(m);
    float* gsave = dalloc<float>(m->P);
    MOSES_CUDA(cudaMemcpyAsync(gsave, m->g, m->P * 4, cudaMemcpyDeviceToDevice, m->st));
    gradients_host(m, x, y, n, D, adv, beta);
    MOSES_CUDA(cudaMemcpyAsync(out, m->dscal, sizeof(double), cudaMemcpyDeviceToHost, m->st));
    MOSES_CUDA(cudaMemcpyAsync(m->g, gsave, m->P * 4, cudaMemcpyDeviceToDevice, m->st));
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    dfree(gsave);
  });
}

MOSES_API int moses_gradients_device(moses_model_t m, const void* x_dev, int64_t ldx, const float* y_dev, int64_t n,
                                     double* loss_out) {
  return guarded([&] {
    require_model(m);
    check_rows(m, n);
    long long ld0 = 0;
    const void* x0 = stage_device_rows(m, x_dev, ldx, n, &ld0);
    gradients_core(m, x0, ld0, y_dev, n, nullptr, 0.0);
    if (loss_out) {
      MOSES_CUDA(cudaMemcpyAsync(loss_out, m->dscal, sizeof(double), cudaMemcpyDeviceToHost, m->st));
      MOSES_CUDA(cudaStreamSynchronize(m->st));
    }
  });
}

MOSES_API int moses_set_async(int32_t on) {
  g_async = on != 0;
  return MOSES_OK;
}

MOSES_API int moses_profile_begin(void) {
  return guarded([&] {
    Profiler& p = prof();
    std::lock_guard<std::mutex> lk(p.mu);
    for (auto& r : p.rec) p.pool.push_back(r.second);
    p.rec.clear();
    p.on = true;
  });
}

MOSES_API int moses_profile_end(double* ms_by_cat, int64_t* count_by_cat, int32_t ncat) {
  return guarded([&] {
    Profiler& p = prof();
    std::lock_guard<std::mutex> lk(p.mu);
    p.on = false;
    for (int c = 0; c < ncat; ++c) {
      ms_by_cat[c] = 0.0;
      count_by_cat[c] = 0;
    }
    for (auto& r : p.rec) {
      MOSES_CUDA(cudaEventSynchronize(r.second.second));
      float ms = 0.f;
      MOSES_CUDA(cudaEventElapsedTime(&ms, r.second.first, r.second.second));
      if (r.first < ncat) {
        ms_by_cat[r.first] += ms;
        count_by_cat[r.first] += 1;
      }
    }
  });
}

MOSES_API int moses_gradients_download(moses_model_t m, double* g, int64_t count) {
  return guarded([&] {
    require_model(m);
    if (count != m->P) fail(MOSES_ERR_SHAPE_MISMATCH, "gradient count mismatch");
    download_f32(m, m->g, count, g);
  });
}
MOSES_API int moses_gradients_upload(moses_model_t m, const double* g, int64_t count) {
  return guarded([&] {
    require_model(m);
    if (count != m->P) fail(MOSES_ERR_SHAPE_MISMATCH, "gradient count mismatch");
    upload_f32(m, g, count, m->g);
    m->xi_valid = false;
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

static const uint8_t* upload_mask(moses_model* m, const uint8_t* mask, int64_t len) {
  if (!mask) return nullptr;
  if (len != m->P) fail(MOSES_ERR_SHAPE_MISMATCH, "mask length != parameter count");
  MOSES_CUDA(cudaMemcpyAsync(m->mask, mask, m->P, cudaMemcpyHostToDevice, m->st));
  m->mask_valid = true;
  return m->mask;
}

MOSES_API int moses_apply_update(moses_model_t m, double lr, double mu, const uint8_t* mask, int64_t mask_len,
                                 int32_t use_momentum) {
  return guarded([&] {
    require_model(m);
    const uint8_t* dm = upload_mask(m, mask, mask_len);
    {
      ProfScope ps(P_UPDATE, m->st);
      sgd_update(m->w, m->mom, m->g, dm, m->P, float(lr), float(mu), use_momentum != 0, m->shadow(), m->st);
      m->post_update();
    }
    note_launch(1);
    m->xi_valid = false;
    if (sync_updates()) MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

MOSES_API int moses_adam_update(moses_model_t m, double lr, double b1, double b2, double eps, int32_t step,
                                const uint8_t* mask, int64_t mask_len) {
  return guarded([&] {
    require_model(m);
    if (step < 1) fail(MOSES_ERR_INVALID_ARG, "adam step must be >= 1");
    if (!m->m1) {
      m->m1 = dalloc<float>(m->P);
      m->m2 = dalloc<float>(m->P);
      MOSES_CUDA(cudaMemsetAsync(m->m1, 0, m->P * 4, m->st));
      MOSES_CUDA(cudaMemsetAsync(m->m2, 0, m->P * 4, m->st));
    }
    const uint8_t* dm = upload_mask(m, mask, mask_len);
    const float c1 = float(1.0 - std::pow(b1, step)), c2 = float(1.0 - std::pow(b2, step));
    adam_update(m->w, m->m1, m->m2, m->g, dm, m->P, float(lr), float(b1), float(b2), float(eps), c1, c2, m->shadow(),
                m->st);
    m->post_update();
    note_launch(1);
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

MOSES_API int moses_train_step(moses_model_t m, const double* x, const double* y, int64_t n, int32_t D, double lr,
                               double mu, double* loss_out) {
  return guarded([&] {
    gradients_host(m, x, y, n, D, nullptr, 0.0);
    sgd_update(m->w, m->mom, m->g, nullptr, m->P, float(lr), float(mu), true, m->shadow(), m->st);
    m->post_update();
    note_launch(1);
    if (loss_out) {
      MOSES_CUDA(cudaMemcpyAsync(loss_out, m->dscal, sizeof(double), cudaMemcpyDeviceToHost, m->st));
      MOSES_CUDA(cudaStreamSynchronize(m->st));
    }
  });
}

// ---- CUDA graph of one device-resident training step: gather batch (device counter) ->
// gradients -> momentum update -> advance counter. Replayed with one cudaGraphLaunch per step.
static long long g_graph_kernels = 0;
MOSES_API int moses_train_graph_create(moses_model_t m, const void* x_base, int64_t ldx, const float* y_base,
                                       int64_t n_batches, int64_t batch, double lr, double mu, int32_t with_update) {
  return guarded([&] {
    require_model(m);
    if (m->split && !m->bsplit())
      fail(MOSES_ERR_INVALID_ARG, "training graphs are not available for FP32 (3xTF32) handles");
    check_rows(m, batch);
    if (ldx != m->ld[0]) fail(MOSES_ERR_INVALID_ARG, "dataset row stride must equal moses_packed_ld");
    if (n_batches < 1) fail(MOSES_ERR_INVALID_ARG, "n_batches must be >= 1");
    for (cudaGraphExec_t* e : {&m->train_exec, &m->train_exec2})
      if (*e) {
        cudaGraphExecDestroy(*e);
        *e = nullptr;
      }
    if (!m->dcounter) m->dcounter = dalloc<long long>(1);
    MOSES_CUDA(cudaMemsetAsync(m->dcounter, 0, sizeof(long long), m->st));
    const long long row_bytes = ldx * m->in_esz();
    auto body = [&] {
      gather_batch(x_base, row_bytes, y_base, m->dcounter, n_batches, batch, m->act[0], m->labels, m->st,
                   m->act_lo(0));
      if (m->comm_mode == 2) {  // data-parallel exact batch: collectives inside the graph
        dp_exact_step(m, m->act[0], m->ld[0], m->labels, batch, with_update != 0, float(lr), float(mu));
        advance_counter(m->dcounter, m->st);
        return;
      }
      const SgdFuse fz{float(lr), float(mu), m->dcounter};
      const bool fused = gradients_core(m, m->act[0], m->ld[0], m->labels, batch, nullptr, 0.0, nullptr,
                                        (with_update && !m->comm) ? &fz : nullptr);
      if (with_update && !fused) {
        if (m->comm) comm_allreduce_f32(m->comm, m->g, m->P, true, m->st);  // throughput-mode DP average
        update_momentum(m, float(lr), float(mu), m->st);
      }
      if (!fz.folded) advance_counter(m->dcounter, m->st);
    };
    {  // eager warm-up without the update (configures kernels, validates shapes; params untouched)
      gather_batch(x_base, row_bytes, y_base, m->dcounter, n_batches, batch, m->act[0], m->labels, m->st,
                   m->act_lo(0));
      if (m->comm_mode == 2) dp_exact_step(m, m->act[0], m->ld[0], m->labels, batch, false, 0.f, 0.f);
      else gradients_core(m, m->act[0], m->ld[0], m->labels, batch, nullptr, 0.0);
    }
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    cudaGraph_t graph;
    MOSES_CUDA(cudaStreamBeginCapture(m->st, cudaStreamCaptureModeThreadLocal));
    try {
      body();
    } catch (...) {
      cudaStreamEndCapture(m->st, &graph);
      throw;
    }
    MOSES_CUDA(cudaStreamEndCapture(m->st, &graph));
    size_t nodes = 0;
    MOSES_CUDA(cudaGraphGetNodes(graph, nullptr, &nodes));
    std::vector<cudaGraphNode_t> nv(nodes);
    MOSES_CUDA(cudaGraphGetNodes(graph, nv.data(), &nodes));
    long long kernels = 0;
    for (auto n : nv) {
      cudaGraphNodeType t;
      MOSES_CUDA(cudaGraphNodeGetType(n, &t));
      kernels += t == cudaGraphNodeTypeKernel;
    }
    g_graph_kernels = kernels;
    MOSES_CUDA(cudaGraphInstantiate(&m->train_exec, graph, 0));
    MOSES_CUDA(cudaGraphDestroy(graph));
  });
}
MOSES_API int moses_train_graph_create_pooled(moses_model_t m, const void* x_base, int64_t ldx, const float* y_base,
                                              const int64_t* prog_off_dev, int64_t n_batches, int64_t batch_programs,
                                              int64_t rows_pad, double lr, double mu, int32_t with_update) {
  return guarded([&] {
    require_model(m);
    if (m->split && !m->bsplit())
      fail(MOSES_ERR_INVALID_ARG, "training graphs are not available for FP32 (3xTF32) handles");
    check_rows(m, rows_pad);
    if (ldx != m->ld[0]) fail(MOSES_ERR_INVALID_ARG, "dataset row stride must equal moses_packed_ld");
    if (n_batches < 1 || batch_programs < 1) fail(MOSES_ERR_INVALID_ARG, "empty batch plan");
    if (m->comm_mode == 2)
      fail(MOSES_ERR_INVALID_ARG, "exact-batch data parallelism takes unpooled rows (moses_train_graph_create)");
    for (cudaGraphExec_t* e : {&m->train_exec, &m->train_exec2})
      if (*e) {
        cudaGraphExecDestroy(*e);
        *e = nullptr;
      }
    if (!m->dcounter) m->dcounter = dalloc<long long>(1);
    if (!m->pcounter) m->pcounter = dalloc<long long>(1);
    if (!m->alt.act) {
      m->alt.act = dalloc<uint8_t>(size_t(m->cap) * m->ld[0] * m->esz * (m->split ? 2 : 1));
      MOSES_CUDA(cudaMemsetAsync(m->alt.act, 0, size_t(m->cap) * m->ld[0] * m->esz * (m->split ? 2 : 1), m->st));
      m->alt.labels = dalloc<float>(m->cap);
      m->alt.seg_off = dalloc<long long>(m->cap + 1);
      m->alt.seg_rows = dalloc<int>(m->cap);
    }
    if (!m->st3) MOSES_CUDA(cudaStreamCreateWithFlags(&m->st3, cudaStreamNonBlocking));
    if (!m->pf_fork) MOSES_CUDA(cudaEventCreateWithFlags(&m->pf_fork, cudaEventDisableTiming));
    if (!m->pf_join) MOSES_CUDA(cudaEventCreateWithFlags(&m->pf_join, cudaEventDisableTiming));
    const long long row_bytes = ldx * m->in_esz();
    const auto* po = reinterpret_cast<const long long*>(prog_off_dev);
    const moses_model::BatchBuf bufA{m->act[0], m->labels, m->seg_off, m->seg_rows};
    const moses_model::BatchBuf bufs[2] = {bufA, m->alt};
    auto gather_into = [&](const moses_model::BatchBuf& b, cudaStream_t st) {
      gather_pooled(x_base, row_bytes, y_base, po, m->pcounter, n_batches, batch_programs, rows_pad, b.act, b.labels,
                    b.seg_off, b.seg_rows, st, const_cast<void*>(m->x0_lo(b.act)));
    };
    // eager warm-up (lazy workspaces, kernel attributes) on both buffers; parameters untouched
    MOSES_CUDA(cudaMemsetAsync(m->pcounter, 0, sizeof(long long), m->st));
    for (const auto& b : bufs) {
      gather_into(b, m->st);
      Pool pool{b.seg_off, b.seg_rows, rows_pad};
      gradients_core(m, b.act, m->ld[0], b.labels, batch_programs, nullptr, 0.0, &pool);
    }
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    auto step_body = [&](int cur) {
      const auto& c = bufs[cur];
      const auto& nx = bufs[cur ^ 1];
      Pool pool{c.seg_off, c.seg_rows, rows_pad};
      MOSES_CUDA(cudaEventRecord(m->pf_fork, m->st));  // side branch: the next batch into the other buffer
      MOSES_CUDA(cudaStreamWaitEvent(m->st3, m->pf_fork, 0));
      gather_into(nx, m->st3);
      advance_counter(m->pcounter, m->st3);
      MOSES_CUDA(cudaEventRecord(m->pf_join, m->st3));
      const SgdFuse fz{float(lr), float(mu)};
      const bool fused = gradients_core(m, c.act, m->ld[0], c.labels, batch_programs, nullptr, 0.0, &pool,
                                        (with_update && !m->comm) ? &fz : nullptr);
      if (with_update && !fused) {
        if (m->comm) comm_allreduce_f32(m->comm, m->g, m->P, true, m->st);  // throughput-mode DP average
        update_momentum(m, float(lr), float(mu), m->st);
      }
      MOSES_CUDA(cudaStreamWaitEvent(m->st, m->pf_join, 0));
    };
    auto capture = [&](std::initializer_list<int> seq, cudaGraphExec_t* out) -> long long {
      cudaGraph_t graph;
      MOSES_CUDA(cudaStreamBeginCapture(m->st, cudaStreamCaptureModeThreadLocal));
      try {
        for (int cur : seq) step_body(cur);
      } catch (...) {
        cudaStreamEndCapture(m->st, &graph);
        throw;
      }
      MOSES_CUDA(cudaStreamEndCapture(m->st, &graph));
      size_t nodes = 0;
      MOSES_CUDA(cudaGraphGetNodes(graph, nullptr, &nodes));
      std::vector<cudaGraphNode_t> nv(nodes);
      MOSES_CUDA(cudaGraphGetNodes(graph, nv.data(), &nodes));
      long long k = 0;
      for (auto n : nv) {
        cudaGraphNodeType t;
        MOSES_CUDA(cudaGraphNodeGetType(n, &t));
        k += t == cudaGraphNodeTypeKernel;
      }
      MOSES_CUDA(cudaGraphInstantiate(out, graph, 0));
      MOSES_CUDA(cudaGraphDestroy(graph));
      return k;
    };
    const long long kernels = capture({0}, &m->train_exec);
    capture({1}, &m->train_exec2);
    g_graph_kernels = kernels + 1;  // + the prefetch's share: one gather per step
    // batch 0 into buffer A; the first launch computes on A and prefetches batch 1 into B
    MOSES_CUDA(cudaMemsetAsync(m->pcounter, 0, sizeof(long long), m->st));
    gather_into(bufA, m->st);
    advance_counter(m->pcounter, m->st);
    note_launch(2);
    m->train_parity = 0;
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

// tuner.cpp:146-147 (gradients + momentum apply_update) on host float64 statement rows, queued
// asynchronously: staging slot k % 2 is uploaded on a copy stream (overlapping the previous step's
// kernels) and consumed by a per-slot CUDA graph (pack -> gradients -> fused update) on the model
// stream; the loss is copied to loss_out when the step completes.
MOSES_API int moses_train_step_pooled_async(moses_model_t m, const double* x, int64_t n_stmt, int32_t D,
                                            const int64_t* offsets, int64_t programs, const double* y, double lr,
                                            double mu, double* loss_out) {
  return guarded([&] {
    require_model(m);
    if (m->esz != 2) fail(MOSES_ERR_INVALID_ARG, "the asynchronous pooled step needs a bf16 or split-bf16 handle");
    if (D != m->dims[0]) fail(MOSES_ERR_DIM_MISMATCH, "statement feature width != model input width");
    if (programs < 1 || offsets[0] != 0 || offsets[programs] != n_stmt)
      fail(MOSES_ERR_SHAPE_MISMATCH, "offsets must span the statement rows");
    for (int64_t p = 0; p < programs; ++p)
      if (offsets[p + 1] < offsets[p]) fail(MOSES_ERR_SHAPE_MISMATCH, "offsets must be non-decreasing");
    check_rows(m, n_stmt);
    if (programs > m->cap) fail(MOSES_ERR_CAPACITY, "more programs than the handle capacity");
    if (!m->st_copy) MOSES_CUDA(cudaStreamCreateWithFlags(&m->st_copy, cudaStreamNonBlocking));
    auto& a = m->aslot[m->async_steps % 3];
    if (!a.x) {
      a.x = dalloc<double>(m->cap * D);
      a.y = dalloc<double>(m->cap);
      a.off = dalloc<long long>(m->cap + 1);
      a.dims = dalloc<long long>(2);
      MOSES_CUDA(cudaMallocHost(&a.dims_host, 2 * sizeof(long long)));
      MOSES_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&a.box_host), sizeof(double), cudaHostAllocMapped));
      MOSES_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&a.box_dev), a.box_host, 0));
      MOSES_CUDA(cudaEventCreateWithFlags(&a.ready, cudaEventDisableTiming));
      MOSES_CUDA(cudaEventCreateWithFlags(&a.free, cudaEventDisableTiming));
      const size_t act_bytes = size_t(m->cap) * size_t(m->ld[0]) * size_t(m->esz) * (m->split ? 2 : 1);
      MOSES_CUDA(cudaMalloc(&a.act, act_bytes));
      MOSES_CUDA(cudaMemsetAsync(a.act, 0, act_bytes, m->st));
      a.labels = dalloc<float>(m->cap);
      a.seg_off = dalloc<long long>(m->cap + 1);
      a.seg_rows = dalloc<int>(m->cap);
      MOSES_CUDA(cudaMemsetAsync(a.labels, 0, sizeof(float) * m->cap, m->st));
      MOSES_CUDA(cudaMemsetAsync(a.seg_off, 0, sizeof(long long) * (m->cap + 1), m->st));
      MOSES_CUDA(cudaMemsetAsync(a.seg_rows, 0xff, sizeof(int) * m->cap, m->st));
    }
    auto* act_s = static_cast<__nv_bfloat16*>(a.act);
    __nv_bfloat16* act_s_lo = m->split ? act_s + m->cap * m->ld[0] : nullptr;
    auto pack_slot = [&](cudaStream_t ps) {
      pack_pooled<__nv_bfloat16>(a.x, a.y, a.off, a.dims, D, m->cap, act_s, m->ld[0], a.labels, a.seg_off, a.seg_rows,
                                 ps, act_s_lo);
    };
    // the per-slot graph: pooled gradients of the slot's packed batch -> fused momentum update (the
    // slot is packed on the copy stream right after its upload, outside the graph)
    if (!a.exec || a.programs != programs || a.lr != float(lr) || a.mu != float(mu)) {
      if (a.exec) {
        MOSES_CUDA(cudaStreamSynchronize(m->st));
        cudaGraphExecDestroy(a.exec);
        a.exec = nullptr;
      }
      Pool pool{a.seg_off, a.seg_rows, m->cap};
      SgdFuse fz{float(lr), float(mu)};
      fz.loss_src = m->dscal;
      fz.loss_copy = a.box_dev;
      // one eager pass first (lazy workspaces must not be allocated while capturing), on an empty
      // batch: `programs` programs with no statements -> no pairs, zero gradients, no update
      MOSES_CUDA(cudaMemsetAsync(a.x, 0, sizeof(double) * m->cap * D, m->st));
      MOSES_CUDA(cudaMemsetAsync(a.y, 0, sizeof(double) * m->cap, m->st));
      MOSES_CUDA(cudaMemsetAsync(a.off, 0, sizeof(long long) * (m->cap + 1), m->st));
      a.dims_host[0] = 0;
      a.dims_host[1] = programs;
      MOSES_CUDA(cudaMemcpyAsync(a.dims, a.dims_host, 2 * sizeof(long long), cudaMemcpyHostToDevice, m->st));
      pack_slot(m->st);
      gradients_core(m, a.act, m->ld[0], a.labels, programs, nullptr, 0.0, &pool, nullptr);
      cudaGraph_t graph;
      MOSES_CUDA(cudaStreamSynchronize(m->st));
      MOSES_CUDA(cudaStreamBeginCapture(m->st, cudaStreamCaptureModeThreadLocal));
      try {
        if (!gradients_core(m, a.act, m->ld[0], a.labels, programs, nullptr, 0.0, &pool, &fz)) {
          sgd_update(m->w, m->mom, m->g, nullptr, m->P, float(lr), float(mu), true, m->shadow(), m->st);
          m->post_update();
        }
        if (!fz.folded) store_scalar_f64(m->dscal, a.box_dev, m->st);
      } catch (...) {
        cudaStreamEndCapture(m->st, &graph);
        throw;
      }
      MOSES_CUDA(cudaStreamEndCapture(m->st, &graph));
      MOSES_CUDA(cudaGraphInstantiate(&a.exec, graph, 0));
      MOSES_CUDA(cudaGraphDestroy(graph));
      a.programs = programs;
      a.lr = float(lr);
      a.mu = float(mu);
    }
    // the slot's previous upload must have left its pinned dims before they are overwritten, and
    // its previous step's loss must reach the caller before the mailbox is reused
    if (a.used) MOSES_CUDA(cudaEventSynchronize(a.ready));
    if (a.used && a.pending) {
      MOSES_CUDA(cudaEventSynchronize(a.free));
      *a.pending = *a.box_host;
      a.pending = nullptr;
    }
    a.dims_host[0] = n_stmt;
    a.dims_host[1] = programs;
    if (a.used) MOSES_CUDA(cudaStreamWaitEvent(m->st_copy, a.free, 0));  // its previous step consumed it
    MOSES_CUDA(cudaMemcpyAsync(a.x, x, sizeof(double) * n_stmt * D, cudaMemcpyHostToDevice, m->st_copy));
    MOSES_CUDA(cudaMemcpyAsync(a.y, y, sizeof(double) * programs, cudaMemcpyHostToDevice, m->st_copy));
    MOSES_CUDA(cudaMemcpyAsync(a.off, offsets, sizeof(long long) * (programs + 1), cudaMemcpyHostToDevice,
                               m->st_copy));
    MOSES_CUDA(cudaMemcpyAsync(a.dims, a.dims_host, 2 * sizeof(long long), cudaMemcpyHostToDevice, m->st_copy));
    pack_slot(m->st_copy);  // overlaps the previous step
    MOSES_CUDA(cudaEventRecord(a.ready, m->st_copy));
    MOSES_CUDA(cudaStreamWaitEvent(m->st, a.ready, 0));
    MOSES_CUDA(cudaGraphLaunch(a.exec, m->st));
    MOSES_CUDA(cudaEventRecord(a.free, m->st));
    a.pending = loss_out;  // copied from the slot's mailbox once its graph has run
    a.used = true;
    ++m->async_steps;
    note_launch(g_graph_kernels > 0 ? g_graph_kernels : 10);
  });
}

MOSES_API int moses_gradients_pooled(moses_model_t m, const double* x, int64_t n_stmt, int32_t D, const int64_t* offsets,
                                     int64_t programs, const double* y, double* loss_out) {
  return guarded([&] {
    require_model(m);
    if (D != m->dims[0]) fail(MOSES_ERR_DIM_MISMATCH, "statement feature width != model input width");
    if (programs < 0 || offsets[0] != 0 || offsets[programs] != n_stmt)
      fail(MOSES_ERR_SHAPE_MISMATCH, "offsets must span the statement rows");
    for (int64_t p = 0; p < programs; ++p)
      if (offsets[p + 1] < offsets[p]) fail(MOSES_ERR_SHAPE_MISMATCH, "offsets must be non-decreasing");
    check_rows(m, n_stmt);
    std::vector<int> rows(static_cast<size_t>(n_stmt));
    for (int64_t p = 0; p < programs; ++p)
      for (int64_t r = offsets[p]; r < offsets[p + 1]; ++r) rows[size_t(r)] = int(p);
    upload_rows(m, x, n_stmt, 0);
    upload_f32(m, y, programs, m->labels);
    MOSES_CUDA(cudaMemcpyAsync(m->seg_off, offsets, sizeof(long long) * (programs + 1), cudaMemcpyHostToDevice, m->st));
    if (n_stmt) MOSES_CUDA(cudaMemcpyAsync(m->seg_rows, rows.data(), sizeof(int) * n_stmt, cudaMemcpyHostToDevice, m->st));
    Pool pool{m->seg_off, m->seg_rows, n_stmt};
    gradients_core(m, m->act[0], m->ld[0], m->labels, programs, nullptr, 0.0, &pool);
    if (loss_out) {
      MOSES_CUDA(cudaMemcpyAsync(loss_out, m->dscal, sizeof(double), cudaMemcpyDeviceToHost, m->st));
    }
    MOSES_CUDA(cudaStreamSynchronize(m->st));  // host vectors above must outlive the async copies
  });
}

MOSES_API int moses_synth_offsets(uint64_t seed, int64_t programs, int32_t max_stmts, int64_t* offsets) {
  // statements per program 1 + below(max_stmts) of stream KeyBuilder(seed,"stmts",p)
  return guarded([&] {
    if (max_stmts < 1) fail(MOSES_ERR_INVALID_ARG, "max_stmts must be >= 1");
    offsets[0] = 0;
    for (int64_t p = 0; p < programs; ++p) {
      KeyBuilder k;
      k.add(seed).add("stmts").add(uint64_t(p));
      Rng r{k.h};
      const uint64_t n = uint64_t(max_stmts), thr = (0 - n) % n;
      uint64_t v;
      do v = r.next(); while (v < thr);
      offsets[p + 1] = offsets[p] + 1 + int64_t(v % n);
    }
  });
}

MOSES_API int moses_train_graph_launch(moses_model_t m, int64_t steps) {
  return guarded([&] {
    require_model(m);
    if (!m->train_exec) fail(MOSES_ERR_INVALID_ARG, "no training graph (moses_train_graph_create)");
    for (int64_t i = 0; i < steps; ++i) {
      MOSES_CUDA(cudaGraphLaunch(m->train_parity && m->train_exec2 ? m->train_exec2 : m->train_exec, m->st));
      if (m->train_exec2) m->train_parity ^= 1;
    }
    note_launch(steps * g_graph_kernels);
  });
}
MOSES_API int moses_train_graph_kernels(void) { return int(g_graph_kernels); }

MOSES_API int moses_train_step_device(moses_model_t m, const void* x_dev, int64_t ldx, const float* y_dev, int64_t n,
                                      double lr, double mu, double* loss_out) {
  return guarded([&] {
    require_model(m);
    check_rows(m, n);
    const SgdFuse fz{float(lr), float(mu)};
    long long ld0 = 0;
    const void* x0 = stage_device_rows(m, x_dev, ldx, n, &ld0);
    if (!gradients_core(m, x0, ld0, y_dev, n, nullptr, 0.0, nullptr, &fz)) {
      ProfScope ps(P_UPDATE, m->st);
      sgd_update(m->w, m->mom, m->g, nullptr, m->P, float(lr), float(mu), true, m->shadow(), m->st);
      m->post_update();
      note_launch(1);
    }
    if (loss_out) {
      MOSES_CUDA(cudaMemcpyAsync(loss_out, m->dscal, sizeof(double), cudaMemcpyDeviceToHost, m->st));
      MOSES_CUDA(cudaStreamSynchronize(m->st));
    }
  });
}

MOSES_API int moses_ranking_accuracy(moses_model_t m, const double* x, const double* y, const int64_t* boff,
                                     int32_t nb, int32_t D, double* acc, int64_t* pairs, int64_t* conc) {
  return guarded([&] {
    require_model(m);
    if (D != m->dims[0]) fail(MOSES_ERR_DIM_MISMATCH, "feature width != model input width");
    const long long n = nb > 0 ? boff[nb] : 0;
    float* s = dalloc<float>(n);
    float* yd = dalloc<float>(n);
    long long* seg = dalloc<long long>(n);
    long long* so = dalloc<long long>(nb + 1);
    std::vector<long long> seg_h(n);
    for (int b = 0; b < nb; ++b)
      for (long long r = boff[b]; r < boff[b + 1]; ++r) seg_h[r] = b;
    MOSES_CUDA(cudaMemcpyAsync(seg, seg_h.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, m->st));
    MOSES_CUDA(cudaMemcpyAsync(so, boff, sizeof(long long) * (nb + 1), cudaMemcpyHostToDevice, m->st));
    for (long long r = 0; r < n;) {
      const long long c = std::min(n - r, m->cap);
      upload_rows(m, x + r * D, c, 0);
      dispatch_forward(m, m->act[0], m->ld[0], c, nullptr, false);
      head_scores(m->head_part, m->last_tiles, m->cap, m->head_b(), c, s + r, m->st);
      note_launch(1);
      r += c;
    }
    upload_f32(m, y, n, yd);
    accuracy_counts(s, yd, seg, so, n, nullptr, nullptr, m->dcount, m->st);
    note_launch(1);
    unsigned long long tot[2] = {0, 0};
    MOSES_CUDA(cudaMemcpyAsync(tot, m->dcount, sizeof(tot), cudaMemcpyDeviceToHost, m->st));
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    *pairs = (int64_t)tot[0];
    *conc = (int64_t)tot[1];
    *acc = tot[0] == 0 ? 0.0 : double(tot[1]) / double(tot[0]);
    dfree(s);
    dfree(yd);
    dfree(seg);
    dfree(so);
  });
}

MOSES_API int moses_ranking_loss(const double* s, const double* y, int64_t n, double* loss, int64_t* pairs) {
  return guarded([&] {
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    const int ns = rank_splits(n);
    const size_t bytes = size_t(n) * 48 + size_t(ns) * n * 24 + 8192;
    Carver cv{static_cast<uint8_t*>(sc.ensure(bytes))};
    double* s64 = cv.take<double>(n);
    double* y64 = cv.take<double>(n);
    float* sf = cv.take<float>(n);
    float* yf = cv.take<float>(n);
    float* ca = cv.take<float>(n);
    float* cb = cv.take<float>(n);
    RankWs ws{cv.take<double>(ns * n), cv.take<double>(ns * n), cv.take<long long>(ns * n), ns};
    double* dl = cv.take<double>(4);
    long long* dp = cv.take<long long>(2);
    if (n > 0) {
      MOSES_CUDA(cudaMemcpyAsync(s64, s, 8 * n, cudaMemcpyHostToDevice, sc.st));
      MOSES_CUDA(cudaMemcpyAsync(y64, y, 8 * n, cudaMemcpyHostToDevice, sc.st));
      f64_to_f32(s64, n, sf, sc.st);
      f64_to_f32(y64, n, yf, sc.st);
      rank_pairs(sf, yf, n, ws, sc.st);
      note_launch(3);  // two conversions + pairs
    }
    rank_finalize(ws, n, 0, nullptr, 0, 0, nullptr, 0.0, {dl, dp, ca, cb, dl + 1}, sc.st);
    note_launch(1);
    long long p = 0;
    MOSES_CUDA(cudaMemcpyAsync(loss, dl, 8, cudaMemcpyDeviceToHost, sc.st));
    MOSES_CUDA(cudaMemcpyAsync(&p, dp, 8, cudaMemcpyDeviceToHost, sc.st));
    MOSES_CUDA(cudaStreamSynchronize(sc.st));
    if (pairs) *pairs = p;
  });
}

// ---------------------------------------------------------------- lottery
MOSES_API int moses_xi_scores(moses_model_t m, int32_t normalize, double* xi_out, int64_t count) {
  return guarded([&] {
    require_model(m);
    xi_scores(m->w, m->g, m->P, normalize != 0, m->sel, m->xi, m->st);
    note_launch(normalize ? 3 : 2);
    m->xi_valid = true;
    m->xi_norm = normalize != 0;
    if (xi_out) {
      if (count != m->P) fail(MOSES_ERR_SHAPE_MISMATCH, "xi count mismatch");
      download_f32(m, m->xi, count, xi_out);
    }
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

MOSES_API int moses_xi_upload(moses_model_t m, const double* xi, int64_t count, int32_t normalized) {
  return guarded([&] {
    require_model(m);
    if (count != m->P) fail(MOSES_ERR_SHAPE_MISMATCH, "xi count mismatch");
    upload_f32(m, xi, count, m->xi);
    m->xi_valid = true;
    m->xi_norm = normalized != 0;
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

MOSES_API int moses_mask_upload(moses_model_t m, const uint8_t* mask, int64_t count) {
  return guarded([&] {
    require_model(m);
    upload_mask(m, mask, count);
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

static long long partition_validate(moses_model* m, int mode, double value, bool normalized) {
  const long long n = m->P;
  if (n == 0) fail(MOSES_ERR_SHAPE_MISMATCH, "empty score array");
  if (mode == MOSES_MODE_THRESHOLD) {
    if (!normalized) fail(MOSES_ERR_UNNORMALIZED_THRESHOLD, "threshold partition needs normalized scores");
    return -1;
  }
  if (mode != MOSES_MODE_RATIO) fail(MOSES_ERR_INVALID_ARG, "unknown partition mode");
  if (!(value > 0.0) || value > 1.0) fail(MOSES_ERR_INVALID_RATIO, "ratio must lie in (0,1], got " + std::to_string(value));
  return (long long)std::ceil(value * double(n));  // lottery.cpp:160, fp64 like the reference
}

static long long finish_mask(moses_model* m, int mode, long long keep, uint8_t* mask_out, int64_t count) {
  long long pop;
  if (mode == MOSES_MODE_RATIO) pop = std::min(keep, m->P);
  else pop = popcount_mask(m->mask, m->P, m->dcount, m->st), note_launch(1);
  if (mask_out) {
    if (count != m->P) fail(MOSES_ERR_SHAPE_MISMATCH, "mask count mismatch");
    MOSES_CUDA(cudaMemcpyAsync(mask_out, m->mask, m->P, cudaMemcpyDeviceToHost, m->st));
  }
  MOSES_CUDA(cudaStreamSynchronize(m->st));
  m->mask_valid = true;
  return pop;
}

MOSES_API int moses_partition(moses_model_t m, int32_t mode, double value, int32_t phase, uint8_t* mask_out,
                              int64_t count, int64_t* popcount) {
  (void)phase;  // carried by the caller's ParamMask (lottery.hpp:25-32)
  return guarded([&] {
    require_model(m);
    if (!m->xi_valid) fail(MOSES_ERR_SHAPE_MISMATCH, "no xi scores on the device (call moses_xi_scores)");
    const long long keep = partition_validate(m, mode, value, m->xi_norm);
    if (mode == MOSES_MODE_RATIO && keep >= m->P) {
      MOSES_CUDA(cudaMemsetAsync(m->mask, 1, m->P, m->st));
    } else {
      partition_from_xi(m->xi, m->P, mode, float(value), keep, m->sel, m->mask, m->st);
      note_launch(mode == MOSES_MODE_RATIO ? 9 : 3);
    }
    const long long pop = finish_mask(m, mode, keep, mask_out, count);
    if (popcount) *popcount = pop;
  });
}

MOSES_API int moses_transferable_step(moses_model_t m, double alpha) {
  return guarded([&] {
    require_model(m);
    if (!m->mask_valid) fail(MOSES_ERR_SHAPE_MISMATCH, "mask length != parameter count");
    lottery_apply(m->w, m->g, m->mask, m->P, float(alpha), 1.f, true, false, m->shadow(), m->st);
    m->post_update();
    note_launch(1);
    m->xi_valid = false;
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

static float decay_factor(double alpha, double lambda, bool* noop) {
  const double rate = alpha * lambda;
  if (!(rate >= 0.0) || rate >= 1.0)
    fail(MOSES_ERR_UNSTABLE_DECAY, "decay rate alpha*lambda = " + std::to_string(rate) + " must lie in [0,1)");
  *noop = rate == 0.0;
  return float(1.0 - rate);
}

MOSES_API int moses_variant_decay(moses_model_t m, double alpha, double lambda) {
  return guarded([&] {
    require_model(m);
    if (!m->mask_valid) fail(MOSES_ERR_SHAPE_MISMATCH, "mask length != parameter count");
    bool noop = false;
    const float f = decay_factor(alpha, lambda, &noop);
    if (noop) return;
    lottery_apply(m->w, m->g, m->mask, m->P, 0.f, f, false, true, m->shadow(), m->st);
    m->post_update();
    note_launch(1);
    m->xi_valid = false;
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

static void lottery_step_impl(moses_model* m, int32_t mode, double value, double alpha, double lambda,
                              uint8_t* mask_out, int64_t count, int64_t* popcount, const AdamOpt* adam) {
  {
    require_model(m);
    const long long keep = partition_validate(m, mode, value, true /* the tuner normalises in threshold mode */);
    // step on kept scalars; decay the rest (reference order: step, then decay validation)
    const double rate = alpha * lambda;
    const bool decay_ok = (rate >= 0.0) && rate < 1.0;
    const bool decay = decay_ok && rate != 0.0;
    if (mode == MOSES_MODE_RATIO && keep >= m->P) {
      MOSES_CUDA(cudaMemsetAsync(m->mask, 1, m->P, m->st));
      if (adam) {  // every scalar is transferable: masked Adam over all of them, no decay
        adam_update(m->w, adam->m1, adam->m2, m->g, nullptr, m->P, float(alpha), adam->b1, adam->b2, adam->eps,
                    adam->c1, adam->c2, m->shadow(), m->st);
      } else {
        lottery_apply(m->w, m->g, m->mask, m->P, float(alpha), float(1.0 - rate), true, decay, m->shadow(), m->st);
      }
      m->post_update();
      note_launch(1);
    } else {
      if (!m->lot_ws) {
        MOSES_CUDA(cudaMalloc(&m->lot_ws, lottery_ws_bytes(m->P)));
        MOSES_CUDA(cudaMemsetAsync(m->lot_ws, 0, lottery_ws_bytes(m->P), m->st));  // barrier state of the resident step
      }
      ProfScope ps(P_SELECT, m->st);
      // the step writes every operand shadow itself (split pairs included)
      const int launched = lottery_step_fused(m->w, m->g, m->P, mode, float(value), keep, float(alpha),
                                              float(1.0 - rate), decay, m->shadow_full(), m->mask, m->lot_ws, m->dcount,
                                              m->st, adam);
      note_launch(launched);
    }
    m->xi_valid = false;
    long long pop = std::min(keep, m->P);
    if (mode == MOSES_MODE_THRESHOLD) {  // the counted kept scalars, through the pinned scalar slot
      if (!m->host_sc) MOSES_CUDA(cudaMallocHost(&m->host_sc, 4 * sizeof(double)));
      unsigned long long* h = reinterpret_cast<unsigned long long*>(m->host_sc + 3);
      MOSES_CUDA(cudaMemcpyAsync(h, m->dcount, sizeof(*h), cudaMemcpyDeviceToHost, m->st));
      MOSES_CUDA(cudaStreamSynchronize(m->st));
      pop = (long long)*h;
    }
    if (mask_out) {
      if (count != m->P) fail(MOSES_ERR_SHAPE_MISMATCH, "mask count mismatch");
      MOSES_CUDA(cudaMemcpyAsync(mask_out, m->mask, m->P, cudaMemcpyDeviceToHost, m->st));
    }
    if (sync_updates() || mask_out) MOSES_CUDA(cudaStreamSynchronize(m->st));
    m->mask_valid = true;
    if (popcount) *popcount = pop;
    if (!decay_ok) {
      bool noop;
      decay_factor(alpha, lambda, &noop);
    }
  }
}

MOSES_API int moses_lottery_step(moses_model_t m, int32_t mode, double value, int32_t phase, double alpha,
                                 double lambda, uint8_t* mask_out, int64_t count, int64_t* popcount) {
  (void)phase;
  return guarded([&] { lottery_step_impl(m, mode, value, alpha, lambda, mask_out, count, popcount, nullptr); });
}

MOSES_API int moses_lottery_step_adam(moses_model_t m, int32_t mode, double value, int32_t phase, double lr,
                                      double beta1, double beta2, double eps, int32_t step, double lambda,
                                      uint8_t* mask_out, int64_t count, int64_t* popcount) {
  (void)phase;
  return guarded([&] {
    require_model(m);
    if (step < 1) fail(MOSES_ERR_INVALID_ARG, "adam step must be >= 1");
    if (!m->m1) {
      m->m1 = dalloc<float>(m->P);
      m->m2 = dalloc<float>(m->P);
      MOSES_CUDA(cudaMemsetAsync(m->m1, 0, m->P * 4, m->st));
      MOSES_CUDA(cudaMemsetAsync(m->m2, 0, m->P * 4, m->st));
    }
    const AdamOpt o{m->m1, m->m2, float(beta1), float(beta2), float(eps), float(1.0 - std::pow(beta1, step)),
                    float(1.0 - std::pow(beta2, step))};
    lottery_step_impl(m, mode, value, lr, lambda, mask_out, count, popcount, &o);
  });
}



// ---------------------------------------------------------------- adversary
MOSES_API int moses_adversary_create(const double* replay, int64_t mrows, int32_t D, int32_t width, double step,
                                     moses_adversary_t* out) {
  return guarded([&] {
    *out = nullptr;
    if (mrows == 0) fail(MOSES_ERR_ADVERSARY_DISABLED, "replay buffer must be non-empty");  // lottery.cpp:168-169
    if (width <= 0) fail(MOSES_ERR_BAD_DIMS, "penultimate width must be positive");
    auto a = std::make_unique<moses_adversary>();
    a->D = D;
    a->W = width;
    a->m = mrows;
    a->eta = float(step);
    a->replay = dalloc<float>(mrows * D);
    a->u = dalloc<float>(width);
    a->c = dalloc<float>(1);
    std::vector<float> tmp(mrows * D);
    for (long long i = 0; i < mrows * D; ++i) tmp[i] = float(replay[i]);
    MOSES_CUDA(cudaMemcpy(a->replay, tmp.data(), 4 * tmp.size(), cudaMemcpyHostToDevice));
    MOSES_CUDA(cudaMemset(a->u, 0, 4 * width));
    MOSES_CUDA(cudaMemset(a->c, 0, 4));
    // the adversary is used on model streams (non-blocking: no implicit order with the legacy stream)
    MOSES_CUDA(cudaDeviceSynchronize());
    *out = a.release();
  });
}
MOSES_API int moses_adversary_destroy(moses_adversary_t a) {
  return guarded([&] { delete a; });
}
MOSES_API int moses_adversary_get(moses_adversary_t a, double* w, int32_t width, double* b) {
  return guarded([&] {
    if (width != a->W) fail(MOSES_ERR_DIM_MISMATCH, "width mismatch");
    std::vector<float> t(width + 1);
    MOSES_CUDA(cudaDeviceSynchronize());  // model streams may still be updating the discriminator
    MOSES_CUDA(cudaMemcpy(t.data(), a->u, 4 * width, cudaMemcpyDeviceToHost));
    MOSES_CUDA(cudaMemcpy(t.data() + width, a->c, 4, cudaMemcpyDeviceToHost));
    for (int j = 0; j < width; ++j) w[j] = t[j];
    *b = t[width];
  });
}
MOSES_API int moses_adversary_set(moses_adversary_t a, const double* w, int32_t width, double b) {
  return guarded([&] {
    if (width != a->W) fail(MOSES_ERR_DIM_MISMATCH, "width mismatch");
    std::vector<float> t(width + 1);
    for (int j = 0; j < width; ++j) t[j] = float(w[j]);
    t[width] = float(b);
    MOSES_CUDA(cudaDeviceSynchronize());  // no model stream may still read the old discriminator
    MOSES_CUDA(cudaMemcpy(a->u, t.data(), 4 * width, cudaMemcpyHostToDevice));
    MOSES_CUDA(cudaMemcpy(a->c, t.data() + width, 4, cudaMemcpyHostToDevice));
    MOSES_CUDA(cudaDeviceSynchronize());
  });
}

MOSES_API int moses_adversarial_step(moses_adversary_t a, moses_model_t m, const double* x, int64_t n, int32_t D,
                                     double beta, double* dloss, double* conf) {
  return guarded([&] {
    require_model(m);
    if (!a) fail(MOSES_ERR_ADVERSARY_DISABLED, "null adversary");
    if (a->m == 0) fail(MOSES_ERR_ADVERSARY_DISABLED, "adversary has an empty replay buffer");
    if (n == 0) fail(MOSES_ERR_ADVERSARY_DISABLED, "empty activation batch");
    if (a->W != m->W()) fail(MOSES_ERR_DIM_MISMATCH, "activation width != discriminator width");
    if (D != m->dims[0] || a->D != m->dims[0]) fail(MOSES_ERR_DIM_MISMATCH, "feature width != model input width");
    check_rows(m, a->m + n);
    upload_replay(m, a);
    upload_rows(m, x, n, a->m);
    dispatch_forward(m, m->act[0], m->ld[0], a->m + n, a->u, true);
    if (m->esz == 2)
      adversary_step<__nv_bfloat16>(m->head_part2, m->last_tiles, m->cap, static_cast<__nv_bfloat16*>(m->act[m->L - 1]),
                                    m->ld[m->L - 1], a->m, n, m->W(), a->u, a->c, a->eta, m->dscal + 2, m->adv_ws, m->st,
                                    m->act_lo_t<__nv_bfloat16>(m->L - 1));
    else
      adversary_step<float>(m->head_part2, m->last_tiles, m->cap, static_cast<float*>(m->act[m->L - 1]),
                            m->ld[m->L - 1], a->m, n, m->W(), a->u, a->c, a->eta, m->dscal + 2, m->adv_ws, m->st,
                            m->act_lo_t<float>(m->L - 1));
    note_launch(3);
    double l = 0;
    MOSES_CUDA(cudaMemcpyAsync(&l, m->dscal + 2, 8, cudaMemcpyDeviceToHost, m->st));
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    if (dloss) *dloss = l;
    if (conf) *conf = -beta * l;
  });
}

// evolve (search.cpp:41-71, SearchParams search.hpp:13-20) with the scorer on the device: every
// generation's configurations are encoded on the device straight into packed model rows (from
// their enumeration indices) and scored by the model there; the GA's own RngStream walk
// (sample_config / mutate_config / epsilon draws, space.cpp:94-121) and the sort of <= a few
// hundred candidates by (score desc, configuration asc) stay on the host — both are sequential
// by definition. Configurations compare lexicographically by value, which for sorted domains is
// the order of their mixed-radix enumeration index. m == NULL scores with the linear test scorer
// sum_k lin_w[k] * value_k (host, double) instead of the model.
namespace {
struct EvolveSpace {
  int nk;
  std::vector<long long> dom;
  std::vector<int> size, off;
  unsigned long long idx_of(const std::vector<int>& dg) const {
    unsigned long long id = 0;
    for (int k = 0; k < nk; ++k) id = id * (unsigned long long)size[k] + (unsigned long long)dg[k];
    return id;
  }
  std::vector<int> digits(unsigned long long id) const {
    std::vector<int> dg(static_cast<size_t>(nk));
    for (int k = nk - 1; k >= 0; --k) {
      dg[size_t(k)] = int(id % (unsigned long long)size[k]);
      id /= (unsigned long long)size[k];
    }
    return dg;
  }
};
struct GaRng {  // RngStream (rng.hpp)
  unsigned long long s;
  unsigned long long next() {
    s += 0x9e3779b97f4a7c15ull;
    unsigned long long z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  unsigned long long below(unsigned long long n) {
    const unsigned long long t = (0ull - n) % n;
    for (;;) {
      const unsigned long long r = next();
      if (r >= t) return r % n;
    }
  }
  double uniform01() { return double(next() >> 11) * 0x1.0p-53; }
};
}  // namespace

// accessors for the other translation units (tuner.cu); C++ linkage inside the extern "C" block
extern "C++" {
namespace moses {
void set_last_error(const std::string& msg) { g_err = msg; }
int model_device(const moses_model* m) { return m->device; }
std::vector<int> model_dims(const moses_model* m) { return m->dims; }
}  // namespace moses
}

MOSES_API int moses_evolve(moses_model_t m, const double* lin_w, const double* task4, const int64_t* domains,
                          const int32_t* domain_sizes, const int32_t* roles, int32_t n_knobs, int32_t population,
                          int32_t generations, int32_t mutation_count, int32_t survivors, double epsilon_random,
                          uint64_t seed, int64_t* values_out, double* scores_out, int64_t capacity, int64_t* n_out) {
  return guarded([&] {
    // check_params (search.cpp:11-19)
    if (population < 1 || mutation_count < 1 || survivors < 1)
      fail(MOSES_ERR_INVALID_CONFIG, "population, mutation_count and survivors must be positive");
    if (generations < 0) fail(MOSES_ERR_INVALID_CONFIG, "generations must be non-negative");
    if (survivors > population) fail(MOSES_ERR_INVALID_CONFIG, "survivors cannot exceed the population");
    if (!(epsilon_random >= 0.0 && epsilon_random <= 1.0))
      fail(MOSES_ERR_INVALID_CONFIG, "epsilon_random must lie in [0,1]");
    if (m == nullptr && lin_w == nullptr) fail(MOSES_ERR_INVALID_ARG, "no scorer");
    if (m != nullptr && m->dims[0] < 10) fail(MOSES_ERR_DIM_MISMATCH, "model input width below the feature width");
    // build_space / validate_task (space.cpp:41-92)
    if (n_knobs <= 0 || n_knobs > 8) fail(MOSES_ERR_INVALID_ARG, "knob count must lie in [1, 8]");
    EvolveSpace sp;
    sp.nk = n_knobs;
    int off = 0;
    unsigned long long space = 1;
    for (int k = 0; k < n_knobs; ++k) {
      if (domain_sizes[k] <= 0) fail(MOSES_ERR_INVALID_TASK, "knob domain must be non-empty");
      for (int j = 1; j < domain_sizes[k]; ++j)
        if (domains[off + j - 1] >= domains[off + j]) fail(MOSES_ERR_INVALID_TASK, "knob domain must be strictly increasing");
      if (space > ~0ull / (unsigned long long)domain_sizes[k]) fail(MOSES_ERR_SPACE_TOO_LARGE, "knob space overflows 64 bits");
      space *= (unsigned long long)domain_sizes[k];
      sp.size.push_back(domain_sizes[k]);
      sp.off.push_back(off);
      off += domain_sizes[k];
    }
    sp.dom.assign(domains, domains + off);
    std::vector<int> mutable_knobs;
    for (int k = 0; k < n_knobs; ++k)
      if (sp.size[size_t(k)] > 1) mutable_knobs.push_back(k);

    GaRng rng{0xcbf29ce484222325ull};
    {  // KeyBuilder(seed, "evolve")
      auto step = [&](unsigned char b) {
        rng.s ^= b;
        rng.s *= 0x100000001b3ull;
      };
      for (int i = 0; i < 8; ++i) step((unsigned char)(seed >> (8 * i)));
      for (const char* c = "evolve"; *c; ++c) step((unsigned char)*c);
      step(0);
    }
    auto sample = [&] {  // sample_config (space.cpp:94-100)
      std::vector<int> dg(static_cast<size_t>(n_knobs));
      for (int k = 0; k < n_knobs; ++k) dg[size_t(k)] = int(rng.below((unsigned long long)sp.size[size_t(k)]));
      return sp.idx_of(dg);
    };
    auto mutate = [&](unsigned long long id) {  // mutate_config (space.cpp:102-121)
      if (mutable_knobs.empty()) fail(MOSES_ERR_IMMUTABLE_SPACE, "every knob domain is a singleton");
      std::vector<int> dg = sp.digits(id);
      const int ki = mutable_knobs[size_t(rng.below(mutable_knobs.size()))];
      const int old_pos = dg[size_t(ki)];
      int pick = int(rng.below((unsigned long long)(sp.size[size_t(ki)] - 1)));
      if (pick >= old_pos) ++pick;
      dg[size_t(ki)] = pick;
      return sp.idx_of(dg);
    };
    // scoring: device encode (from indices) + predict, or the linear test scorer
    unsigned long long* didx = nullptr;
    void* feat = nullptr;
    float* dsc = nullptr;
    const long long maxn = std::max<long long>(population, (long long)survivors * (1 + mutation_count));
    cudaStream_t st = m ? m->st : nullptr;
    auto release = [&] {
      if (st) cudaStreamSynchronize(st);
      dfree(didx);
      dfree(feat);
      dfree(dsc);
    };
    struct Cand {
      unsigned long long idx;
      double score;
    };
    auto score_all = [&](const std::vector<unsigned long long>& ids) {
      std::vector<Cand> pop(ids.size());
      if (m == nullptr) {
        for (size_t i = 0; i < ids.size(); ++i) {
          const std::vector<int> dg = sp.digits(ids[i]);
          double sc = 0.0;
          for (int k = 0; k < n_knobs; ++k) sc = sc + lin_w[k] * double(sp.dom[size_t(sp.off[size_t(k)] + dg[size_t(k)])]);
          pop[i] = {ids[i], sc};
        }
        return pop;
      }
      const long long n = (long long)ids.size();
      MOSES_CUDA(cudaMemcpyAsync(didx, ids.data(), sizeof(unsigned long long) * n, cudaMemcpyHostToDevice, st));
      // rows in the handle's device input type (split handles: fp32, split into their planes per chunk)
      note_launch(encode_configs_idx(task4, reinterpret_cast<const long long*>(domains), domain_sizes, roles, n_knobs,
                                     didx, n, m->in_esz() == 2 ? MOSES_DTYPE_BF16 : MOSES_DTYPE_F32, feat, m->ld[0],
                                     m->dims[0], st));
      for (long long r = 0; r < n;) {
        const long long c = std::min(n - r, m->cap);
        long long ld0 = 0;
        const void* x0 = stage_device_rows(m, static_cast<uint8_t*>(feat) + r * m->ld[0] * m->in_esz(), m->ld[0], c, &ld0);
        dispatch_forward(m, x0, ld0, c, nullptr, false);
        head_scores(m->head_part, m->last_tiles, m->cap, m->head_b(), c, dsc + r, st);
        note_launch(1);
        r += c;
      }
      std::vector<float> hs(static_cast<size_t>(n));
      MOSES_CUDA(cudaMemcpyAsync(hs.data(), dsc, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
      MOSES_CUDA(cudaStreamSynchronize(st));
      for (size_t i = 0; i < ids.size(); ++i) pop[i] = {ids[i], double(hs[i])};
      return pop;
    };
    auto sort_desc = [](std::vector<Cand>& pop) {  // search.cpp:32-37
      std::sort(pop.begin(), pop.end(), [](const Cand& a, const Cand& b) {
        if (a.score != b.score) return a.score > b.score;
        return a.idx < b.idx;
      });
    };
    std::vector<Cand> pop;
    try {
      if (m) {
        didx = dalloc<unsigned long long>(size_t(maxn));
        feat = dalloc<uint8_t>(size_t(maxn) * m->ld[0] * m->in_esz());
        dsc = dalloc<float>(size_t(maxn));
      }
      std::vector<unsigned long long> ids;
      ids.reserve(size_t(population));
      for (int i = 0; i < population; ++i) ids.push_back(sample());
      pop = score_all(ids);
      sort_desc(pop);
      for (int gen = 0; gen < generations; ++gen) {
        const size_t keep = std::min<size_t>(size_t(survivors), pop.size());
        std::vector<unsigned long long> next;
        next.reserve(keep * size_t(1 + mutation_count));
        for (size_t s2 = 0; s2 < keep; ++s2) next.push_back(pop[s2].idx);
        for (size_t s2 = 0; s2 < keep; ++s2)
          for (int k = 0; k < mutation_count; ++k)
            next.push_back(rng.uniform01() < epsilon_random ? sample() : mutate(pop[s2].idx));
        pop = score_all(next);
        sort_desc(pop);
      }
    } catch (...) {
      release();
      throw;
    }
    release();
    if ((long long)pop.size() > capacity) fail(MOSES_ERR_CAPACITY, "output capacity below the final population");
    for (size_t i = 0; i < pop.size(); ++i) {
      const std::vector<int> dg = sp.digits(pop[i].idx);
      for (int k = 0; k < n_knobs; ++k)
        if (values_out) values_out[i * n_knobs + k] = sp.dom[size_t(sp.off[size_t(k)] + dg[size_t(k)])];
      if (scores_out) scores_out[i] = pop[i].score;
    }
    if (n_out) *n_out = (int64_t)pop.size();
  });
}

// The Moses branch of a tuning step (tuner.cpp:251-262) in one call: gradients with the
// adversary term -> discriminator step -> lottery step, with one host synchronisation. The
// discriminator step reuses the forward pass the gradients just ran on the same rows (replay
// [0, m), batch [m, m+n), discriminator logits in the same epilogue) — moses_adversarial_step
// would re-upload and recompute exactly these values, since the model has not changed in between.
MOSES_API int moses_moses_step(moses_model_t m, moses_adversary_t a, const double* x, const double* y, int64_t n,
                              int32_t D, double beta, int32_t mode, double value, int32_t phase, double alpha,
                              double lambda, double* loss_out, double* dloss_out, int64_t* popcount) {
  (void)phase;
  return guarded([&] {
    require_model(m);
    if (!a) fail(MOSES_ERR_ADVERSARY_DISABLED, "null adversary");
    if (a->m == 0) fail(MOSES_ERR_ADVERSARY_DISABLED, "adversary has an empty replay buffer");
    if (n == 0) fail(MOSES_ERR_ADVERSARY_DISABLED, "empty activation batch");
    if (a->W != m->W()) fail(MOSES_ERR_DIM_MISMATCH, "activation width != discriminator width");
    gradients_host(m, x, y, n, D, a, beta);
    if (beta == 0.0) {  // the gradients ran without the adversary rows: forward them for the discriminator
      upload_replay(m, a);
      upload_rows(m, x, n, a->m);
      dispatch_forward(m, m->act[0], m->ld[0], a->m + n, a->u, true);
      note_launch(1);
    }
    if (m->esz == 2)
      adversary_step<__nv_bfloat16>(m->head_part2, m->last_tiles, m->cap, static_cast<__nv_bfloat16*>(m->act[m->L - 1]),
                                    m->ld[m->L - 1], a->m, n, m->W(), a->u, a->c, a->eta, m->dscal + 2, m->adv_ws, m->st,
                                    m->act_lo_t<__nv_bfloat16>(m->L - 1));
    else
      adversary_step<float>(m->head_part2, m->last_tiles, m->cap, static_cast<float*>(m->act[m->L - 1]),
                            m->ld[m->L - 1], a->m, n, m->W(), a->u, a->c, a->eta, m->dscal + 2, m->adv_ws, m->st,
                            m->act_lo_t<float>(m->L - 1));
    note_launch(2);
    // the scalars land in pinned memory asynchronously (a pageable copy would block the host before the
    // lottery step is even launched); one synchronisation at the end
    if (!m->host_sc) MOSES_CUDA(cudaMallocHost(&m->host_sc, 4 * sizeof(double)));
    double* sc = m->host_sc;
    MOSES_CUDA(cudaMemcpyAsync(sc, m->dscal, 3 * sizeof(double), cudaMemcpyDeviceToHost, m->st));
    lottery_step_impl(m, mode, value, alpha, lambda, nullptr, 0, popcount, nullptr);
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    if (loss_out) *loss_out = sc[0];
    if (dloss_out) *dloss_out = sc[2];
  });
}

MOSES_API int moses_adversarial_term(moses_adversary_t a, const double* hs, int64_t ms, const double* ht, int64_t nt,
                                     int32_t width, double beta, double* dloss, double* conf) {
  return guarded([&] {
    if (!a || a->m == 0) fail(MOSES_ERR_ADVERSARY_DISABLED, "adversary has an empty replay buffer");
    if (ms == 0 || nt == 0) fail(MOSES_ERR_ADVERSARY_DISABLED, "empty activation batch");
    if (width != a->W) fail(MOSES_ERR_DIM_MISMATCH, "activation width != discriminator width");
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    const long long R = ms + nt;
    const size_t bytes = size_t(R) * width * 12 + size_t(R) * 16 + size_t(width) * 16 + column_dot_ws_floats(R, width) * 4 + 16384;
    Carver cv{static_cast<uint8_t*>(sc.ensure(bytes))};
    double* h64 = cv.take<double>(R * width);
    float* H = cv.take<float>(R * width);
    float* z = cv.take<float>(R);
    float* ws = cv.take<float>(round_up(R, 64) + round_up(width + 1, 64) + 64 + 16 + column_dot_ws_floats(R, width) + 64);
    double* dl = cv.take<double>(2);
    MOSES_CUDA(cudaMemcpyAsync(h64, hs, 8 * ms * width, cudaMemcpyHostToDevice, sc.st));
    MOSES_CUDA(cudaMemcpyAsync(h64 + ms * width, ht, 8 * nt * width, cudaMemcpyHostToDevice, sc.st));
    f64_to_f32(h64, R * width, H, sc.st);
    // logits as a single "tile" of partials: z_r = H_r . u
    row_dot(H, width, R, width, a->u, z, sc.st);
    adversary_step<float>(z, 1, R, H, width, ms, nt, width, a->u, a->c, a->eta, dl, ws, sc.st);
    note_launch(5);
    double l = 0;
    MOSES_CUDA(cudaMemcpyAsync(&l, dl, 8, cudaMemcpyDeviceToHost, sc.st));
    MOSES_CUDA(cudaStreamSynchronize(sc.st));
    if (dloss) *dloss = l;
    if (conf) *conf = -beta * l;
  });
}

MOSES_API int moses_discriminator_cross_entropy(const double* zs, int64_t m, const double* zt, int64_t n, double* out) {
  return guarded([&] {
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    Carver cv{static_cast<uint8_t*>(sc.ensure(size_t(m + n) * 8 + 4096))};
    double* z = cv.take<double>(m + n);
    double* o = cv.take<double>(1);
    MOSES_CUDA(cudaMemcpyAsync(z, zs, 8 * m, cudaMemcpyHostToDevice, sc.st));
    MOSES_CUDA(cudaMemcpyAsync(z + m, zt, 8 * n, cudaMemcpyHostToDevice, sc.st));
    disc_ce(z, m, n, o, sc.st);
    note_launch(1);
    MOSES_CUDA(cudaMemcpyAsync(out, o, 8, cudaMemcpyDeviceToHost, sc.st));
    MOSES_CUDA(cudaStreamSynchronize(sc.st));
  });
}

// ---------------------------------------------------------------- candidate selection
MOSES_API int moses_topk_device(const float* scores, int64_t n, int64_t k, int64_t* idx_out) {
  return guarded([&] {
    if (k <= 0 || n <= 0) return;
    if (k > n) k = n;
    if (k > kTopkMax) fail(MOSES_ERR_INVALID_ARG, "k must be <= 4096");
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    const size_t selb = select_ws_bytes(n, nullptr);
    Carver cv{static_cast<uint8_t*>(sc.ensure(selb + (kTopkMax * 12) + topk_fast_ws_bytes(n) + 8192))};
    uint8_t* selbase = cv.take<uint8_t>(selb);
    unsigned* ok = cv.take<unsigned>(kTopkMax);
    long long* oi = cv.take<long long>(kTopkMax);
    void* fast_ws = cv.take<uint8_t>(topk_fast_ws_bytes(n));
    SelectWs ws;
    select_ws_carve(selbase, n, &ws);
    long long* hb = sc.pinned();  // [0] = not-conclusive flag (first 4 bytes), [1, k] = indices
    bool done = false;
    {
      ProfScope ps(P_TOPK, sc.st);
      // one launch (one read of the pool) when the sampled threshold is conclusive: it writes its flag
      // and the indices straight into pinned host memory (no copy behind it); else the exact radix passes
      if (topk_fast_launch(scores, n, k, fast_ws, ok, sc.host_dev + 1, reinterpret_cast<unsigned*>(sc.host_dev),
                           sc.st)) {
        note_launch(1);
        MOSES_CUDA(cudaStreamSynchronize(sc.st));
        done = *reinterpret_cast<const volatile unsigned*>(hb) == 0;
      }
      if (!done) {
        topk_select(scores, n, k, ws, ok, oi, sc.st);
        note_launch(10);
        MOSES_CUDA(cudaMemcpyAsync(hb + 1, oi, sizeof(long long) * k, cudaMemcpyDeviceToHost, sc.st));
        MOSES_CUDA(cudaStreamSynchronize(sc.st));
      }
    }
    std::memcpy(idx_out, hb + 1, sizeof(long long) * k);
  });
}

// ====================================================================== NCCL communicators + data parallel
MOSES_API int moses_comm_unique_id(uint8_t* id_out, int64_t cap) {
  return guarded([&] {
    if (id_out == nullptr || cap < int64_t(sizeof(ncclUniqueId))) fail(MOSES_ERR_INVALID_ARG, "id buffer too small");
    ncclUniqueId id;
    MOSES_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

MOSES_API int moses_comm_init_rank(const uint8_t* id, int32_t nranks, int32_t rank, moses_comm_t* out) {
  return guarded([&] {
    *out = nullptr;
    if (id == nullptr || nranks < 1 || rank < 0 || rank >= nranks) fail(MOSES_ERR_INVALID_ARG, "bad rank / size");
    auto c = std::make_unique<moses_comm>();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    MOSES_CUDA(cudaGetDevice(&c->device));
    MOSES_NCCL(nccl().CommInitRank(&c->comm, nranks, uid, rank));
    c->nranks = nranks;
    c->rank = rank;
    *out = c.release();
  });
}

MOSES_API int moses_comm_init_all(int32_t ndev, const int32_t* devices, moses_comm_t* out) {
  return guarded([&] {
    if (ndev < 1 || devices == nullptr || out == nullptr) fail(MOSES_ERR_INVALID_ARG, "empty device list");
    std::vector<ncclComm_t> comms(static_cast<size_t>(ndev));
    MOSES_NCCL(nccl().CommInitAll(comms.data(), ndev, devices));
    for (int i = 0; i < ndev; ++i) {
      auto* c = new moses_comm();
      c->comm = comms[size_t(i)];
      c->nranks = ndev;
      c->rank = i;
      c->device = devices[i];
      out[i] = c;
    }
  });
}

MOSES_API int moses_comm_destroy(moses_comm_t c) {
  return guarded([&] {
    if (c == nullptr) return;
    if (c->comm) nccl().CommDestroy(c->comm);
    delete c;
  });
}

MOSES_API int moses_comm_info(moses_comm_t c, int32_t* nranks, int32_t* rank, int32_t* device) {
  return guarded([&] {
    if (c == nullptr) fail(MOSES_ERR_INVALID_ARG, "null communicator");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    if (device) *device = c->device;
  });
}

MOSES_API int moses_model_set_comm(moses_model_t m, moses_comm_t c, int32_t mode) {
  return guarded([&] {
    require_model(m);
    if (mode < 0 || mode > 2 || (mode != 0 && c == nullptr)) fail(MOSES_ERR_INVALID_ARG, "bad data-parallel mode");
    if (c != nullptr && c->device != m->device) fail(MOSES_ERR_INVALID_ARG, "communicator and model on different devices");
    for (cudaGraphExec_t* e : {&m->train_exec, &m->train_exec2})  // graphs captured for the old mode
      if (*e) {
        cudaGraphExecDestroy(*e);
        *e = nullptr;
      }
    m->comm = mode == 0 ? nullptr : c;
    m->comm_mode = mode == 0 ? 0 : mode;
  });
}

MOSES_API int moses_dp_allreduce_gradients(moses_model_t m, int32_t average) {
  return guarded([&] {
    require_model(m);
    if (!m->comm) fail(MOSES_ERR_INVALID_ARG, "no communicator (moses_model_set_comm)");
    comm_allreduce_f32(m->comm, m->g, m->P, average != 0, m->st);
    if (sync_updates()) MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

MOSES_API int moses_dp_train_step(moses_model_t m, const void* x_dev, int64_t ldx, const float* y_dev, int64_t n,
                                  double lr, double mu, double* loss_out) {
  return guarded([&] {
    require_model(m);
    if (!m->comm) fail(MOSES_ERR_INVALID_ARG, "no communicator (moses_model_set_comm)");
    check_rows(m, n);
    long long ld0 = 0;
    const void* x0 = stage_device_rows(m, x_dev, ldx, n, &ld0);
    if (m->comm_mode == 2) {
      dp_exact_step(m, x0, ld0, y_dev, n, true, float(lr), float(mu));
    } else {
      gradients_core(m, x0, ld0, y_dev, n, nullptr, 0.0);
      comm_allreduce_f32(m->comm, m->g, m->P, true, m->st);
      update_momentum(m, float(lr), float(mu), m->st);
    }
    if (loss_out) {
      MOSES_CUDA(cudaMemcpyAsync(loss_out, m->dscal, sizeof(double), cudaMemcpyDeviceToHost, m->st));
      MOSES_CUDA(cudaStreamSynchronize(m->st));
    } else if (sync_updates()) {
      MOSES_CUDA(cudaStreamSynchronize(m->st));
    }
  });
}

MOSES_API int moses_dp_exact_forward(moses_model_t m, const void* x_dev, int64_t ldx, const float* y_dev, int64_t n,
                                     float* s_slot, float* y_slot) {
  return guarded([&] {
    require_model(m);
    check_rows(m, n);
    long long ld0 = 0;
    const void* x0 = stage_device_rows(m, x_dev, ldx, n, &ld0);
    dp_exact_forward(m, x0, ld0, y_dev, n, s_slot, y_slot);
  });
}

MOSES_API int moses_dp_exact_rank(moses_model_t m, const float* s_global, const float* y_global, int64_t n_global,
                                  int64_t p0, double* totals_dev) {
  return guarded([&] {
    require_model(m);
    dp_exact_rank(m, s_global, y_global, n_global, p0, totals_dev);
  });
}

MOSES_API int moses_dp_exact_backward(moses_model_t m, int64_t n_global, const double* totals_dev, double* loss_out) {
  return guarded([&] {
    require_model(m);
    dp_exact_backward(m, n_global, totals_dev);
    if (loss_out) MOSES_CUDA(cudaMemcpyAsync(loss_out, m->dscal, sizeof(double), cudaMemcpyDeviceToHost, m->st));
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

// cfg4 across ranks: local top-k of this rank's contiguous shard [row0, row0 + n_local), the k winners'
// (score, global index) all-gathered over NCCL, merged with the reference comparator (score desc,
// index asc: search.cpp:32-37) — identical on every rank, equal to the single-device top-k of the pool.
MOSES_API int moses_topk_sharded(moses_comm_t c, const float* scores_dev, int64_t n_local, int64_t row0, int64_t k,
                                 int64_t* idx_out) {
  return guarded([&] {
    if (c == nullptr) fail(MOSES_ERR_INVALID_ARG, "null communicator");
    if (k <= 0) return;
    if (k > kTopkMax) fail(MOSES_ERR_INVALID_ARG, "k must be <= 4096");
    const long long kk = std::min<long long>(k, std::max<long long>(n_local, 0));
    MOSES_CUDA(cudaSetDevice(c->device));
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    const long long nsel = std::max<long long>(n_local, 1);
    const size_t selb = select_ws_bytes(nsel, nullptr);
    const size_t gather_b = size_t(k) * (c->nranks + 1) * (sizeof(float) + sizeof(long long));
    Carver cv{static_cast<uint8_t*>(sc.ensure(selb + kTopkMax * 12 + topk_fast_ws_bytes(nsel) + gather_b + 16384))};
    uint8_t* selbase = cv.take<uint8_t>(selb);
    unsigned* ok = cv.take<unsigned>(kTopkMax);
    long long* oi = cv.take<long long>(kTopkMax);
    void* fast_ws = cv.take<uint8_t>(topk_fast_ws_bytes(nsel));
    float* ws_s = cv.take<float>(size_t(k));
    long long* ws_i = cv.take<long long>(size_t(k));
    float* all_s = cv.take<float>(size_t(k) * c->nranks);
    long long* all_i = cv.take<long long>(size_t(k) * c->nranks);
    if (kk > 0) {
      SelectWs ws;
      select_ws_carve(selbase, n_local, &ws);
      ProfScope ps(P_TOPK, sc.st);
      if (topk_fast(scores_dev, n_local, kk, fast_ws, ok, oi, sc.st)) note_launch(1);
      else {
        topk_select(scores_dev, n_local, kk, ws, ok, oi, sc.st);
        note_launch(10);
      }
    }
    topk_winners(scores_dev, oi, kk, k, row0, ws_s, ws_i, sc.st);
    note_launch(1);
    MOSES_NCCL(nccl().GroupStart());
    comm_allgather_bytes(c, ws_s, all_s, k * sizeof(float), sc.st);
    comm_allgather_bytes(c, ws_i, all_i, k * sizeof(long long), sc.st);
    MOSES_NCCL(nccl().GroupEnd());
    std::vector<float> hs(size_t(k) * c->nranks);
    std::vector<long long> hi(size_t(k) * c->nranks);
    MOSES_CUDA(cudaMemcpyAsync(hs.data(), all_s, sizeof(float) * hs.size(), cudaMemcpyDeviceToHost, sc.st));
    MOSES_CUDA(cudaMemcpyAsync(hi.data(), all_i, sizeof(long long) * hi.size(), cudaMemcpyDeviceToHost, sc.st));
    MOSES_CUDA(cudaStreamSynchronize(sc.st));
    std::vector<size_t> order;
    for (size_t i = 0; i < hi.size(); ++i)
      if (hi[i] >= 0) order.push_back(i);
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
      if (hs[a] != hs[b]) return hs[a] > hs[b];
      return hi[a] < hi[b];
    });
    for (long long i = 0; i < k; ++i) idx_out[i] = i < (long long)order.size() ? hi[order[size_t(i)]] : -1;
  });
}

MOSES_API int moses_topk(const double* scores, int64_t n, int64_t k, int64_t* idx_out) {
  return guarded([&] {
    if (k <= 0 || n <= 0) return;
    float* d = dalloc<float>(n);
    double* d64 = dalloc<double>(n);
    MOSES_CUDA(cudaMemcpy(d64, scores, 8 * n, cudaMemcpyHostToDevice));
    f64_to_f32(d64, n, d, nullptr);
    note_launch(1);
    MOSES_CUDA(cudaDeviceSynchronize());
    const int rc = moses_topk_device(d, n, k, idx_out);
    dfree(d);
    dfree(d64);
    if (rc) throw Status(rc, g_err);
  });
}

MOSES_API int64_t moses_select_batch(const uint64_t* hashes, int64_t n, const uint64_t* measured, int64_t nm,
                                     int64_t batch_size, int64_t* out) {
  if (batch_size < 1) {
    g_err = "batch size must be positive";
    return -MOSES_ERR_INVALID_CONFIG;
  }
  std::unordered_set<uint64_t> meas(measured, measured + nm), taken;
  int64_t c = 0;
  for (int64_t i = 0; i < n && c < batch_size; ++i) {
    if (meas.count(hashes[i]) || !taken.insert(hashes[i]).second) continue;
    out[c++] = i;
  }
  return c;
}

// ---------------------------------------------------------------- extensions
MOSES_API int moses_segment_sum_device(const void* h, int32_t dtype, int64_t ld, int32_t width, const int64_t* off,
                                       int64_t programs, float* out) {
  return guarded([&] {
    if (dtype == MOSES_DTYPE_BF16)
      segment_sum<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(h), ld, width, reinterpret_cast<const long long*>(off),
                                 programs, out, width, nullptr);
    else
      segment_sum<float>(static_cast<const float*>(h), ld, width, reinterpret_cast<const long long*>(off), programs, out,
                         width, nullptr);
    note_launch(1);
  });
}

MOSES_API int moses_segment_sum(const double* h, int64_t rows, int32_t width, const int64_t* off, int64_t programs,
                                double* out) {
  return guarded([&] {
    if (programs < 0 || off[0] != 0 || off[programs] != rows) fail(MOSES_ERR_SHAPE_MISMATCH, "offsets must span the rows");
    const int wp = int(round_up(width, 4));
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    const size_t bytes = size_t(rows) * width * 8 + size_t(rows) * wp * 4 + size_t(programs + 1) * 8 +
                         size_t(programs) * wp * 12 + 8192;
    Carver cv{static_cast<uint8_t*>(sc.ensure(bytes))};
    double* h64 = cv.take<double>(rows * width);
    float* H = cv.take<float>(rows * wp);
    long long* doff = cv.take<long long>(programs + 1);
    float* o = cv.take<float>(programs * wp);
    double* o64 = cv.take<double>(programs * wp);
    MOSES_CUDA(cudaMemcpyAsync(h64, h, 8 * rows * width, cudaMemcpyHostToDevice, sc.st));
    MOSES_CUDA(cudaMemcpyAsync(doff, off, 8 * (programs + 1), cudaMemcpyHostToDevice, sc.st));
    MOSES_CUDA(cudaMemsetAsync(H, 0, 4 * rows * wp, sc.st));
    strided_f64_to_f32(h64, rows, width, H, wp, sc.st);
    segment_sum<float>(H, wp, wp, reinterpret_cast<const long long*>(doff), programs, o, wp, sc.st);
    unpack_rows<float>(o, programs, width, wp, o64, sc.st);
    note_launch(3);
    MOSES_CUDA(cudaMemcpyAsync(out, o64, 8 * programs * width, cudaMemcpyDeviceToHost, sc.st));
    MOSES_CUDA(cudaStreamSynchronize(sc.st));
  });
}

MOSES_API int moses_mmd2(const double* xs, int64_t m, const double* xt, int64_t n, int32_t width, double sigma,
                         double* out) {
  return guarded([&] {
    if (m <= 0 || n <= 0) fail(MOSES_ERR_INVALID_ARG, "mmd needs non-empty source and target");
    if (width <= 0) fail(MOSES_ERR_INVALID_ARG, "mmd needs a positive width");
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    const long long R = m + n;
    const size_t wsb = mmd_ws_bytes(m, n, width);
    Carver cv{static_cast<uint8_t*>(sc.ensure(size_t(R) * width * 12 + wsb + 8192))};
    double* h64 = cv.take<double>(R * width);
    float* H = cv.take<float>(R * width);
    void* ws = cv.take<uint8_t>(wsb);
    MOSES_CUDA(cudaMemcpyAsync(h64, xs, 8 * m * width, cudaMemcpyHostToDevice, sc.st));
    MOSES_CUDA(cudaMemcpyAsync(h64 + m * width, xt, 8 * n * width, cudaMemcpyHostToDevice, sc.st));
    f64_to_f32(h64, R * width, H, sc.st);
    int launched = 0;
    *out = mmd2_tc(H, m, H + m * width, n, width, width, float(sigma), ws, sc.st, &launched);
    note_launch(1 + launched);
  });
}

// gradients() with the MMD^2 domain term in the adversary's slot (north-star (4); model.cpp:192-244 with
// beta * MMD^2(H_source, H_batch) added to the objective): `source` holds ms source-domain rows (the
// replay rows, D wide), x / y the target batch. loss_out = rank loss + beta * MMD^2. beta == 0 skips the
// term bit-exactly (gradients()).
MOSES_API int moses_gradients_mmd(moses_model_t m, const double* x, const double* y, int64_t n, int32_t D,
                                  const double* source, int64_t ms, double beta, double sigma, double* loss_out) {
  return guarded([&] {
    require_model(m);
    if (D != m->dims[0]) fail(MOSES_ERR_DIM_MISMATCH, "feature width != model input width");
    if (!(sigma > 0.0)) fail(MOSES_ERR_INVALID_ARG, "sigma must be positive");
    const bool on = beta != 0.0 && n > 0;
    if (on && (ms <= 0 || source == nullptr)) fail(MOSES_ERR_ADVERSARY_DISABLED, "MMD needs source rows");
    const long long mrep = on ? ms : 0;
    check_rows(m, mrep + n);
    if (on) upload_rows(m, source, ms, 0);
    upload_rows(m, x, n, mrep);
    upload_f32(m, y, n, m->labels);
    const MmdTerm mt{mrep, beta, sigma};
    gradients_core(m, m->act[0], m->ld[0], m->labels, n, nullptr, 0.0, nullptr, nullptr, on ? &mt : nullptr);
    if (loss_out) MOSES_CUDA(cudaMemcpyAsync(loss_out, m->dscal, sizeof(double), cudaMemcpyDeviceToHost, m->st));
    MOSES_CUDA(cudaStreamSynchronize(m->st));
  });
}

// MMD^2 and its gradient w.r.t. every source and target row (host float64 rows; device fp32 math).
MOSES_API int moses_mmd2_grad(const double* xs, int64_t m, const double* xt, int64_t n, int32_t width, double sigma,
                              double* value, double* grad_s, double* grad_t) {
  return guarded([&] {
    if (m <= 0 || n <= 0 || width <= 0) fail(MOSES_ERR_SHAPE_MISMATCH, "empty MMD input");
    if (!(sigma > 0.0)) fail(MOSES_ERR_INVALID_ARG, "sigma must be positive");
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    const long long R = m + n;
    const size_t bytes = sizeof(double) * R * width + sizeof(float) * R * width * 2 + sizeof(double) * (R + 2) + 4096;
    Carver cv{static_cast<uint8_t*>(sc.ensure(bytes))};
    double* h64 = cv.take<double>(size_t(R) * width);
    float* h = cv.take<float>(size_t(R) * width);
    float* g = cv.take<float>(size_t(R) * width);
    double* vp = cv.take<double>(size_t(R));
    double* val = cv.take<double>(2);
    MOSES_CUDA(cudaMemcpyAsync(h64, xs, sizeof(double) * m * width, cudaMemcpyHostToDevice, sc.st));
    MOSES_CUDA(cudaMemcpyAsync(h64 + m * width, xt, sizeof(double) * n * width, cudaMemcpyHostToDevice, sc.st));
    f64_to_f32(h64, R * width, h, sc.st);
    mmd_grad<float>(h, nullptr, width, R, m, width, float(sigma), g, vp, val, 1.0, false, sc.st);
    note_launch(3);
    f32_to_f64(g, R * width, h64, sc.st);
    MOSES_CUDA(cudaMemcpyAsync(value, val, sizeof(double), cudaMemcpyDeviceToHost, sc.st));
    if (grad_s) MOSES_CUDA(cudaMemcpyAsync(grad_s, h64, sizeof(double) * m * width, cudaMemcpyDeviceToHost, sc.st));
    if (grad_t)
      MOSES_CUDA(cudaMemcpyAsync(grad_t, h64 + m * width, sizeof(double) * n * width, cudaMemcpyDeviceToHost, sc.st));
    MOSES_CUDA(cudaStreamSynchronize(sc.st));
  });
}

MOSES_API int moses_mmd2_device(const float* xs, int64_t m, const float* xt, int64_t n, int32_t width, int64_t ld,
                                double sigma, double* out) {
  return guarded([&] {
    if (m <= 0 || n <= 0) fail(MOSES_ERR_INVALID_ARG, "mmd needs non-empty source and target");
    if (width <= 0 || ld < width) fail(MOSES_ERR_INVALID_ARG, "mmd needs 0 < width <= ld");
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    void* ws = sc.ensure(mmd_ws_bytes(m, n, width) + 4096);
    int launched = 0;
    {
      ProfScope ps(P_OTHER, sc.st);
      *out = mmd2_tc(xs, m, xt, n, width, ld, float(sigma), ws, sc.st, &launched);
    }
    note_launch(launched);
  });
}

MOSES_API int moses_encode_configs_device(const double* task4, const int64_t* domains, const int32_t* domain_sizes,
                                         const int32_t* roles, int32_t n_knobs, uint64_t first, int64_t n,
                                         int32_t dtype, void* feat_dev, int64_t ld, int32_t D, uint64_t* hash_dev,
                                         int64_t* values_dev) {
  return guarded([&] {
    if (dtype != MOSES_DTYPE_F32 && dtype != MOSES_DTYPE_BF16 && dtype != MOSES_DTYPE_F64)
      fail(MOSES_ERR_INVALID_ARG, "unknown dtype");
    note_launch(encode_configs(task4, reinterpret_cast<const long long*>(domains), domain_sizes, roles, n_knobs, first,
                               n, dtype, feat_dev, ld, D, reinterpret_cast<unsigned long long*>(hash_dev),
                               reinterpret_cast<long long*>(values_dev), nullptr));
  });
}

MOSES_API int moses_encode_configs(const double* task4, const int64_t* domains, const int32_t* domain_sizes,
                                  const int32_t* roles, int32_t n_knobs, uint64_t first, int64_t n,
                                  double* features_out, uint64_t* hashes_out) {
  return guarded([&] {
    if (n < 0) fail(MOSES_ERR_INVALID_ARG, "negative count");
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    Carver cv{static_cast<uint8_t*>(sc.ensure(size_t(n) * (16 * 8 + 8) + 4096))};
    double* f = cv.take<double>(std::max<int64_t>(n, 1) * 16);
    unsigned long long* h = cv.take<unsigned long long>(std::max<int64_t>(n, 1));
    note_launch(encode_configs(task4, reinterpret_cast<const long long*>(domains), domain_sizes, roles, n_knobs, first,
                               n, MOSES_DTYPE_F64, features_out ? f : nullptr, 16, 16, hashes_out ? h : nullptr,
                               nullptr, sc.st));
    if (features_out && n)
      MOSES_CUDA(cudaMemcpyAsync(features_out, f, sizeof(double) * n * 16, cudaMemcpyDeviceToHost, sc.st));
    if (hashes_out && n) MOSES_CUDA(cudaMemcpyAsync(hashes_out, h, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, sc.st));
    MOSES_CUDA(cudaStreamSynchronize(sc.st));
  });
}

MOSES_API int moses_measure_configs_device(const double* device6, int32_t repeats, const char* device_id,
                                          const char* task_id, const double* task4, const int64_t* domains,
                                          const int32_t* domain_sizes, const int32_t* roles, int32_t n_knobs,
                                          uint64_t seed, uint64_t first, int64_t n, double* clean_ms_dev,
                                          double* throughput_dev, double* latency_dev, double* wall_cost_dev,
                                          float* label_dev) {
  return guarded([&] {
    note_launch(measure_configs(device6, repeats, device_id, task_id, task4,
                                reinterpret_cast<const long long*>(domains), domain_sizes, roles, n_knobs, seed, first,
                                n, clean_ms_dev, throughput_dev, latency_dev, wall_cost_dev, label_dev, nullptr));
  });
}

MOSES_API int moses_true_best(const double* device6, const double* task4, const int64_t* domains,
                              const int32_t* domain_sizes, const int32_t* roles, int32_t n_knobs,
                              int64_t* best_values, double* best_latency) {
  return guarded([&] {
    Scratch& sc = scratch();
    std::lock_guard<std::mutex> lk(sc.mu);
    sc.ensure(64);
    note_launch(true_best(device6, task4, reinterpret_cast<const long long*>(domains), domain_sizes, roles, n_knobs,
                          reinterpret_cast<long long*>(best_values), best_latency, sc.st));
  });
}

// ---------------------------------------------------------------- training-data pipeline
static int out_kind_of(int32_t dtype) {
  if (dtype != MOSES_DTYPE_F32 && dtype != MOSES_DTYPE_BF16 && dtype != MOSES_DTYPE_F64)
    fail(MOSES_ERR_INVALID_ARG, "unknown dtype");
  return dtype;
}
MOSES_API int moses_generate_dataset_device(const double* device6, int32_t repeats, const char* device_id,
                                           const char* task_id, const double* task4, const int64_t* domains,
                                           const int32_t* domain_sizes, const int32_t* roles, int32_t n_knobs,
                                           int64_t samples, uint64_t seed, int32_t dtype, void* feat_dev, int64_t ld,
                                           int32_t D, int64_t* values_dev, double* throughput_dev,
                                           double* latency_dev, double* wall_cost_dev, float* label_dev) {
  return guarded([&] {
    const int ok = out_kind_of(dtype);
    note_launch(generate_task_dataset(device6, repeats, device_id, task_id, task4,
                                      reinterpret_cast<const long long*>(domains), domain_sizes, roles, n_knobs, samples,
                                      seed, ok, feat_dev, ld, D, reinterpret_cast<long long*>(values_dev),
                                      throughput_dev, latency_dev, wall_cost_dev, label_dev, nullptr, nullptr));
  });
}
MOSES_API int moses_encode_values_device(const double* task4, const int64_t* domains, const int32_t* domain_sizes,
                                        const int32_t* roles, int32_t n_knobs, const int64_t* values_dev, int64_t n,
                                        int32_t dtype, void* feat_dev, int64_t ld, int32_t D, uint64_t* hash_dev,
                                        int64_t* bad_row) {
  long long bad = -1;
  const int rc = guarded([&] {
    const int ok = out_kind_of(dtype);
    if (feat_dev != nullptr && (D < 10 || ld < D)) fail(MOSES_ERR_INVALID_ARG, "feature rows need D >= 10 and ld >= D");
    note_launch(encode_values(task4, reinterpret_cast<const long long*>(domains), domain_sizes, roles, n_knobs,
                              reinterpret_cast<const long long*>(values_dev), n, ok, feat_dev, ld, D,
                              reinterpret_cast<unsigned long long*>(hash_dev), nullptr, &bad, nullptr));
  });
  if (bad_row) *bad_row = bad;
  return rc;
}
MOSES_API uint64_t moses_epoch_seed(uint64_t seed, uint64_t epoch) { return epoch_seed(seed, epoch); }
MOSES_API int moses_ranking_plan(const int32_t* record_task, int64_t n_records, const char* const* task_ids,
                                int32_t n_task_ids, int32_t batch_size, uint64_t seed, int64_t* rows_out,
                                int64_t* batch_off, int32_t* batch_task, int64_t* n_batches, int64_t* dropped) {
  return guarded([&] {
    long long drop = 0;
    const long long nb = ranking_plan(record_task, n_records, task_ids, n_task_ids, batch_size, seed,
                                      reinterpret_cast<long long*>(rows_out), reinterpret_cast<long long*>(batch_off),
                                      batch_task, &drop);
    if (n_batches) *n_batches = nb;
    if (dropped) *dropped = drop;
  });
}
MOSES_API int moses_replay_rows(int64_t n_records, int64_t size, uint64_t seed, int64_t* rows_out, int64_t* n_out) {
  return guarded([&] {
    const long long k = replay_rows(n_records, size, seed, reinterpret_cast<long long*>(rows_out));
    if (n_out) *n_out = k;
  });
}

namespace {
// ---- epochs over ranking-batch plans (moses_train_plan_device, moses_pretrain_device)
struct PlanShape {
  long long B = 0, nfull = 0, total = 0;
};
PlanShape plan_check(moses_model* m, const long long* rows, const long long* off, long long nb, long long n_records) {
  PlanShape ps;
  if (nb < 0) fail(MOSES_ERR_INVALID_ARG, "negative batch count");
  if (nb == 0) return ps;
  if (rows == nullptr || off == nullptr) fail(MOSES_ERR_INVALID_ARG, "null plan");
  if (off[0] != 0) fail(MOSES_ERR_INVALID_ARG, "batch_off[0] must be 0");
  for (long long b = 0; b < nb; ++b) {
    const long long len = off[b + 1] - off[b];
    if (len < 2) fail(MOSES_ERR_INVALID_ARG, "plan batch " + std::to_string(b) + " has fewer than 2 rows");
    ps.B = std::max(ps.B, len);
  }
  check_rows(m, ps.B);
  for (long long b = 0; b < nb; ++b) ps.nfull += (off[b + 1] - off[b]) == ps.B;
  ps.total = off[nb];
  for (long long i = 0; i < ps.total; ++i)
    if (rows[i] < 0 || rows[i] >= n_records)
      fail(MOSES_ERR_SHAPE_MISMATCH, "plan row " + std::to_string(rows[i]) + " outside the dataset");
  return ps;
}
void plan_reserve(moses_model* m, long long total, long long nb) {
  auto& ps = m->plan;
  if (total > ps.cap_rows || nb + 1 > ps.cap_b) {
    if (ps.exec) {
      cudaGraphExecDestroy(ps.exec);
      ps.exec = nullptr;
    }
    MOSES_CUDA(cudaStreamSynchronize(m->st));
    if (total > ps.cap_rows) {
      dfree(ps.rows);
      ps.rows = dalloc<long long>(total);
      ps.cap_rows = total;
    }
    if (nb + 1 > ps.cap_b) {
      dfree(ps.off);
      ps.off = dalloc<long long>(nb + 1);
      ps.cap_b = nb + 1;
    }
  }
  if (!ps.counter) ps.counter = dalloc<long long>(1);
  if (!ps.loss_sum) ps.loss_sum = dalloc<double>(1);
  if (m->split && !m->bsplit() && !ps.stage) ps.stage = dalloc<float>(m->cap * m->ld[0]);
}
// one step over plan batch *counter (n rows): gather -> gradients -> momentum update -> loss sum
void plan_step(moses_model* m, const void* x, long long ldx, const float* y, long long n, float lr, float mu) {
  auto& ps = m->plan;
  const long long row_bytes = ldx * m->in_esz();
  if (m->split && !m->bsplit()) {  // 3xTF32 operands: hi/lo split of the gathered fp32 rows
    gather_plan(x, row_bytes, y, ps.rows, ps.off, ps.counter, n, ps.stage, m->labels, m->st);
    pack_rows_f32<float>(ps.stage, n, m->dims[0], ldx, static_cast<float*>(m->act[0]), m->ld[0], m->st,
                         m->act_lo_t<float>(0));
    note_launch(1);
  } else {  // split-bf16 handles split the gathered fp32 rows into their hi/lo planes in the gather
    gather_plan(x, row_bytes, y, ps.rows, ps.off, ps.counter, n, m->act[0], m->labels, m->st, m->act_lo(0));
  }
  const SgdFuse fz{lr, mu, ps.counter, m->dscal, ps.loss_sum};
  if (!gradients_core(m, m->act[0], m->ld[0], m->labels, n, nullptr, 0.0, nullptr, &fz)) {
    sgd_update(m->w, m->mom, m->g, nullptr, m->P, lr, mu, true, m->shadow(), m->st);
    m->post_update();
    note_launch(1);
  }
  if (!fz.folded) {
    accum_f64(m->dscal, ps.loss_sum, m->st);
    advance_counter(ps.counter, m->st);
    note_launch(2);
  }
  note_launch(1);
}
// full-size batches replay one CUDA graph, captured once per dataset / size / hyper-parameters;
// needs the plan's rows on the device (the warm-up gathers batch 0's slots)
bool plan_graph(moses_model* m, const void* x, long long ldx, const float* y, const PlanShape& sh, float lr, float mu) {
  auto& ps = m->plan;
  if ((m->split && !m->bsplit()) || sh.nfull < 4) return false;
  if (ps.exec && ps.x == x && ps.y == y && ps.ldx == ldx && ps.batch == sh.B && ps.lr == lr && ps.mu == mu) return true;
  if (ps.exec) {
    cudaGraphExecDestroy(ps.exec);
    ps.exec = nullptr;
  }
  // eager warm-up without the update (configures kernels; parameters untouched)
  MOSES_CUDA(cudaMemsetAsync(ps.counter, 0, sizeof(long long), m->st));
  gather_plan(x, ldx * m->in_esz(), y, ps.rows, ps.off, ps.counter, sh.B, m->act[0], m->labels, m->st, m->act_lo(0));
  gradients_core(m, m->act[0], m->ld[0], m->labels, sh.B, nullptr, 0.0);
  MOSES_CUDA(cudaStreamSynchronize(m->st));
  const long long before = moses_kernel_launches();
  cudaGraph_t graph;
  MOSES_CUDA(cudaStreamBeginCapture(m->st, cudaStreamCaptureModeThreadLocal));
  try {
    plan_step(m, x, ldx, y, sh.B, lr, mu);
  } catch (...) {
    cudaStreamEndCapture(m->st, &graph);
    throw;
  }
  MOSES_CUDA(cudaStreamEndCapture(m->st, &graph));
  ps.graph_kernels = moses_kernel_launches() - before;
  note_launch(-ps.graph_kernels);  // captured, not launched
  MOSES_CUDA(cudaGraphInstantiate(&ps.exec, graph, 0));
  MOSES_CUDA(cudaGraphDestroy(graph));
  ps.x = x;
  ps.y = y;
  ps.ldx = ldx;
  ps.batch = sh.B;
  ps.lr = lr;
  ps.mu = mu;
  return true;
}
// enqueue one epoch (rows / offsets already on the device); the loss sum is left in ps.loss_sum
void plan_epoch(moses_model* m, const void* x, long long ldx, const float* y, const long long* off, long long nb,
                const PlanShape& sh, float lr, float mu, bool graph) {
  auto& ps = m->plan;
  MOSES_CUDA(cudaMemsetAsync(ps.counter, 0, sizeof(long long), m->st));
  MOSES_CUDA(cudaMemsetAsync(ps.loss_sum, 0, sizeof(double), m->st));
  for (long long b = 0; b < nb; ++b) {
    const long long len = off[b + 1] - off[b];
    if (graph && len == sh.B) {
      MOSES_CUDA(cudaGraphLaunch(ps.exec, m->st));
      note_launch(ps.graph_kernels);
    } else {
      plan_step(m, x, ldx, y, len, lr, mu);
    }
  }
}
}  // namespace

MOSES_API int moses_train_plan_device(moses_model_t m, const void* x_base, int64_t ldx, const float* y_base,
                                     int64_t n_records, const int64_t* rows, const int64_t* batch_off,
                                     int64_t n_batches, double lr, double mu, double* mean_loss) {
  return guarded([&] {
    require_model(m);
    if (ldx != m->ld[0]) fail(MOSES_ERR_INVALID_ARG, "dataset row stride must equal moses_packed_ld");
    const auto* r = reinterpret_cast<const long long*>(rows);
    const auto* off = reinterpret_cast<const long long*>(batch_off);
    const PlanShape sh = plan_check(m, r, off, n_batches, n_records);
    if (n_batches == 0) {
      if (mean_loss) *mean_loss = 0.0;  // tuner.cpp:152-154: empty epoch
      return;
    }
    if (x_base == nullptr || y_base == nullptr) fail(MOSES_ERR_INVALID_ARG, "null dataset");
    plan_reserve(m, sh.total, n_batches);
    auto& ps = m->plan;
    MOSES_CUDA(cudaMemcpyAsync(ps.rows, r, sizeof(long long) * sh.total, cudaMemcpyHostToDevice, m->st));
    MOSES_CUDA(cudaMemcpyAsync(ps.off, off, sizeof(long long) * (n_batches + 1), cudaMemcpyHostToDevice, m->st));
    const bool graph = plan_graph(m, x_base, ldx, y_base, sh, float(lr), float(mu));
    plan_epoch(m, x_base, ldx, y_base, off, n_batches, sh, float(lr), float(mu), graph);
    if (mean_loss) {
      double sum = 0.0;
      MOSES_CUDA(cudaMemcpyAsync(&sum, ps.loss_sum, sizeof(double), cudaMemcpyDeviceToHost, m->st));
      MOSES_CUDA(cudaStreamSynchronize(m->st));
      *mean_loss = sum / double(n_batches);
    }
  });
}

// pretrain (tuner.cpp:130-156) over a device-resident dataset: per epoch KeyBuilder(seed, "epoch", e)
// -> make_ranking_batches -> one step per batch. The host computes epoch e+1's plan (into pinned
// memory) while the device runs epoch e; plan uploads and per-epoch loss sums are stream-ordered,
// so the only synchronisation is the final read of the per-epoch losses.
static void pretrain_impl(moses_model* m, const void* x_base, int64_t ldx, const float* y_base,
                          const int32_t* record_task, int64_t n_records, const char* const* task_ids,
                          int32_t n_task_ids, int32_t batch_size, uint64_t seed, int32_t epochs, double lr, double mu,
                          double* epoch_mean_loss, int64_t* dropped_singletons) {
  {
    require_model(m);
    if (n_records <= 0) fail(MOSES_ERR_EMPTY_DATASET, "no records to pretrain on");
    if (ldx != m->ld[0]) fail(MOSES_ERR_INVALID_ARG, "dataset row stride must equal moses_packed_ld");
    if (x_base == nullptr || y_base == nullptr) fail(MOSES_ERR_INVALID_ARG, "null dataset");
    if (epochs < 0) fail(MOSES_ERR_INVALID_CONFIG, "negative epoch count");
    if (epochs == 0) return;
    struct Slot {
      long long* rows = nullptr;  // pinned
      long long* off = nullptr;   // pinned
      long long nb = 0;
      cudaEvent_t up = nullptr;
    } slot[2];
    double* losses = nullptr;
    auto cleanup = [&] {
      cudaStreamSynchronize(m->st);
      for (auto& s : slot) {
        if (s.rows) cudaFreeHost(s.rows);
        if (s.off) cudaFreeHost(s.off);
        if (s.up) cudaEventDestroy(s.up);
      }
      dfree(losses);
    };
    std::vector<long long> nbs(size_t(epochs), 0);
    long long drop0 = 0;
    try {
      for (auto& s : slot) {
        MOSES_CUDA(cudaMallocHost(reinterpret_cast<void**>(&s.rows), sizeof(long long) * n_records));
        MOSES_CUDA(cudaMallocHost(reinterpret_cast<void**>(&s.off), sizeof(long long) * (n_records / 2 + 2)));
        MOSES_CUDA(cudaEventCreateWithFlags(&s.up, cudaEventDisableTiming));
      }
      losses = dalloc<double>(size_t(epochs));
      auto make_plan = [&](int e) {
        Slot& s = slot[e & 1];
        MOSES_CUDA(cudaEventSynchronize(s.up));  // the upload two epochs back has read this slot
        long long drop = 0;
        s.nb = ranking_plan(record_task, n_records, task_ids, n_task_ids, batch_size, epoch_seed(seed, uint64_t(e)),
                            s.rows, s.off, nullptr, &drop);
        if (e == 0) drop0 = drop;
      };
      make_plan(0);
      plan_reserve(m, n_records, n_records / 2 + 1);
      auto& ps = m->plan;
      for (int e = 0; e < epochs; ++e) {
        Slot& s = slot[e & 1];
        const PlanShape sh = plan_check(m, s.rows, s.off, s.nb, n_records);
        nbs[size_t(e)] = s.nb;
        if (s.nb > 0) {
          MOSES_CUDA(cudaMemcpyAsync(ps.rows, s.rows, sizeof(long long) * sh.total, cudaMemcpyHostToDevice, m->st));
          MOSES_CUDA(cudaMemcpyAsync(ps.off, s.off, sizeof(long long) * (s.nb + 1), cudaMemcpyHostToDevice, m->st));
          MOSES_CUDA(cudaEventRecord(s.up, m->st));
          const bool graph = plan_graph(m, x_base, ldx, y_base, sh, float(lr), float(mu));
          plan_epoch(m, x_base, ldx, y_base, s.off, s.nb, sh, float(lr), float(mu), graph);
          MOSES_CUDA(cudaMemcpyAsync(losses + e, ps.loss_sum, sizeof(double), cudaMemcpyDeviceToDevice, m->st));
        } else {
          MOSES_CUDA(cudaMemsetAsync(losses + e, 0, sizeof(double), m->st));
        }
        if (e + 1 < epochs) make_plan(e + 1);  // overlaps the epoch just enqueued
      }
      std::vector<double> h(static_cast<size_t>(epochs));
      MOSES_CUDA(cudaMemcpyAsync(h.data(), losses, sizeof(double) * epochs, cudaMemcpyDeviceToHost, m->st));
      MOSES_CUDA(cudaStreamSynchronize(m->st));
      if (epoch_mean_loss)
        for (int e = 0; e < epochs; ++e) epoch_mean_loss[e] = nbs[size_t(e)] ? h[size_t(e)] / double(nbs[size_t(e)]) : 0.0;
      if (dropped_singletons) *dropped_singletons = drop0;
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  }
}

MOSES_API int moses_pretrain_device(moses_model_t m, const void* x_base, int64_t ldx, const float* y_base,
                                   const int32_t* record_task, int64_t n_records, const char* const* task_ids,
                                   int32_t n_task_ids, int32_t batch_size, uint64_t seed, int32_t epochs, double lr,
                                   double mu, double* epoch_mean_loss, int64_t* dropped_singletons) {
  return guarded([&] {
    pretrain_impl(m, x_base, ldx, y_base, record_task, n_records, task_ids, n_task_ids, batch_size, seed, epochs, lr,
                  mu, epoch_mean_loss, dropped_singletons);
  });
}

// pretrain(store, tasks, hyper) (tuner.cpp:130-156) from host records: the store is staged on the
// device grouped by task (first-appearance order, store order within a task — the per-task row
// lists make_ranking_batches shuffles are unchanged, so every batch holds the same records), each
// task's rows are validated and encoded on the device (encode_features, one shared knob template),
// labels are the measured throughputs, then the epoch loop runs on the handle.
MOSES_API int moses_pretrain(moses_model_t m, int32_t n_tasks, const char* const* task_ids, const double* task4,
                            const int64_t* domains, const int32_t* domain_sizes, const int32_t* roles,
                            int32_t n_knobs, const int32_t* record_task, const int64_t* values,
                            const double* throughput, int64_t n_records, int32_t batch_size, uint64_t seed,
                            int32_t epochs, double lr, double mu, double* epoch_mean_loss,
                            int64_t* dropped_singletons) {
  return guarded([&] {
    require_model(m);
    if (n_records <= 0) fail(MOSES_ERR_EMPTY_DATASET, "no records to pretrain on");
    if (m->dims[0] < 10) fail(MOSES_ERR_DIM_MISMATCH, "model input width below the 10 live feature entries");
    if (n_tasks <= 0 || task_ids == nullptr || task4 == nullptr || record_task == nullptr || values == nullptr ||
        throughput == nullptr)
      fail(MOSES_ERR_INVALID_ARG, "null store or task table");
    // group by task: first-appearance order, store order within a task
    std::vector<int> order;
    std::vector<std::vector<long long>> rows(static_cast<size_t>(n_tasks));
    for (long long i = 0; i < n_records; ++i) {
      const int t = record_task[i];
      if (t < 0 || t >= n_tasks) fail(MOSES_ERR_INVALID_TASK, "record " + std::to_string(i) + ": unknown task id");
      if (rows[t].empty()) order.push_back(t);
      rows[t].push_back(i);
    }
    std::vector<long long> vals_g(size_t(n_records) * n_knobs);
    std::vector<float> lab_g(static_cast<size_t>(n_records));
    std::vector<int32_t> task_g(static_cast<size_t>(n_records));
    std::vector<long long> first(size_t(n_tasks) + 1, 0);
    long long pos = 0;
    for (int t : order) {
      first[t] = pos;
      for (long long i : rows[t]) {
        std::copy(values + i * n_knobs, values + (i + 1) * n_knobs, vals_g.begin() + pos * n_knobs);
        lab_g[size_t(pos)] = float(throughput[i]);
        task_g[size_t(pos)] = t;
        ++pos;
      }
    }
    const long long ld = m->ld[0];
    void* X = nullptr;
    long long* V = nullptr;
    float* Y = nullptr;
    auto release = [&] {
      cudaStreamSynchronize(m->st);
      dfree(X);
      dfree(V);
      dfree(Y);
    };
    try {
      X = dalloc<uint8_t>(size_t(n_records) * ld * m->in_esz());
      V = dalloc<long long>(size_t(n_records) * n_knobs);
      Y = dalloc<float>(size_t(n_records));
      MOSES_CUDA(cudaMemcpyAsync(V, vals_g.data(), sizeof(long long) * vals_g.size(), cudaMemcpyHostToDevice, m->st));
      MOSES_CUDA(cudaMemcpyAsync(Y, lab_g.data(), sizeof(float) * lab_g.size(), cudaMemcpyHostToDevice, m->st));
      MOSES_CUDA(cudaMemsetAsync(X, 0, size_t(n_records) * ld * m->in_esz(), m->st));
      const int kind = m->in_esz() == 2 ? MOSES_DTYPE_BF16 : MOSES_DTYPE_F32;
      for (int t : order) {
        long long bad = -1;
        const long long cnt = (long long)rows[t].size();
        try {
          note_launch(encode_values(task4 + 4 * t, reinterpret_cast<const long long*>(domains), domain_sizes, roles,
                                    n_knobs, V + first[t] * n_knobs, cnt, kind,
                                    static_cast<uint8_t*>(X) + first[t] * ld * m->in_esz(), ld, m->dims[0], nullptr,
                                    nullptr, &bad, m->st));
        } catch (const Status& e) {
          if (bad >= 0)  // report the caller's record index
            fail(e.code, "record " + std::to_string(rows[t][size_t(bad)]) + " (task " + task_ids[t] +
                             "): value not in its knob's domain");
          throw;
        }
      }
      pretrain_impl(m, X, ld, Y, task_g.data(), n_records, task_ids, n_tasks, batch_size, seed, epochs, lr, mu,
                    epoch_mean_loss, dropped_singletons);
    } catch (...) {
      release();
      throw;
    }
    release();
  });
}

// Job pool over independent pretrain runs (the reference's (strategy, seed) pool, tuner.cpp:57-69,
// 331-374): jobs are claimed in order by `threads` workers (0: MOSES_LAB_THREADS or the hardware
// concurrency, capped at the job count); every job owns its model handle and therefore its CUDA
// streams, so the GPU runs the jobs' small, latency-bound steps concurrently. The first failing
// job's status is returned; the others still run to completion or to their own error.
static void pretrain_jobs_impl(int32_t n_jobs, const moses_model_t* models, const uint64_t* seeds,
                               const void* const* x_of, int64_t ldx, const float* const* y_of,
                               const int32_t* record_task, int64_t n_records, const char* const* task_ids,
                               int32_t n_task_ids, int32_t batch_size, int32_t epochs, double lr, double mu,
                               int32_t threads, double* epoch_mean_loss, int64_t* dropped_singletons) {
  {
    if (n_jobs < 0 || (n_jobs > 0 && (models == nullptr || seeds == nullptr)))
      fail(MOSES_ERR_INVALID_ARG, "invalid job list");
    if (n_jobs == 0) return;
    int width = threads;
    if (width <= 0) {
      width = int(std::thread::hardware_concurrency());
      if (const char* env = std::getenv("MOSES_LAB_THREADS"); env != nullptr && *env != '\0') {
        char* end = nullptr;
        const long v = std::strtol(env, &end, 10);
        if (end == env || *end != '\0' || v < 0)
          fail(MOSES_ERR_INVALID_CONFIG, std::string("bad MOSES_LAB_THREADS value '") + env + "'");
        if (v > 0) width = int(v);
      }
    }
    width = std::max(1, std::min(width, n_jobs));
    for (int j = 0; j < n_jobs; ++j) {
      if (models[j] == nullptr) fail(MOSES_ERR_INVALID_ARG, "null model handle in the job list");
      for (int i = 0; i < j; ++i)
        if (models[i] == models[j])
          fail(MOSES_ERR_INVALID_ARG, "model handle listed twice in the job list (jobs " + std::to_string(i) + ", " +
                                          std::to_string(j) + "): a handle must not be used concurrently");
    }
    std::atomic<int> next{0};
    std::mutex mu_err;
    int first_job = -1, first_code = 0;
    std::string first_msg;
    auto worker = [&] {
      for (;;) {
        const int j = next.fetch_add(1);
        if (j >= n_jobs) return;
        try {
          // new threads start on device 0: every job runs on its handle's device
          MOSES_CUDA(cudaSetDevice(models[j]->device));
          pretrain_impl(models[j], x_of[j], ldx, y_of[j], record_task, n_records, task_ids, n_task_ids, batch_size,
                        seeds[j], epochs, lr, mu, epoch_mean_loss ? epoch_mean_loss + size_t(j) * epochs : nullptr,
                        dropped_singletons ? dropped_singletons + j : nullptr);
        } catch (const Status& e) {
          std::lock_guard<std::mutex> lk(mu_err);
          if (first_job < 0 || j < first_job) {
            first_job = j;
            first_code = e.code;
            first_msg = e.what();
          }
        } catch (const std::exception& e) {
          std::lock_guard<std::mutex> lk(mu_err);
          if (first_job < 0 || j < first_job) {
            first_job = j;
            first_code = MOSES_ERR_INVALID_ARG;
            first_msg = e.what();
          }
        }
      }
    };
    if (width == 1) {
      worker();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < width; ++t) pool.emplace_back(worker);
      for (auto& t : pool) t.join();
    }
    if (first_job >= 0) fail(first_code, "job " + std::to_string(first_job) + ": " + first_msg);
  }
}

MOSES_API int moses_pretrain_jobs(int32_t n_jobs, const moses_model_t* models, const uint64_t* seeds,
                                 const void* x_base, int64_t ldx, const float* y_base, const int32_t* record_task,
                                 int64_t n_records, const char* const* task_ids, int32_t n_task_ids,
                                 int32_t batch_size, int32_t epochs, double lr, double mu, int32_t threads,
                                 double* epoch_mean_loss, int64_t* dropped_singletons) {
  return guarded([&] {
    const std::vector<const void*> xs(size_t(std::max(n_jobs, 0)), x_base);
    const std::vector<const float*> ys(size_t(std::max(n_jobs, 0)), y_base);
    pretrain_jobs_impl(n_jobs, models, seeds, xs.data(), ldx, ys.data(), record_task, n_records, task_ids, n_task_ids,
                       batch_size, epochs, lr, mu, threads, epoch_mean_loss, dropped_singletons);
  });
}

// The job grid across GPUs (tuner.cpp:331-374): job j runs on its handle's device
// with that device's copy of the store (x_of[j], y_of[j]); handles created round-robin on the GPUs of
// the process map the (strategy, seed) grid onto all of them.
MOSES_API int moses_pretrain_jobs_mapped(int32_t n_jobs, const moses_model_t* models, const uint64_t* seeds,
                                        const void* const* x_of, int64_t ldx, const float* const* y_of,
                                        const int32_t* record_task, int64_t n_records, const char* const* task_ids,
                                        int32_t n_task_ids, int32_t batch_size, int32_t epochs, double lr, double mu,
                                        int32_t threads, double* epoch_mean_loss, int64_t* dropped_singletons) {
  return guarded([&] {
    if (n_jobs > 0 && (x_of == nullptr || y_of == nullptr)) fail(MOSES_ERR_INVALID_ARG, "null per-job dataset list");
    for (int32_t j = 0; j < n_jobs; ++j) {
      if (models == nullptr || models[j] == nullptr) fail(MOSES_ERR_INVALID_ARG, "null model handle in the job list");
      cudaPointerAttributes pa{};
      if (cudaPointerGetAttributes(&pa, x_of[j]) == cudaSuccess && pa.type == cudaMemoryTypeDevice &&
          pa.device != models[j]->device)
        fail(MOSES_ERR_INVALID_ARG, "job " + std::to_string(j) + ": dataset and model on different devices");
    }
    pretrain_jobs_impl(n_jobs, models, seeds, x_of, ldx, y_of, record_task, n_records, task_ids, n_task_ids,
                       batch_size, epochs, lr, mu, threads, epoch_mean_loss, dropped_singletons);
  });
}

struct moses_records : moses::Records {};
MOSES_API int moses_records_create(moses_records_t* out) {
  return guarded([&] {
    if (!out) fail(MOSES_ERR_INVALID_ARG, "null output");
    *out = new moses_records();
  });
}
MOSES_API int moses_records_read(const char* path, moses_records_t* out) {
  return guarded([&] {
    if (!out) fail(MOSES_ERR_INVALID_ARG, "null output");
    *out = nullptr;
    std::unique_ptr<Records> r(Records::read(path));
    auto* h = new moses_records();
    static_cast<Records&>(*h) = std::move(*r);
    *out = h;
  });
}
MOSES_API void moses_records_destroy(moses_records_t r) { delete r; }
MOSES_API int moses_records_append(moses_records_t r, const char* task_id, const char* device_id, int64_t n,
                                  int32_t n_values, const int64_t* values, const double* thr, const double* lat,
                                  const double* wall, const uint64_t* seq) {
  return guarded([&] {
    if (!r || !task_id || !device_id || n < 0 || n_values < 0 || (n > 0 && (!thr || !lat || !wall || !seq)) ||
        (n > 0 && n_values > 0 && !values))
      fail(MOSES_ERR_INVALID_ARG, "invalid record batch");
    auto intern = [](std::vector<std::string>& tab, std::map<std::string, int>& ix, const std::string& s) {
      auto it = ix.find(s);
      if (it != ix.end()) return it->second;
      tab.push_back(s);
      ix.emplace(s, int(tab.size()) - 1);
      return int(tab.size()) - 1;
    };
    if (n == 0) return;
    const int t = intern(r->task_ids, r->task_ix, task_id), d = intern(r->device_ids, r->device_ix, device_id);
    for (int64_t i = 0; i < n; ++i) {
      r->task.push_back(t);
      r->device.push_back(d);
      r->value_off.push_back(r->value_off.back() + n_values);
      r->values.insert(r->values.end(), values + i * n_values, values + (i + 1) * n_values);
      r->throughput.push_back(thr[i]);
      r->latency.push_back(lat[i]);
      r->wall_cost.push_back(wall[i]);
      r->seq.push_back(seq[i]);
    }
  });
}
MOSES_API int moses_records_write(moses_records_t r, const char* path) {
  return guarded([&] {
    if (!r) fail(MOSES_ERR_INVALID_ARG, "null records");
    r->write(path);
  });
}
MOSES_API int moses_records_shape(moses_records_t r, int64_t* n_records, int64_t* n_values, int32_t* n_tasks,
                                 int32_t* n_devices) {
  return guarded([&] {
    if (!r) fail(MOSES_ERR_INVALID_ARG, "null records");
    if (n_records) *n_records = r->size();
    if (n_values) *n_values = (int64_t)r->values.size();
    if (n_tasks) *n_tasks = int32_t(r->task_ids.size());
    if (n_devices) *n_devices = int32_t(r->device_ids.size());
  });
}
MOSES_API const char* moses_records_task_id(moses_records_t r, int32_t t) {
  return (r && t >= 0 && t < int32_t(r->task_ids.size())) ? r->task_ids[t].c_str() : nullptr;
}
MOSES_API const char* moses_records_device_id(moses_records_t r, int32_t d) {
  return (r && d >= 0 && d < int32_t(r->device_ids.size())) ? r->device_ids[d].c_str() : nullptr;
}
MOSES_API int moses_records_export(moses_records_t r, int32_t* task_index, int32_t* device_index, int64_t* value_off,
                                  int64_t* values, double* thr, double* lat, double* wall, uint64_t* seq) {
  return guarded([&] {
    if (!r) fail(MOSES_ERR_INVALID_ARG, "null records");
    const size_t n = size_t(r->size());
    if (task_index) std::copy(r->task.begin(), r->task.end(), task_index);
    if (device_index) std::copy(r->device.begin(), r->device.end(), device_index);
    if (value_off) std::copy(r->value_off.begin(), r->value_off.end(), value_off);
    if (values) std::copy(r->values.begin(), r->values.end(), values);
    if (thr) std::copy_n(r->throughput.begin(), n, thr);
    if (lat) std::copy_n(r->latency.begin(), n, lat);
    if (wall) std::copy_n(r->wall_cost.begin(), n, wall);
    if (seq) std::copy_n(r->seq.begin(), n, seq);
  });
}
MOSES_API int moses_debug_set_rank_grid(int32_t on) {
  debug_set_rank_grid(on != 0);
  return MOSES_OK;
}
MOSES_API int moses_debug_set_rank_sym(int32_t on) {
  debug_set_rank_sym(on != 0);
  return MOSES_OK;
}
MOSES_API int moses_debug_force_serial_sampling(int32_t on) {
  debug_force_serial_sampling(on != 0);
  return MOSES_OK;
}

MOSES_API int moses_synth_features_device(uint64_t seed, int64_t row0, int64_t n, int32_t D, int32_t dtype, void* dst,
                                          int64_t ld) {
  return guarded([&] {
    if (dtype == MOSES_DTYPE_BF16) synth_features<__nv_bfloat16>(seed, row0, n, D, static_cast<__nv_bfloat16*>(dst), ld, nullptr);
    else synth_features<float>(seed, row0, n, D, static_cast<float*>(dst), ld, nullptr);
    note_launch(1);
  });
}
MOSES_API int moses_synth_labels_device(uint64_t seed, int64_t row0, int64_t n, float* dst) {
  return guarded([&] {
    synth_labels(seed, row0, n, dst, nullptr);
    note_launch(1);
  });
}

// ---------------------------------------------------------------- files (host byte formats)
static void put_u32(std::vector<uint8_t>& o, uint32_t v) { for (int i = 0; i < 4; ++i) o.push_back(uint8_t(v >> (8 * i))); }
static void put_u64(std::vector<uint8_t>& o, uint64_t v) { for (int i = 0; i < 8; ++i) o.push_back(uint8_t(v >> (8 * i))); }
static uint64_t get_u64(const uint8_t* p) { uint64_t v = 0; for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i); return v; }
static uint32_t get_u32(const uint8_t* p) { uint32_t v = 0; for (int i = 0; i < 4; ++i) v |= uint32_t(p[i]) << (8 * i); return v; }

MOSES_API int64_t moses_serialize(const int32_t* dims, int32_t nd, const double* params, const double* mom, uint8_t* out,
                                  int64_t cap) {
  std::vector<uint8_t> b;
  const int rc = guarded([&] {
    check_dims(dims, nd, true);
    if (dims[1] != 512 || dims[2] != 512) fail(MOSES_ERR_BAD_DIMS, "only the {D,512,512,1} shape has a file form");
    std::vector<int> d(dims, dims + nd);
    const long long P = level_off(d, 3);
    b.reserve(12 + 16 * P);
    b.insert(b.end(), {'M', 'O', 'S', 'M'});
    put_u32(b, 1);
    put_u32(b, uint32_t(dims[0]));
    for (long long i = 0; i < P; ++i) put_u64(b, std::bit_cast<uint64_t>(params[i]));
    for (long long i = 0; i < P; ++i) put_u64(b, std::bit_cast<uint64_t>(mom ? mom[i] : 0.0));
  });
  if (rc) return -rc;
  if (out && cap >= (int64_t)b.size()) std::memcpy(out, b.data(), b.size());
  return (int64_t)b.size();
}

MOSES_API int moses_deserialize(const uint8_t* bytes, int64_t len, int32_t* dims_out, double* params, double* mom,
                                int64_t cap) {
  return guarded([&] {
    if (len < 12 || std::memcmp(bytes, "MOSM", 4) != 0) fail(MOSES_ERR_CORRUPT_STREAM, "bad magic or truncated header");
    const uint32_t ver = get_u32(bytes + 4);
    if (ver != 1) fail(MOSES_ERR_VERSION_MISMATCH, "format version " + std::to_string(ver) + ", expected 1");
    const uint32_t D = get_u32(bytes + 8);
    if (D == 0 || D > 4096) fail(MOSES_ERR_CORRUPT_STREAM, "implausible input width");
    std::vector<int> d = {int(D), 512, 512, 1};
    const long long P = level_off(d, 3);
    if (len != 12 + 16 * P) fail(MOSES_ERR_CORRUPT_STREAM, "stream is " + std::to_string(len) + " bytes");
    for (int i = 0; i < 4; ++i) dims_out[i] = d[i];
    if (cap < P) fail(MOSES_ERR_CAPACITY, "output capacity too small");
    for (long long i = 0; i < P; ++i) {
      params[i] = std::bit_cast<double>(get_u64(bytes + 12 + 8 * i));
      const double v = std::bit_cast<double>(get_u64(bytes + 12 + 8 * (P + i)));
      if (mom) mom[i] = v;
      if (!std::isfinite(params[i]) || !std::isfinite(v)) fail(MOSES_ERR_CORRUPT_STREAM, "non-finite parameter value");
    }
  });
}

MOSES_API int64_t moses_write_mask(const uint8_t* mask, int64_t n, int32_t phase, int32_t mode, double value,
                                   uint8_t* out, int64_t cap) {
  std::vector<uint8_t> b = {'M', 'O', 'S', 'K'};
  put_u64(b, uint64_t(n));
  put_u32(b, uint32_t(phase));
  b.push_back(mode == MOSES_MODE_THRESHOLD ? 1 : 2);
  put_u64(b, std::bit_cast<uint64_t>(value));
  std::vector<uint8_t> bits((n + 7) / 8, 0);
  for (int64_t i = 0; i < n; ++i)
    if (mask[i]) bits[i / 8] |= uint8_t(1u << (i % 8));
  b.insert(b.end(), bits.begin(), bits.end());
  if (out && cap >= (int64_t)b.size()) std::memcpy(out, b.data(), b.size());
  return (int64_t)b.size();
}

MOSES_API int moses_read_mask(const uint8_t* buf, int64_t len, uint8_t* mask_out, int64_t cap, int64_t* n,
                              int32_t* phase, int32_t* mode, double* value) {
  return guarded([&] {
    if (len < 25 || std::memcmp(buf, "MOSK", 4) != 0) fail(MOSES_ERR_CORRUPT_STREAM, "bad magic or truncated header");
    const uint64_t cnt = get_u64(buf + 4);
    const uint8_t mb = buf[16];
    if (mb != 1 && mb != 2) fail(MOSES_ERR_CORRUPT_STREAM, "unknown mode byte");
    if ((uint64_t)len != 25 + (cnt + 7) / 8) fail(MOSES_ERR_CORRUPT_STREAM, "mask file size mismatch");
    *n = (int64_t)cnt;
    *phase = int32_t(get_u32(buf + 12));
    *mode = mb;
    *value = std::bit_cast<double>(get_u64(buf + 17));
    if (mask_out) {
      if (cap < (int64_t)cnt) fail(MOSES_ERR_CAPACITY, "mask capacity too small");
      for (uint64_t i = 0; i < cnt; ++i) mask_out[i] = (buf[25 + i / 8] >> (i % 8)) & 1;
    }
  });
}

MOSES_API int moses_model_device_ptrs(moses_model_t m, float** params, float** grads, float** momentum) {
  return guarded([&] {
    require_model(m);
    if (params) *params = m->w;
    if (grads) *grads = m->g;
    if (momentum) *momentum = m->mom;
  });
}
MOSES_API int moses_model_stream(moses_model_t m, void** stream) {
  return guarded([&] {
    require_model(m);
    *stream = m->st;
  });
}

}  // extern "C"

// ---------------------------------------------------------------- test hook: one raw GEMM on device buffers
extern "C" MOSES_API int moses_debug_gemm(int elem, int M, int N, int K, const void* A, long long lda, int a_mn,
                                          const void* B, long long ldb, int b_mn, int epi, void* out, long long ldo,
                                          const float* bias, int relu, int bn, const void* mask, long long ldm) {
  return guarded([&] {
    GemmCall c{};
    c.M = M;
    c.N = N;
    c.K = K;
    c.A = {A, lda, a_mn != 0};
    c.B = {B, ldb, b_mn != 0};
    c.epi = EpiKind(epi);
    c.out = out;
    c.ldo = ldo;
    c.bias = bias;
    c.relu = relu;
    c.bn = bn;
    c.mask = mask;
    c.ldm = ldm;
    launch_gemm(elem, c, nullptr);
    note_launch(1);
    MOSES_CUDA(cudaDeviceSynchronize());
  });
}

// Timing harness for kernel tuning (tools/gemm_latency.py): launches the GEMM `iters` times
// back to back on a private stream and reports the mean device time per launch.
extern "C" MOSES_API int moses_debug_gemm_timed(int elem, int M, int N, int K, const void* A, long long lda, int a_mn,
                                                const void* B, long long ldb, int b_mn, int epi, void* out,
                                                long long ldo, const float* bias, int relu, int bn, const void* mask,
                                                long long ldm, int iters, float* ms_out) {
  return guarded([&] {
    GemmCall c{};
    c.M = M;
    c.N = N;
    c.K = K;
    c.A = {A, lda, a_mn != 0};
    c.B = {B, ldb, b_mn != 0};
    c.epi = EpiKind(epi);
    c.out = out;
    c.ldo = ldo;
    c.bias = bias;
    c.relu = relu;
    c.bn = bn;
    c.mask = mask;
    c.ldm = ldm;
    cudaStream_t st;
    cudaEvent_t e0, e1;
    MOSES_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    MOSES_CUDA(cudaEventCreate(&e0));
    MOSES_CUDA(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) launch_gemm(elem, c, st);
    MOSES_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) launch_gemm(elem, c, st);
    MOSES_CUDA(cudaEventRecord(e1, st));
    MOSES_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    MOSES_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_out = ms / float(iters);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

namespace moses {
extern int g_mn_swz[2], g_mn_layout[2], g_mn_sbo[2], g_mn_kstep[2];
}
extern "C" MOSES_API int moses_debug_set_mn(int which, int swz, int layout, int sbo, int kstep) {
  moses::g_mn_swz[which] = swz;
  moses::g_mn_layout[which] = layout;
  moses::g_mn_sbo[which] = sbo;
  moses::g_mn_kstep[which] = kstep;
  return 0;
}

namespace moses {
extern int g_persistent;
}
extern "C" MOSES_API int moses_debug_set_persistent(int on) {
  moses::g_persistent = on;
  return 0;
}

namespace moses {
extern int g_cluster;
}
namespace moses {
extern unsigned long long* g_chain_trace;
}
namespace moses { void rank_trace_read(unsigned long long* out); void rank_cta_trace_read(unsigned long long* out); }
// rank_sym_kernel per-CTA stamps: 512 x {start, scores, pairs, grid sync, rows} (globaltimer ns)
extern "C" MOSES_API int moses_debug_rank_cta_trace(unsigned long long* out2560) {
  return guarded([&] { moses::rank_cta_trace_read(out2560); });
}
extern "C" MOSES_API int moses_debug_lottery_trace(unsigned long long* out8) {
  return guarded([&] { moses::lottery_res_trace_read(out8); });
}
extern "C" MOSES_API int moses_debug_topk_trace(unsigned long long* out16) {
  return guarded([&] { moses::topk_trace_read(out16); });
}
extern "C" MOSES_API int moses_debug_rank_trace(unsigned long long* out16) {
  return guarded([&] { moses::rank_trace_read(out16); });
}
extern "C" MOSES_API int moses_debug_set_rank_fused(int on) {
  moses::g_rank_fused = on;
  return 0;
}
// device buffer of 4*8*8 u64 that receives chain-kernel phase timestamps (nullptr: off)
extern "C" MOSES_API int moses_debug_set_chain_trace(void* dev_buf) {
  moses::g_chain_trace = static_cast<unsigned long long*>(dev_buf);
  return 0;
}
extern "C" MOSES_API int moses_debug_set_group(int on) {
  moses::g_group = on;
  return 0;
}
// split-bf16 weight gradients: 1 = split over K in clusters (gemm_wgrad_sk.cuh), 0 = one CTA per
// 128 x 64 tile (gemm_group.cuh); splits > 0 forces the cluster width
extern "C" MOSES_API int moses_debug_set_wgrad_sk(int on, int splits) {
  moses::g_wgrad_sk = on;
  moses::g_wgrad_sk_splits = splits;
  return 0;
}
// experiments: TMEM promotion interval (k-blocks of 64 rows; 0 = default) and a device buffer of
// 131 u64 clock64 stamps of block 0 (nullptr: off)
extern "C" MOSES_API int moses_debug_set_chain_pair(int on) {
  moses::g_chain_pair = on;
  return 0;
}
extern "C" MOSES_API int moses_debug_set_wgrad_early(int on) {
  moses::g_wgrad_early = on;
  return 0;
}
extern "C" MOSES_API int moses_debug_wgrad_sk_probe(int kc, void* trace) {
  moses::g_wgrad_sk_kc = kc;
  moses::g_wgrad_sk_trace = static_cast<unsigned long long*>(trace);
  return 0;
}
extern "C" MOSES_API int moses_debug_set_chain(int on) {
  moses::g_chain = on;
  return 0;
}
namespace moses {
extern int g_fwd;
extern int g_pair;
}
extern "C" MOSES_API int moses_debug_set_pair(int on) {
  moses::g_pair = on;
  return 0;
}
extern "C" MOSES_API int moses_debug_set_fwd(int on) {
  moses::g_fwd = on;
  return 0;
}
extern "C" MOSES_API int moses_debug_set_cluster(int on) {
  moses::g_cluster = on;
  return 0;
}
