// kernels.cuh — host-side launch wrappers for the non-GEMM kernels (kernels.cu).
#pragma once
#include "common.cuh"

namespace moses {

// Operand shadow of the fp32 master parameters written by every update kernel:
// kind 0 none, 1 bf16 (kind::f16 operand), 2 tf32-rounded fp32 (kind::tf32 operand),
// 3 (refresh_shadow only) 3xTF32 hi/lo pair: hi at ptr[i], lo at ptr[shadow_lo_offset(n) + i].
// operand shadow written by update kernels: 0 none, 1 bf16, 2 tf32-rounded fp32, 3 tf32 hi/lo pair
// (lo at ptr + shadow_lo_offset(n), refresh_shadow only), 4 bf16 hi/lo pair (MOSES_PREC_BF16X3: lo at
// ptr + lo_off elements; sgd_update and refresh_shadow)
struct Shadow {
  void* ptr;
  int kind;
  long long lo_off = 0;
};
// low half of a kind-3 shadow starts 128-byte aligned (TMA operands need 16-byte alignment)
__host__ __device__ constexpr long long shadow_lo_offset(long long n) { return (n + 31) / 32 * 32; }
void refresh_shadow(const float* w, long long n, Shadow sh, cudaStream_t s);

// ---- data movement
template <typename T>
void pack_rows(const double* src_d, long long n, int D, T* dst, long long ld, cudaStream_t s, T* lo = nullptr);
template <typename T>
void pack_rows_f32(const float* src_d, long long n, int D, long long lds, T* dst, long long ld, cudaStream_t s,
                   T* lo = nullptr);
template <typename T>
void set_ones_column(T* act, long long rows, int col, long long ld, cudaStream_t s);
template <typename T>
void unpack_rows(const T* src, long long n, int W, long long ld, double* dst_d, cudaStream_t s,
                 const T* lo = nullptr);
void f32_to_f64(const float* src, long long n, double* dst, cudaStream_t s);
void f64_to_f32(const double* src, long long n, float* dst, cudaStream_t s);
void f32_to_bf16(const float* src, long long n, __nv_bfloat16* dst, cudaStream_t s);
void strided_f64_to_f32(const double* src, long long rows, int W, float* dst, long long ldd, cudaStream_t s);
// batch b = (*counter % nb): rows [b*batch, (b+1)*batch) of a packed dataset -> dst, labels -> ydst
void gather_batch(const void* x_base, long long row_bytes, const float* y_base, const long long* counter, long long nb,
                  long long batch, void* dst, float* ydst, cudaStream_t s, void* dst_lo = nullptr);
void advance_counter(long long* c, cudaStream_t s);
// plan batch *counter: rows[off[b] .. off[b] + n) of a packed dataset -> dst, labels -> ydst
void gather_plan(const void* x_base, long long row_bytes, const float* y_base, const long long* rows, const long long* off,
                 const long long* counter, long long n, void* dst, float* ydst, cudaStream_t s, void* dst_lo = nullptr);
void accum_f64(const double* src, double* dst, cudaStream_t s);  // *dst += *src (one thread)
void gather_pooled(const void* x_base, long long row_bytes, const float* y_base, const long long* prog_off,
                   const long long* counter, long long nb, long long B, long long rows_pad, void* dst, float* ydst,
                   long long* seg_off, int* seg_rows, cudaStream_t s, void* dst_lo = nullptr);
// out[r] = H[r] . u  (warp per row)
void row_dot(const float* H, long long ldh, long long R, int W, const float* u, float* out, cudaStream_t s);
// discriminator_cross_entropy (lottery.cpp:207-218) over z[0,m) source and z[m,m+n) target
void disc_ce(const double* z, long long m, long long n, double* out, cudaStream_t s);

// ---- scores / ranking (model.cpp:71-106)
void head_scores(const float* part, int ntiles, long long ld, const float* head_bias, long long rows, float* s,
                 cudaStream_t st);
struct RankWs {
  double* gs_part;
  double* loss_part;
  long long* pairs_part;
  int nsplit;
};
int rank_splits(long long n);
void debug_set_rank_grid(bool on);  // rank_step: force the grid form
void debug_set_rank_sym(bool on);   // rank_step: symmetric form for batches past the cluster form (default on)
void keep_async_pool();             // the default memory pool keeps its memory across synchronisations
void rank_pairs(const float* s, const float* y, long long n, const RankWs& ws, cudaStream_t st);
// same, scores summed from the forward's per-N-tile head partials (+ head bias); s_out optional
void rank_pairs_fused(const float* part, int ntiles, long long ld, const float* hb, const long long* seg, const float* y,
                      long long n, const RankWs& ws, float* s_out, cudaStream_t st);
// Reduces the rank partials (fixed order), normalises by the pair count, folds in the
// adversary's logits when `part2` is given (model.cpp:215-238), and emits per-row
// backward coefficients coefA (ranking) / coefB (adversary) over all R = roff + n rows.
struct FinalizeOut {
  double* loss;       // [1]: rank loss + beta * -CE
  long long* pairs;   // [1]
  float* coefA;       // [R]
  float* coefB;       // [R]
  double* ce;         // [1] discriminator CE (adversary on)
  const int* seg_of_row = nullptr;  // pooled: program of each statement row (-1 = padding)
  long long R_rows = 0;             // pooled: statement rows
  float* gb = nullptr;              // pooled: head-bias gradient
};
void rank_finalize(const RankWs& ws, long long n, long long roff, const float* part2, int ntiles2, long long ld2,
                   const float* adv_bias, double beta, const FinalizeOut& out, cudaStream_t st,
                   const double* totals = nullptr);
// data-parallel exact batches: rows [r0, r0+nr) against all n columns (partials at [split][i - r0]),
// and the (loss sum, pair count) of those rows' partials -> out[0..1]
void rank_pairs_rows(const float* s, const float* y, long long n, long long r0, long long nr, const RankWs& ws,
                     cudaStream_t st);
void rank_local_totals(const RankWs& ws, long long nr, double* out, cudaStream_t st);
// MMD^2 (biased, Gaussian kernel) between rows [0, m) and [m, R) of H (+ H_lo for split operands) and its
// gradient G (R x W fp32, row-major) w.r.t. every row; value_out[0] = scale * MMD^2 (or += when
// accumulate). vpart: R doubles of workspace.
template <typename T>
void mmd_grad(const T* H, const T* H_lo, long long ld, long long R, long long m, int W, float sigma, float* G,
              double* vpart, double* value_out, double scale, bool accumulate, cudaStream_t st);
// sharded top-k: winners' (score, idx + row0) from device indices; slots [k_valid, k) = (-inf, -1)
void topk_winners(const float* s, const long long* idx, long long k_valid, long long k, long long row0, float* out_s,
                  long long* out_i, cudaStream_t st);
// rank_pairs_fused + rank_finalize in one launch (no adversary); `ticket` is a zeroed device
// counter the kernel re-arms. Returns false (nothing launched) when n is out of its range.
bool rank_step(const float* part, int ntiles, long long ld, const float* hb, const long long* seg, const float* y,
               long long n, const RankWs& ws, unsigned int* ticket, float* s_out, const int* seg_of_row, long long R,
               const FinalizeOut& out, cudaStream_t st);
// dZ_last[r][j] = (coefA[r]*wh[j] + coefB[r]*u[j]) * [H[r][j] > 0]
template <typename T>
void head_backward(const float* coefA, const float* coefB, const float* wh, const float* u, const T* H, long long ldh,
                   long long R, int W, T* dz, long long ldz, cudaStream_t st, T* dz_lo = nullptr,
                   const float* extra = nullptr, float extra_scale = 0.f);
// g[j] = sum_r coef[r] * H[r][j] (j < W), g[W] = sum_r coef[r]   (deterministic column reduction)
template <typename T>
void column_dot(const float* coef, const T* H, long long ldh, long long R, int W, float* g, float* ws, cudaStream_t st,
                const float* bias_override = nullptr, const T* H_lo = nullptr);
size_t column_dot_ws_floats(long long R, int W);

// ---- updates (model.cpp:263-296, lottery.cpp:92-120)
void sgd_update(float* w, float* v, const float* g, const uint8_t* mask, long long P, float lr, float mu, bool momentum,
                Shadow shadow, cudaStream_t st);
void adam_update(float* w, float* m1, float* m2, const float* g, const uint8_t* mask, long long P, float lr, float b1,
                 float b2, float eps, float c1, float c2, Shadow shadow, cudaStream_t st);
void variant_decay(float* w, const uint8_t* mask, long long P, float factor, Shadow shadow, cudaStream_t st);

// ---- lottery mask identification (lottery.cpp:35-90), fused with step + decay
struct SelectWs {
  unsigned* keys;       // [n]
  unsigned* hist;       // [2048]
  unsigned* block_hist; // [grid][2048]
  unsigned* state;      // select state (device)
  unsigned long long* counter;
  int grid;
};
size_t select_ws_bytes(long long n, int* grid_out);
void select_ws_carve(void* base, long long n, SelectWs* ws);
// xi = |w*g| -> keys; mode 1 threshold (normalised, strict >), 2 ratio (top ceil(rho*n), ties by index).
// do_step: transferable step (alpha) on kept scalars + variant decay (factor) on the rest.
void lottery_select(const float* w_in, const float* g, long long n, int mode, float theta, long long keep,
                    const SelectWs& ws, uint8_t* mask_out, float* xi_out, bool normalize_xi, cudaStream_t st);
void lottery_apply(float* w, const float* g, const uint8_t* mask, long long n, float alpha, float factor, bool step,
                   bool decay, Shadow shadow, cudaStream_t st);
void xi_scores(const float* w, const float* g, long long n, bool normalize, const SelectWs& ws, float* xi_out,
               cudaStream_t st);
// mask from given xi (identical-input parity path)
void partition_from_xi(const float* xi, long long n, int mode, float theta, long long keep, const SelectWs& ws,
                       uint8_t* mask_out, cudaStream_t st);
long long popcount_mask(const uint8_t* mask, long long n, unsigned long long* dcount, cudaStream_t st);
// lottery.cu: fused xi -> partition -> transferable_step -> variant_decay, xi never materialised
size_t lottery_ws_bytes(long long n);
struct AdamOpt {  // masked Adam on the transferable scalars (null: the reference's plain step)
  float* m1;
  float* m2;
  float b1, b2, eps, c1, c2;
};
int lottery_step_fused(float* w, const float* g, long long n, int mode, float theta, long long keep, float alpha,
                       float factor, bool decay, Shadow sh, uint8_t* mask, void* ws, unsigned long long* popcount_dev,
                       cudaStream_t st, const AdamOpt* adam = nullptr);

// ---- candidate top-k (search.cpp:32-37): (score desc, index asc)
void topk_select(const float* scores, long long n, long long k, const SelectWs& ws, unsigned* out_key, long long* out_idx,
                 cudaStream_t st);
constexpr long long kTopkMax = 4096;
// one-launch sampled top-k (topk.cu); false = not applicable / not conclusive (run topk_select)
size_t topk_fast_ws_bytes(long long n);
// launch only (false = not applicable); *fail_out (device) = 1 when not conclusive, else 0 and the result out
void lottery_res_trace_read(unsigned long long* out8);  // debug: the resident step's phase stamps
void topk_trace_read(unsigned long long* out16);  // debug: the one-launch kernel's phase stamps
bool topk_fast_launch(const float* scores, long long n, long long k, void* ws, unsigned* out_key, long long* out_idx,
                      unsigned* fail_out, cudaStream_t st);
void select_kth_key(long long n, unsigned long long need, const SelectWs& ws, cudaStream_t st);
const unsigned* sel_result_key(const SelectWs& ws);
bool topk_fast(const float* scores, long long n, long long k, void* ws, unsigned* out_key, long long* out_idx,
               cudaStream_t st);

// ---- accuracy (model.cpp:298-312)
void accuracy_counts(const float* s, const float* y, const long long* seg_of_row, const long long* seg_off, long long n,
                     long long* pairs_part, long long* conc_part, unsigned long long* totals, cudaStream_t st);

// ---- adversary (lottery.cpp:135-164)
template <typename T>
void adversary_step(const float* part2, int ntiles, long long ld2, const T* H, long long ldh, long long m, long long n,
                    int W, float* u, float* c, float eta, double* loss_out, float* ws, cudaStream_t st,
                    const T* H_lo = nullptr);

// ---- extensions
template <typename T>
void segment_sum(const T* H, long long ldh, int W, const long long* offsets, long long programs, float* out,
                 long long ldo, cudaStream_t st);
void segment_sum_scalar(const float* v, const long long* offsets, long long programs, float bias, float* out,
                        cudaStream_t st);
// tensor-core MMD^2 (gemm_gram.cuh): rows with stride ld; ws of mmd_ws_bytes(m, n, W)
size_t mmd_ws_bytes(long long m, long long n, int W);
double mmd2_tc(const float* xs, long long m, const float* xt, long long n, int W, long long ld, float sigma, void* ws,
               cudaStream_t s, int* launches);

// ---- synthetic TenSet-shaped data (bit-identical to oracle::synth_*)
template <typename T>
void synth_features(unsigned long long seed, long long row0, long long n, int D, T* dst, long long ld, cudaStream_t st);
void synth_labels(unsigned long long seed, long long row0, long long n, float* dst, cudaStream_t st);

// device -> mapped pinned host scalar without a copy engine
void store_scalar_f64(const double* src, double* dst, cudaStream_t s);
// host-input pooled training step: staging slot -> packed rows, labels, segments (kernels.cu)
template <typename T>
void pack_pooled(const double* xs, const double* ys, const long long* offs, const long long* dims_dev, int D,
                 long long rows_pad, T* act0, long long ld, float* ydst, long long* seg_off, int* seg_rows,
                 cudaStream_t s, T* lo = nullptr);
// simulated hardware (space.cu): measure() labels and the exhaustive noise-free optimum
int measure_configs(const double* dev6, int repeats, const char* device_id, const char* task_id, const double* task4,
                    const long long* domains, const int* sizes, const int* roles, int nk, unsigned long long seed,
                    unsigned long long first, long long n, double* clean_ms, double* thr, double* lat, double* wall,
                    float* label, cudaStream_t st);
// measure() of configurations given by enumeration index (device list; tuner.cu)
int measure_configs_idx(const double* dev6, int repeats, const char* device_id, const char* task_id,
                        const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                        unsigned long long seed, const unsigned long long* idx_dev, long long n, double* thr,
                        double* lat, double* wall, cudaStream_t st);
int true_best(const double* dev6, const double* task4, const long long* domains, const int* sizes, const int* roles,
              int nk, long long* best_values, double* best_latency, cudaStream_t st);
// knob-space candidate generation (space.cu); out_kind 0 f32, 1 bf16, 2 f64
int encode_configs(const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                   unsigned long long first, long long n, int out_kind, void* feat, long long ld, int D,
                   unsigned long long* hash, long long* values_out, cudaStream_t st);
// feature rows of configurations given by enumeration index (device list)
int encode_configs_idx(const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                       const unsigned long long* idx_dev, long long n, int out_kind, void* feat, long long ld, int D,
                       cudaStream_t st);
// generate_dataset for one task (data.cpp:49-65): keyed sample_config draws, features, measure() labels
int generate_task_dataset(const double* dev6, int repeats, const char* device_id, const char* task_id,
                          const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                          long long samples, unsigned long long seed, int out_kind, void* feat, long long ld, int D,
                          long long* values_out, double* thr, double* lat, double* wall, float* label,
                          unsigned long long* idx_out, cudaStream_t st);
void debug_force_serial_sampling(bool on);
// validate_config + encode_features over device rows of knob values (space.cpp:69-81,140-159)
int encode_values(const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                  const long long* values, long long n, int out_kind, void* feat, long long ld, int D,
                  unsigned long long* hash, unsigned long long* idx_out, long long* bad_row, cudaStream_t st);

}  // namespace moses
