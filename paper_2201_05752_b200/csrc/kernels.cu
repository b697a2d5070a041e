// kernels.cu — the non-GEMM sm_100a kernels of the Moses hot path.
//
// Everything here is bandwidth- or latency-bound integer/elementwise work, so
// the rules are: coalesced 16-byte accesses, grids sized to the 148 SMs,
// and fixed-order reductions (no float atomics) so every result is
// bit-reproducible run to run. Integer atomics (histograms, counts) are
// order-independent and therefore deterministic too.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "kernels.cuh"
#include "ptx.cuh"

namespace moses {
namespace {

constexpr int kSMs = 148;

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
__device__ __forceinline__ float tf32_rna(float x);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return tf32_rna(v); }  // fp32 activations feed kind::tf32
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Round-to-nearest tf32 (the tensor core drops the low 13 mantissa bits of a kind::tf32
// operand; pre-rounding keeps the error unbiased).
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// operand shadow of the master parameters: 0 none, 1 bf16, 2 tf32-rounded fp32
template <int KIND>
__device__ __forceinline__ void store_shadow(void* sh, long long i, float w, long long lo_off = 0) {
  if constexpr (KIND == 1) static_cast<__nv_bfloat16*>(sh)[i] = __float2bfloat16_rn(w);
  if constexpr (KIND == 2) static_cast<float*>(sh)[i] = tf32_rna(w);
  if constexpr (KIND == 4) {  // split bf16: hi = rn(w), lo = rn(w - hi)
    const __nv_bfloat16 h = __float2bfloat16_rn(w);
    static_cast<__nv_bfloat16*>(sh)[i] = h;
    static_cast<__nv_bfloat16*>(sh)[i + lo_off] = __float2bfloat16_rn(w - __bfloat162float(h));
  }
}

int grid_for(long long n, int block, int per_sm = 8) {
  long long g = (n + block - 1) / block;
  return int(g < 1 ? 1 : (g > kSMs * per_sm ? kSMs * per_sm : g));
}

// ---------------------------------------------------------------- data movement
// 3xTF32 operands (fp32 parity mode): hi = rna_tf32(v) in dst, lo = rna_tf32(v - hi) in lo.
// Split operands: lo = the residual rounded to the same operand type (tf32 for 3xTF32, bf16 for
// split bf16), so hi + lo carries 2x the operand precision.
template <typename T>
__device__ __forceinline__ void store_operand(T* dst, T* lo, long long i, float v) {
  const T h = from_f<T>(v);
  dst[i] = h;
  if (lo != nullptr) lo[i] = from_f<T>(v - to_f(h));
}
template <typename T>
__device__ __forceinline__ float load_operand(const T* src, const T* lo, long long i) {
  return lo != nullptr ? to_f(src[i]) + to_f(lo[i]) : to_f(src[i]);
}
template <typename T>
__global__ void pack_rows_kernel(const double* __restrict__ src, long long n, int D, T* __restrict__ dst, long long ld,
                                 T* __restrict__ lo) {
  ptx::pdl_launch_dependents();
  const long long total = n * ld;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ld;
    const int c = int(i - r * ld);
    const float v = c < D ? float(src[r * D + c]) : (c == D ? 1.f : 0.f);
    store_operand(dst, lo, i, v);
  }
}
template <typename T>
__global__ void pack_rows_f32_kernel(const float* __restrict__ src, long long n, int D, long long lds, T* __restrict__ dst,
                                     long long ld, T* __restrict__ lo) {
  const long long total = n * ld;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ld;
    const int c = int(i - r * ld);
    const float v = c < D ? src[r * lds + c] : (c == D ? 1.f : 0.f);
    store_operand(dst, lo, i, v);
  }
}
template <typename T>
__global__ void set_col_kernel(T* act, long long rows, int col, long long ld) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x)
    act[r * ld + col] = from_f<T>(1.f);
}
template <typename T>
__global__ void unpack_rows_kernel(const T* __restrict__ src, long long n, int W, long long ld, double* __restrict__ dst,
                                   const T* __restrict__ lo) {
  const long long total = n * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / W;
    const int c = int(i - r * W);
    dst[i] = lo != nullptr ? double(to_f(src[r * ld + c])) + double(to_f(lo[r * ld + c])) : double(to_f(src[r * ld + c]));
  }
}
__global__ void f32_to_f64_kernel(const float* s, long long n, double* d) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) d[i] = s[i];
}
__global__ void f64_to_f32_kernel(const double* s, long long n, float* d) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) d[i] = float(s[i]);
}
__global__ void f32_to_bf16_kernel(const float* s, long long n, __nv_bfloat16* d) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = __float2bfloat16_rn(s[i]);
}

__global__ void strided_f64_to_f32_kernel(const double* s, long long rows, int W, float* d, long long ldd) {
  const long long total = rows * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / W;
    d[r * ldd + (i - r * W)] = float(s[i]);
  }
}
__global__ void row_dot_kernel(const float* __restrict__ H, long long ldh, long long R, int W, const float* __restrict__ u,
                               float* __restrict__ out) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < R; r += nw) {
    float acc = 0.f;
    for (int j = lane; j < W; j += 32) acc = fmaf(H[r * ldh + j], u[j], acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = acc;
  }
}

// ---------------------------------------------------------------- device-resident batch gather (graph replay)
// Every gather moves 16-byte chunks of packed rows. With a lo plane (split-bf16 handles) the dataset
// rows are fp32 and chunk i (4 values) lands as 4 bf16 hi values at dst[4i..] and 4 bf16 lo values
// at lo[4i..] (lo = rn(v - hi)).
__device__ __forceinline__ void put_chunk(uint8_t* __restrict__ dst, uint8_t* __restrict__ lo, long long i, uint4 v) {
  if (lo == nullptr) {
    reinterpret_cast<uint4*>(dst)[i] = v;
    return;
  }
  const float f[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
  const __nv_bfloat162 h0 = __floats2bfloat162_rn(f[0], f[1]), h1 = __floats2bfloat162_rn(f[2], f[3]);
  const __nv_bfloat162 l0 = __floats2bfloat162_rn(f[0] - __low2float(h0), f[1] - __high2float(h0));
  const __nv_bfloat162 l1 = __floats2bfloat162_rn(f[2] - __low2float(h1), f[3] - __high2float(h1));
  uint2 hv, lv;
  hv.x = *reinterpret_cast<const uint32_t*>(&h0);
  hv.y = *reinterpret_cast<const uint32_t*>(&h1);
  lv.x = *reinterpret_cast<const uint32_t*>(&l0);
  lv.y = *reinterpret_cast<const uint32_t*>(&l1);
  reinterpret_cast<uint2*>(dst)[i] = hv;
  reinterpret_cast<uint2*>(lo)[i] = lv;
}
__global__ void gather_batch_kernel(const uint8_t* __restrict__ x_base, long long row_bytes, const float* __restrict__ y_base,
                                    const long long* __restrict__ counter, long long nb, long long batch,
                                    uint8_t* __restrict__ dst, float* __restrict__ ydst, uint8_t* __restrict__ dlo) {
  ptx::pdl_launch_dependents();
  const long long b = (*counter) % nb;
  const uint4* src = reinterpret_cast<const uint4*>(x_base + b * batch * row_bytes);
  const long long n16 = batch * row_bytes / 16;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
    put_chunk(dst, dlo, i, src[i]);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < batch; i += (long long)gridDim.x * blockDim.x)
    ydst[i] = y_base[b * batch + i];
}
// Plan batch b = *counter: rows rows[off[b] + r] (r < n) of a packed dataset -> dst rows [0, n),
// labels -> ydst. One warp per row, 16-byte lanes.
__global__ void gather_plan_kernel(const uint8_t* __restrict__ x_base, long long row_bytes, const float* __restrict__ y_base,
                                   const long long* __restrict__ rows, const long long* __restrict__ off,
                                   const long long* __restrict__ counter, long long n, uint8_t* __restrict__ dst,
                                   float* __restrict__ ydst, uint8_t* __restrict__ dlo) {
  ptx::pdl_launch_dependents();
  const long long base = off[*counter];
  const int lane = threadIdx.x & 31;
  const long long w16 = row_bytes / 16;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long src_row = rows[base + r];
    const uint4* src = reinterpret_cast<const uint4*>(x_base + src_row * row_bytes);
    for (long long c = lane; c < w16; c += 32) put_chunk(dst, dlo, r * w16 + c, src[c]);
    if (lane == 0) ydst[r] = y_base[src_row];
  }
}
__global__ void accum_f64_kernel(const double* __restrict__ src, double* __restrict__ dst) { *dst += *src; }
// TenSet-shaped batch: programs [b*B, (b+1)*B) of a CSR-packed statement dataset -> statement rows
// [0, R_b) of dst, batch-relative offsets, program of each row (-1 on padding rows up to rows_pad).
__global__ void gather_pooled_kernel(const uint8_t* __restrict__ x_base, long long row_bytes, const float* __restrict__ y_base,
                                     const long long* __restrict__ prog_off, const long long* __restrict__ counter,
                                     long long nb, long long B, long long rows_pad, uint8_t* __restrict__ dst,
                                     float* __restrict__ ydst, long long* __restrict__ seg_off, int* __restrict__ seg_rows,
                                     uint8_t* __restrict__ dlo) {
  ptx::pdl_launch_dependents();
  const long long b = (*counter) % nb;
  const long long p0 = b * B, r0 = prog_off[p0], Rb = prog_off[p0 + B] - r0;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nthr = (long long)gridDim.x * blockDim.x;
  const uint4* src = reinterpret_cast<const uint4*>(x_base + r0 * row_bytes);
  const long long n16 = Rb * row_bytes / 16;
  for (long long i = tid; i < n16; i += nthr) put_chunk(dst, dlo, i, src[i]);
  for (long long p = tid; p <= B; p += nthr) {
    const long long lo = prog_off[p0 + p] - r0;
    seg_off[p] = lo;
    if (p < B) {
      ydst[p] = y_base[p0 + p];
      const long long hi = prog_off[p0 + p + 1] - r0;
      for (long long r = lo; r < hi; ++r) seg_rows[r] = int(p);
    }
  }
  for (long long r = Rb + tid; r < rows_pad; r += nthr) seg_rows[r] = -1;
}
// Host-input pooled step (moses_train_step_pooled_async): one staging slot of float64 statement
// rows / labels / CSR offsets -> packed bf16 model rows (+ the constant column), fp32 labels, the
// batch's segment offsets and row -> program map. Rows [n_stmt, rows_pad) keep their (finite)
// contents and are masked by seg_rows = -1. *n_stmt_dev / *programs_dev are read on the device so
// one captured graph serves every batch size up to the capacity.
template <typename T>
__global__ void pack_pooled_kernel(const double* __restrict__ xs, const double* __restrict__ ys,
                                   const long long* __restrict__ offs, const long long* __restrict__ dims_dev, int D,
                                   long long rows_pad, T* __restrict__ act0, long long ld, float* __restrict__ ydst,
                                   long long* __restrict__ seg_off, int* __restrict__ seg_rows, T* __restrict__ lo) {
  ptx::pdl_launch_dependents();
  const long long n_stmt = dims_dev[0], programs = dims_dev[1];
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nthr = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n_stmt * ld; i += nthr) {
    const long long r = i / ld;
    const int c = int(i - r * ld);
    const float v = c < D ? float(xs[r * D + c]) : (c == D ? 1.f : 0.f);
    store_operand(act0, lo, i, v);
  }
  for (long long p = tid; p <= programs; p += nthr) {
    seg_off[p] = offs[p];
    if (p < programs) {
      ydst[p] = float(ys[p]);
      for (long long r = offs[p]; r < offs[p + 1]; ++r) seg_rows[r] = int(p);
    }
  }
  for (long long r = n_stmt + tid; r < rows_pad; r += nthr) seg_rows[r] = -1;
}

__global__ void store_scalar_f64_kernel(const double* src, double* dst) { *dst = *src; }
__global__ void advance_counter_kernel(long long* c) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *c += 1;
}

// ---------------------------------------------------------------- scores from head partials
__global__ void head_scores_kernel(const float* __restrict__ part, int ntiles, long long ld, const float* __restrict__ hb,
                                   long long rows, float* __restrict__ s) {
  const float b = hb[0];
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int t = 0; t < ntiles; ++t) acc += part[t * ld + r];  // fixed tile order
    s[r] = acc + b;
  }
}

// ---------------------------------------------------------------- pairwise ranking (model.cpp:71-106)
// Row i accumulates, over its column split, every pair it belongs to:
//   y_i > y_j : i is "hi": gs_i -= sigma(-(s_i - s_j)), loss += softplus(-(s_i - s_j)), pairs++
//   y_j > y_i : i is "lo": gs_i += sigma(-(s_j - s_i))
// Each distinct-label pair is counted once (at its hi row), as in the reference's i<j loop.
constexpr int kRankBlock = 128;
constexpr int kRankChunk = 32;  // j columns per block: n=512 -> 4 x 16 blocks, n=4096 -> 32 x 128
// Scores come either from `s` or, fused, from the last forward epilogue's per-N-tile partials
// (s_r = b + sum_t part[t][r], the same fixed order as head_scores_kernel).
// With `seg` (CSR program offsets over statement rows) the score of program r is the segment sum of
// its statements' head dots (segment-sum pooling folded into the head).
// 1 / (1 + e) for e in (0, 1]: MUFU reciprocal (<= 1 ulp), no IEEE slow-path branch in the pair loops
__device__ __forceinline__ float rcp_pair(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// exp(-|d|) as one MUFU ex2 of the flush-to-zero kind (no denormal fix-up instructions), for every form
// of the pair loop alike (the row coefficients stay bit-identical across forms); lg2 for the softplus sums
__device__ __forceinline__ float ex2_ftz(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_ftz(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float score_of(const float* __restrict__ s, const float* __restrict__ part, int ntiles,
                                          long long ld, float hb, const long long* __restrict__ seg, long long r) {
  if (part == nullptr) return s[r];
  float acc = 0.f;
  if (seg == nullptr) {
    for (int t = 0; t < ntiles; ++t) acc += part[t * ld + r];
  } else {
    for (long long i = seg[r]; i < seg[r + 1]; ++i) {
      float a = 0.f;
      for (int t = 0; t < ntiles; ++t) a += part[t * ld + i];
      acc += a;
    }
  }
  return acc + hb;
}
__global__ void __launch_bounds__(kRankBlock) rank_pairs_kernel(const float* __restrict__ s, const float* __restrict__ part,
                                                                int ntiles, long long ld, const float* __restrict__ hbp,
                                                                const long long* __restrict__ seg,
                                                                const float* __restrict__ y, long long n, double* gs_part,
                                                                double* loss_part, long long* pairs_part,
                                                                float* __restrict__ s_out, long long r0, long long nr) {
  // rows [r0, r0 + nr) of the batch against all n columns (data-parallel exact batches: a rank's
  // own rows against the all-gathered batch); partials at [split][i - r0]
  __shared__ float ss[kRankChunk], sy[kRankChunk];
  const float hb = part ? hbp[0] : 0.f;
  const long long i = r0 + blockIdx.x * (long long)kRankBlock + threadIdx.x;
  const long long j0 = (long long)blockIdx.y * kRankChunk;
  const int cnt = int(min((long long)kRankChunk, n - j0));
  if (threadIdx.x < cnt) {
    ss[threadIdx.x] = score_of(s, part, ntiles, ld, hb, seg, j0 + threadIdx.x);
    sy[threadIdx.x] = y[j0 + threadIdx.x];
  }
  __syncthreads();
  if (i >= r0 + nr) return;
  const float si = score_of(s, part, ntiles, ld, hb, seg, i), yi = y[i];
  if (s_out != nullptr && blockIdx.y == 0) s_out[i - r0] = si;
  float gs = 0.f, loss = 0.f;
  int pairs = 0;
#pragma unroll 4
  for (int q = 0; q < cnt; ++q) {
    const float yj = sy[q];
    if (yi == yj) continue;
    const bool hi = yi > yj;
    const float d = hi ? si - ss[q] : ss[q] - si;  // s_hi - s_lo
    const float e = ex2_ftz(fabsf(d) * -1.4426950408889634f);
    const float inv = rcp_pair(1.f + e);
    const float sig_neg = d >= 0.f ? e * inv : inv;  // sigma(-d)
    if (hi) {
      gs -= sig_neg;
      loss += (d >= 0.f ? 0.f : -d) + log1pf(e);
      ++pairs;
    } else {
      gs += sig_neg;
    }
  }
  const long long o = (long long)blockIdx.y * nr + (i - r0);
  gs_part[o] = gs;
  loss_part[o] = loss;
  pairs_part[o] = pairs;
}

// per-row reduction of the split partials (fixed split order)
__global__ void rank_rows_kernel(double* gs_part, double* loss_part, long long* pairs_part, int nsplit, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double g = 0.0, l = 0.0;
    long long p = 0;
    for (int sp = 0; sp < nsplit; ++sp) {
      g += gs_part[sp * n + i];
      l += loss_part[sp * n + i];
      p += pairs_part[sp * n + i];
    }
    gs_part[i] = g;
    loss_part[i] = l;
    pairs_part[i] = p;
  }
}

__device__ __forceinline__ float stable_sigmoid(float x) {  // model.cpp:64-68
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}
__device__ __forceinline__ double softplus_d(double v) { return fmax(v, 0.0) + log1p(exp(-fabs(v))); }

constexpr int kFinBlock = 1024;
__global__ void __launch_bounds__(kFinBlock) rank_finalize_kernel(const double* gs_part, const double* loss_part,
                                                                  const long long* pairs_part, int nsplit, long long n,
                                                                  long long roff, const float* part2, int ntiles2,
                                                                  long long ld2, const float* adv_bias, double beta,
                                                                  double* loss_out, long long* pairs_out, float* coefA,
                                                                  float* coefB, double* ce_out,
                                                                  const int* __restrict__ seg_of_row, long long R_rows,
                                                                  float* gb_out, const double* totals) {
  ptx::pdl_launch_dependents();
  using BR = cub::BlockReduce<double, kFinBlock>;
  using BRL = cub::BlockReduce<long long, kFinBlock>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ typename BRL::TempStorage tmpl;
  __shared__ double sh_loss;
  __shared__ long long sh_pairs;
  long long p = 0;
  double l = 0.0;
  for (long long i = threadIdx.x; i < n; i += kFinBlock)  // fixed order: row-major over (row, split)
    for (int sp = 0; sp < nsplit; ++sp) {
      p += pairs_part[sp * n + i];
      l += loss_part[sp * n + i];
    }
  long long ptot = BRL(tmpl).Sum(p);
  __syncthreads();
  double ltot = BR(tmp).Sum(l);
  if (totals != nullptr) {  // data-parallel exact batch: every rank's partials, all-reduced
    ltot = totals[0];
    ptot = (long long)llrint(totals[1]);
  }
  if (threadIdx.x == 0) {
    sh_pairs = ptot;
    sh_loss = ptot > 0 ? ltot / double(ptot) : 0.0;
  }
  __syncthreads();
  const long long pairs = sh_pairs;
  const double inv = pairs > 0 ? 1.0 / double(pairs) : 0.0;
  const long long R = seg_of_row ? R_rows : roff + n;
  if (seg_of_row != nullptr) {
    // pooled: every statement row of program p carries d loss / d s_p (ds_p/dH_i = w_head for i in p);
    // the head bias enters each program once, so its gradient is sum_p gs_p (written to gb_out).
    double gbs = 0.0;
    for (long long q = threadIdx.x; q < n; q += kFinBlock)
      for (int sp = 0; sp < nsplit; ++sp) gbs += gs_part[sp * n + q];
    for (long long r = threadIdx.x; r < R; r += kFinBlock) {
      const int sg = seg_of_row[r];
      float a = 0.f;
      if (sg >= 0 && pairs > 0) {
        double g = 0.0;
        for (int sp = 0; sp < nsplit; ++sp) g += gs_part[sp * n + sg];
        a = float(g * inv);
      }
      coefA[r] = a;
      coefB[r] = 0.f;
    }
    __syncthreads();
    const double gbt = BR(tmp).Sum(gbs);
    if (threadIdx.x == 0 && gb_out) *gb_out = pairs > 0 ? float(gbt * inv) : 0.f;
  } else {
    for (long long r = threadIdx.x; r < R; r += kFinBlock) {
      float a = 0.f;
      if (r >= roff) {
        double g = 0.0;
        for (int sp = 0; sp < nsplit; ++sp) g += gs_part[sp * n + (r - roff)];
        a = pairs > 0 ? float(g * inv) : 0.f;
      }
      coefA[r] = a;
      coefB[r] = 0.f;
    }
  }
  double total = sh_loss;
  if (part2 != nullptr && beta != 0.0 && n > 0) {
    // logits z = c + sum of per-tile partial dots (fixed order); reversed gradient (model.cpp:224-231)
    const float c = adv_bias[0];
    const long long m = roff;
    double ls = 0.0, lt = 0.0;
    for (long long r = threadIdx.x; r < R; r += kFinBlock) {
      float z = 0.f;
      for (int t = 0; t < ntiles2; ++t) z += part2[t * ld2 + r];
      z += c;
      if (r < m) {
        coefB[r] = float(0.5 * beta * double(stable_sigmoid(-z)) / double(m));
        ls += softplus_d(-double(z));
      } else {
        coefB[r] = float(-0.5 * beta * double(stable_sigmoid(z)) / double(n));
        lt += softplus_d(double(z));
      }
    }
    __syncthreads();
    const double lst = BR(tmp).Sum(ls);
    __syncthreads();
    const double ltt = BR(tmp).Sum(lt);
    if (threadIdx.x == 0) {
      const double ce = 0.5 * (lst / double(m) + ltt / double(n));
      total += beta * -ce;
      if (ce_out) *ce_out = ce;
    }
  }
  if (threadIdx.x == 0) {
    *loss_out = total;
    *pairs_out = pairs;
  }
}

// ---------------------------------------------------------------- fused ranking step
// rank_pairs + rank_finalize in ONE launch (no adversary): one cluster of 16 CTAs x 512 threads.
// Each CTA scores its n/16 programs (per-row fixed-order tile sums of the forward's head
// partials, then per-program segment sums — score_of()'s arithmetic), all-gathers the scores
// through DSMEM, and evaluates the pairs of its n/8 programs with rank_pairs_kernel's (row, 32-column split) float
// partials, reduced per row in split order (double) — the same per-row values as the two-kernel
// path. Pair counts, loss and head-bias partials are all-gathered through DSMEM, so every CTA
// knows 1/pairs and writes the backward coefficients of its programs' statement rows itself;
// CTA 0 sums the loss / bias partials in CTA order. Deterministic.
__device__ unsigned long long g_rank_trace[16];
__device__ unsigned long long g_rank_cta_trace[512 * 5];  // rank_sym_kernel: per-CTA phase stamps
__device__ __forceinline__ void rank_cta_stamp(int k) {
  if (threadIdx.x == 0 && blockIdx.x < 512) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    g_rank_cta_trace[blockIdx.x * 5 + k] = v;
  }
}
__device__ __forceinline__ void rank_stamp(int k) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    g_rank_trace[k] = v;
  }
}
constexpr int kRankCluster = 16;  // non-portable cluster size (B200 supports 16)
constexpr int kRankThreads = 512;
constexpr int kRankMaxItems = 4096;  // (rows per CTA) x (32-column splits)
constexpr int kRankMaxRows = 256;    // programs per CTA
struct RankRed {
  long long pairs;
  double loss, gb;
};
__global__ void __launch_bounds__(kRankThreads)
    rank_cluster_kernel(const float* __restrict__ part, int ntiles, long long ld, const float* __restrict__ hbp,
                        const long long* __restrict__ seg, const float* __restrict__ y, long long n, int nsplit,
                        int rows_per_cta, float* __restrict__ s_out, long long R, double* loss_out,
                        long long* pairs_out, float* __restrict__ coefA, float* __restrict__ coefB, float* gb_out) {
  extern __shared__ float rs_smem[];
  float* ss = rs_smem;      // [n] scores (all-gathered through DSMEM)
  float* sy = ss + n;       // [n] labels
  float* pg = sy + n;       // [items] per-(split, row) partials
  float* pl = pg + kRankMaxItems;
  int* pp = reinterpret_cast<int*>(pl + kRankMaxItems);
  float* srow = reinterpret_cast<float*>(pp + kRankMaxItems);  // pooled: this CTA's statement head dots
  __shared__ double row_g[kRankMaxRows];
  __shared__ RankRed red[kRankCluster];  // all-gathered per-CTA totals
  __shared__ double wl[32], wg[32];
  __shared__ long long wp[32];
  __shared__ long long sseg[kRankMaxRows + 1];
  const int t = threadIdx.x;
  rank_stamp(0);
  ptx::pdl_launch_dependents();  // the head backward may be scheduled now; it waits for our completion
  // every CTA of the cluster must be running before a peer writes into its shared memory (the
  // score all-gather below): arrive now, wait right before the first remote store. Without it a
  // late-starting CTA can lose peers' scores and keep the values of the previous launch.
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const uint32_t q = ptx::cluster_ctarank();
  const long long p0 = min(n, (long long)q * rows_per_cta);
  const long long p1 = min(n, p0 + rows_per_cta);
  // labels and batch offsets were written before the forward pass: read them while it drains
  // (programmatic launch); the head partials and bias only after it has completed
  for (long long p = t; p < n; p += blockDim.x) sy[p] = y[p];
  if (seg != nullptr)
    for (long long k = t; k <= p1 - p0; k += blockDim.x) sseg[k] = seg[p0 + k];
  ptx::pdl_wait();
  const float hb = hbp[0];
  // scores of THIS CTA's programs (fixed tile order per statement row, then the segment sum)
  if (seg != nullptr) {
    __syncthreads();
    const long long r0 = sseg[0], r1 = sseg[p1 - p0];
    for (long long r = r0 + t; r < r1; r += blockDim.x) {
      float v[8];
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) v[tt] = tt < ntiles ? __ldg(part + tt * ld + r) : 0.f;
      float a = 0.f;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt)
        if (tt < ntiles) a += v[tt];
      for (int tt = 8; tt < ntiles; ++tt) a += __ldg(part + tt * ld + r);
      srow[r - r0] = a;
    }
    __syncthreads();
    for (long long p = p0 + t; p < p1; p += blockDim.x) {
      float acc = 0.f;
      for (long long i = sseg[p - p0]; i < sseg[p - p0 + 1]; ++i) acc += srow[i - r0];
      ss[p] = acc + hb;
    }
  } else {
    for (long long p = p0 + t; p < p1; p += blockDim.x) {
      float a = 0.f;
      for (int tt = 0; tt < ntiles; ++tt) a += __ldg(part + tt * ld + p);
      ss[p] = a + hb;
    }
  }
  __syncthreads();
  rank_stamp(1);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  // all-gather: every CTA's scores into every peer's ss[] (same offsets)
  for (long long k = t; k < (p1 - p0) * kRankCluster; k += blockDim.x) {
    const long long p = p0 + k / kRankCluster;
    const uint32_t dst = uint32_t(k % kRankCluster);
    if (dst == q) continue;
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(ptx::smem_u32(ss + p)), "r"(dst));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(ss[p]) : "memory");
  }
  ptx::cluster_sync();
  rank_stamp(2);
  // pairs of this CTA's programs: item = (split, local row) — a warp shares one split, so the
  // column reads are shared-memory broadcasts (row-major items put 16 splits 32 floats apart:
  // 16-way bank conflicts, measured 17 us for this phase)
  const int items = rows_per_cta * nsplit;
  for (int it = t; it < items; it += blockDim.x) {
    const int sp = it / rows_per_cta, lr = it - sp * rows_per_cta;
    const long long i = p0 + lr;
    float gs = 0.f, loss = 0.f, lp = 1.f;
    int pairs = 0;
    if (i < n) {
      const float si = ss[i], yi = sy[i];
      const long long j0 = (long long)sp * kRankChunk;
      const int cnt = int(min((long long)kRankChunk, n - j0));
      // branch-free pair terms: w = +1 (i is the hi row), -1 (lo), 0 (tie). gs accumulates the
      // same values in the same order as rank_pairs_kernel (+-0 for ties); the softplus uses
      // log1p(e) = -log(1/(1+e)) on the reciprocal already at hand (MUFU lg2).
#pragma unroll 4
      for (int k = 0; k < cnt; ++k) {
        const float yj = sy[j0 + k];
        const float w = float(yi > yj) - float(yi < yj);
        const float d = w * (si - ss[j0 + k]);
        const float e = ex2_ftz(fabsf(d) * -1.4426950408889634f);
        const float iv = rcp_pair(1.f + e);
        const float sig_neg = d >= 0.f ? e * iv : iv;
        gs = w != 0.f ? gs - w * sig_neg : gs;
        const bool hi = w > 0.f;
        loss += hi ? fmaxf(-d, 0.f) : 0.f;
        lp *= hi ? 1.f + e : 1.f;  // softplus terms log1p(e) as one log of their product (<= 2^32)
        pairs += hi;
      }
      loss += 0.69314718055994531f * lg2_ftz(lp);
    }
    pg[it] = gs;
    pl[it] = loss;
    pp[it] = pairs;
  }
  __syncthreads();
  rank_stamp(3);
  // per-row reduction in split order; CTA totals (row order)
  double l_t = 0.0, g_t = 0.0;
  long long c_t = 0;
  for (int lr = t; lr < rows_per_cta; lr += blockDim.x) {
    double g = 0.0, l = 0.0;
    long long c = 0;
    if (p0 + lr < n) {
      for (int k = 0; k < nsplit; ++k) {
        g += pg[k * rows_per_cta + lr];
        l += pl[k * rows_per_cta + lr];
        c += pp[k * rows_per_cta + lr];
      }
      if (s_out != nullptr) s_out[p0 + lr] = ss[p0 + lr];
    }
    row_g[lr] = g;
    l_t += l;  // a thread's rows are visited in increasing order; warp/CTA order below is fixed
    g_t += g;
    c_t += c;
  }
  // fixed-order CTA reduction: lanes (shuffle tree), then warps in order
  for (int o = 16; o > 0; o >>= 1) {
    l_t += __shfl_down_sync(0xffffffffu, l_t, o);
    g_t += __shfl_down_sync(0xffffffffu, g_t, o);
    c_t += __shfl_down_sync(0xffffffffu, c_t, o);
  }
  if ((t & 31) == 0) {
    wl[t >> 5] = l_t;
    wg[t >> 5] = g_t;
    wp[t >> 5] = c_t;
  }
  __syncthreads();
  if (t == 0) {
    RankRed mine{0, 0.0, 0.0};
    for (int w = 0; w < int(blockDim.x >> 5); ++w) {
      mine.loss += wl[w];
      mine.gb += wg[w];
      mine.pairs += wp[w];
    }
    // all-gather the CTA totals into every CTA's red[q]
    const uint32_t local = ptx::smem_u32(&red[q]);
    for (uint32_t dst = 0; dst < kRankCluster; ++dst) {
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local), "r"(dst));
      asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(mine.pairs) : "memory");
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra + 8), "d"(mine.loss) : "memory");
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra + 16), "d"(mine.gb) : "memory");
    }
  }
  rank_stamp(4);
  ptx::cluster_sync();
  rank_stamp(5);
  long long P = 0;
  double L = 0.0, G = 0.0;
  for (int b = 0; b < kRankCluster; ++b) {  // CTA order
    P += red[b].pairs;
    L += red[b].loss;
    G += red[b].gb;
  }
  const double inv = P > 0 ? 1.0 / double(P) : 0.0;
  if (seg != nullptr) {
    // warp per program: its statement rows are contiguous
    const int wid = t >> 5, ln = t & 31, nw = int(blockDim.x >> 5);
    for (int k = wid; k < int(p1 - p0); k += nw) {
      const float a = P > 0 ? float(row_g[k] * inv) : 0.f;
      for (long long r = sseg[k] + ln; r < sseg[k + 1]; r += 32) {
        coefA[r] = a;
        coefB[r] = 0.f;
      }
    }
    if (q == kRankCluster - 1)
      for (long long r = seg[n] + t; r < R; r += blockDim.x) {
        coefA[r] = 0.f;
        coefB[r] = 0.f;
      }
  } else {
    for (long long r = p0 + t; r < p1; r += blockDim.x) {
      coefA[r] = P > 0 ? float(row_g[r - p0] * inv) : 0.f;
      coefB[r] = 0.f;
    }
  }
  rank_stamp(6);
  if (q == 0 && t == 0) {
    *loss_out = P > 0 ? L * inv : 0.0;
    *pairs_out = P;
    if (gb_out != nullptr) *gb_out = P > 0 ? float(G * inv) : 0.f;
  }
}

// ---------------------------------------------------------------- fused ranking step, grid form
// For batches past the cluster form's limits (n > ~1.4K programs). Every CTA of a plain grid (up
// to one per SM) recomputes all n scores itself (reading the head partials from L2, no
// all-gather), evaluates the pairs of its rows_per_cta
// programs with the same (split, row) items and float partials as rank_pairs_kernel, and writes
// per-row sums (split order, double) to global; the last CTA to finish (self re-arming ticket)
// reduces the rows in row order and writes loss, pair count, head-bias gradient and every
// statement row's backward coefficient. Deterministic and independent of the grid size.
// Every score of the batch into shared memory ss[n] (rank_grid_kernel / rank_sym_kernel prologue):
// fixed tile order per statement row, then the segment sum (score_of()'s arithmetic); loads are
// issued 4 rows x 8 tiles at a time (one L2 round trip for ~2K rows). Pooled: srow[R] / sseg[n+1].
__device__ __forceinline__ void rank_all_scores(const float* __restrict__ part, int ntiles, long long ld, float hb,
                                                const long long* __restrict__ seg, long long n, float* ss, float* srow,
                                                long long* sseg) {
  const int t = threadIdx.x;
  auto row_dot = [&](long long r, long long r1, float* dst) {
    float v[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        const long long rr = r + (long long)u * blockDim.x;
        v[u][tt] = (rr < r1 && tt < ntiles) ? __ldg(part + tt * ld + rr) : 0.f;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long rr = r + (long long)u * blockDim.x;
      if (rr >= r1) continue;
      float a = 0.f;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt)
        if (tt < ntiles) a += v[u][tt];
      for (int tt = 8; tt < ntiles; ++tt) a += __ldg(part + tt * ld + rr);
      dst[u] = a;
    }
  };
  if (seg != nullptr) {
    for (long long k = t; k <= n; k += blockDim.x) sseg[k] = seg[k];
    __syncthreads();
    const long long r0 = sseg[0], r1 = sseg[n];
    for (long long r = r0 + t; r < r1; r += 4LL * blockDim.x) {
      float d[4];
      row_dot(r, r1, d);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (r + (long long)u * blockDim.x < r1) srow[r + (long long)u * blockDim.x - r0] = d[u];
    }
    __syncthreads();
    for (long long p = t; p < n; p += blockDim.x) {
      float acc = 0.f;
      const long long e = sseg[p + 1];
      for (long long i = sseg[p]; i < e; ++i) acc += srow[i - r0];
      ss[p] = acc + hb;
    }
  } else {
    for (long long p = t; p < n; p += 4LL * blockDim.x) {
      float d[4];
      row_dot(p, n, d);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (p + (long long)u * blockDim.x < n) ss[p + (long long)u * blockDim.x] = d[u] + hb;
    }
  }
}

constexpr int kRgThreads = 512;
__global__ void __launch_bounds__(kRgThreads)
    rank_grid_kernel(const float* __restrict__ part, int ntiles, long long ld, const float* __restrict__ hbp,
                     const long long* __restrict__ seg, const int* __restrict__ seg_of_row, const float* __restrict__ y,
                     long long n, int nsplit, int rows_per_cta, float* __restrict__ s_out, long long R,
                     double* __restrict__ row_g, double* __restrict__ row_l, long long* __restrict__ row_p,
                     unsigned int* ticket, double* loss_out, long long* pairs_out, float* __restrict__ coefA,
                     float* __restrict__ coefB, float* gb_out) {
  extern __shared__ float rg_smem[];
  const int items = rows_per_cta * nsplit;
  float* ss = rg_smem;  // [n] scores
  float* sy = ss + n;   // [n] labels
  float* pg = sy + n;   // [items] per-(split, row) partials
  float* pl = pg + items;
  int* pp = reinterpret_cast<int*>(pl + items);
  float* srow = reinterpret_cast<float*>(pp + items);  // pooled: statement-row head dots [R]
  long long* sseg = reinterpret_cast<long long*>(
      (reinterpret_cast<uintptr_t>(srow + (seg ? R : 0)) + 7) & ~uintptr_t(7));  // pooled: CSR offsets [n+1]
  double* sg = reinterpret_cast<double*>(sseg + (seg ? n + 1 : 0));           // last CTA: row sums [n]
  __shared__ bool is_last;
  __shared__ double wl[kRgThreads / 32], wg[kRgThreads / 32];
  __shared__ long long wp[kRgThreads / 32];
  const int t = threadIdx.x;
  const float hb = hbp[0];
  for (long long p = t; p < n; p += blockDim.x) sy[p] = y[p];
  rank_all_scores(part, ntiles, ld, hb, seg, n, ss, srow, sseg);
  __syncthreads();
  const long long p0 = min(n, (long long)blockIdx.x * rows_per_cta);
  for (int it = t; it < items; it += blockDim.x) {  // same items / arithmetic as rank_cluster_kernel
    const int sp = it / rows_per_cta, lr = it - sp * rows_per_cta;
    const long long i = p0 + lr;
    float gs = 0.f, loss = 0.f, lp = 1.f;
    int pairs = 0;
    if (i < n) {
      const float si = ss[i], yi = sy[i];
      const long long j0 = (long long)sp * kRankChunk;
      const int cnt = int(min((long long)kRankChunk, n - j0));
#pragma unroll 4
      for (int k = 0; k < cnt; ++k) {
        const float yj = sy[j0 + k];
        const float w = float(yi > yj) - float(yi < yj);
        const float d = w * (si - ss[j0 + k]);
        const float e = ex2_ftz(fabsf(d) * -1.4426950408889634f);
        const float iv = rcp_pair(1.f + e);
        const float sig_neg = d >= 0.f ? e * iv : iv;
        gs = w != 0.f ? gs - w * sig_neg : gs;
        const bool hi = w > 0.f;
        loss += hi ? fmaxf(-d, 0.f) : 0.f;
        lp *= hi ? 1.f + e : 1.f;  // softplus terms log1p(e) as one log of their product (<= 2^32)
        pairs += hi;
      }
      loss += 0.69314718055994531f * lg2_ftz(lp);
    }
    pg[it] = gs;
    pl[it] = loss;
    pp[it] = pairs;
  }
  __syncthreads();
  for (int lr = t; lr < rows_per_cta; lr += blockDim.x) {
    const long long i = p0 + lr;
    if (i >= n) continue;
    double g = 0.0, l = 0.0;
    long long c = 0;
    for (int k = 0; k < nsplit; ++k) {
      g += pg[k * rows_per_cta + lr];
      l += pl[k * rows_per_cta + lr];
      c += pp[k * rows_per_cta + lr];
    }
    row_g[i] = g;
    row_l[i] = l;
    row_p[i] = c;
    if (s_out != nullptr) s_out[i] = ss[i];
  }
  __threadfence();
  __syncthreads();
  if (t == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // totals in row order: thread-strided (increasing rows), lane tree, warps in order
  double l_t = 0.0, g_t = 0.0;
  long long c_t = 0;
  for (long long i = t; i < n; i += blockDim.x) {
    const double gi = __ldcg(row_g + i);
    sg[i] = gi;
    l_t += __ldcg(row_l + i);
    g_t += gi;
    c_t += __ldcg(row_p + i);
  }
  for (int o = 16; o > 0; o >>= 1) {
    l_t += __shfl_down_sync(0xffffffffu, l_t, o);
    g_t += __shfl_down_sync(0xffffffffu, g_t, o);
    c_t += __shfl_down_sync(0xffffffffu, c_t, o);
  }
  if ((t & 31) == 0) {
    wl[t >> 5] = l_t;
    wg[t >> 5] = g_t;
    wp[t >> 5] = c_t;
  }
  __syncthreads();
  double L = 0.0, G = 0.0;
  long long P = 0;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) {
    L += wl[w];
    G += wg[w];
    P += wp[w];
  }
  const double inv = P > 0 ? 1.0 / double(P) : 0.0;
  if (seg != nullptr) {  // every statement row of program p carries d loss / d s_p; padding rows 0
    for (long long p = t; p < n; p += blockDim.x) {
      const float a = P > 0 ? float(sg[p] * inv) : 0.f;
      for (long long r = sseg[p]; r < sseg[p + 1]; ++r) coefA[r] = a;
    }
    for (long long r = t; r < R; r += blockDim.x) {
      coefB[r] = 0.f;
      if (r < sseg[0] || r >= sseg[n]) coefA[r] = 0.f;
    }
  } else {
    for (long long r = t; r < n; r += blockDim.x) {
      coefA[r] = P > 0 ? float(sg[r] * inv) : 0.f;
      coefB[r] = 0.f;
    }
  }
  if (t == 0) {
    *loss_out = P > 0 ? L * inv : 0.0;
    *pairs_out = P;
    if (gb_out != nullptr) *gb_out = P > 0 ? float(G * inv) : 0.f;
    *ticket = 0u;  // re-arm for the next launch (stream-ordered)
  }
}

// ---------------------------------------------------------------- fused ranking step, symmetric form
// Large batches (cfg5: n = 4096, 8.4M pairs): every unordered pair is evaluated ONCE (the grid form
// evaluates it from both rows). The upper triangle of the n x n pair matrix is cut into 32 x 32
// tiles (bi <= bj), one warp per tile at a time: lane l holds row i = 32 bi + l and at step k meets
// column j = 32 bj + ((l + k) & 31), so each of the 32 steps covers a rotated diagonal; the row term
// -w*sigma stays in the lane, the column term +w*sigma is passed by one shuffle to the lane that
// owns column j. Tile partials (32 row + 32 column floats, loss, pair count) go to global; after a
// grid barrier (cooperative launch) row block b is reduced by CTA b % grid in a fixed term order
// (row parts bj = b..nb-1, then column parts bi = 0..b), so coefficients are deterministic and
// independent of the grid size; the last CTA (ticket) sums loss (tile order) and head-bias
// gradient (CTA order). Same pair arithmetic as rank_grid_kernel (model.cpp:71-106).
constexpr int kRsThreads = 1024, kRsWarps = kRsThreads / 32;
__device__ __forceinline__ long long rs_tile_start(long long b, long long nb) { return b * nb - b * (b - 1) / 2; }
__device__ __forceinline__ void rs_grid_sync(unsigned* bar) {  // bar[0] arrivals, bar[1] generation
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g0, arrived;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(bar + 1) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar) : "memory");
    if (arrived == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      unsigned g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
      } while (g == g0);
    }
  }
  __syncthreads();
}
// The 32 steps of one pair tile (see rank_sym_kernel). DIAG: only j > i; EDGE: columns past n.
// The 32 steps of one pair tile (see rank_sym_kernel); sp[j] = (score, label). DIAG: only j > i;
// EDGE: columns past n. Ties and invalid pairs have w = 0, hence d = 0 and c = 0. The softplus terms
// log1p(e) of a lane's pairs are taken as one log of their product (32 factors in (1, 2]): 2 MUFU
// ops per pair (exp, reciprocal) instead of 3.
template <bool DIAG, bool EDGE>
__device__ __forceinline__ void rs_tile_steps(const float2* sp, float si, float yi, bool vi, int il, int jb, int n32,
                                              int lane, float& gr, float& gc, float& ls, float& pcf) {
  float lp = 1.f;
#pragma unroll 4
  for (int k = 0; k < 32; ++k) {
    const int jl = (lane + k) & 31;
    int j = jb + jl;
    bool valid = vi;
    if (EDGE) {
      valid = valid && j < n32;
      j = min(j, n32 - 1);
    }
    if (DIAG) valid = valid && jl > il;
    const float2 q = sp[j];
    float w = float(yi > q.y) - float(yi < q.y);  // +1: i is the hi row, -1: j is, 0: tie
    if (EDGE || DIAG || !vi) w = valid ? w : 0.f;
    const float d = w * (si - q.x);               // s_hi - s_lo
    const float e = ex2_ftz(fabsf(d) * -1.4426950408889634f);
    const float iv = rcp_pair(1.f + e);
    const float c = w * ((d >= 0.f ? e : 1.f) * iv);  // w * sigma(-d)
    gr -= c;
    gc += __shfl_sync(0xffffffffu, c, (lane - k) & 31);  // the term of the lane meeting column `lane`
    ls += fmaxf(-d, 0.f);
    lp *= fmaf(e, fabsf(w), 1.f);
    pcf += fabsf(w);
  }
  ls += 0.69314718055994531f * lg2_ftz(lp);
}
__global__ void __launch_bounds__(kRsThreads, 1)
    rank_sym_kernel(const float* __restrict__ part, int ntiles, long long ld, const float* __restrict__ hbp,
                    const long long* __restrict__ seg, const float* __restrict__ y, long long n,
                    float* __restrict__ s_out, long long R, float* __restrict__ rowcol, double* __restrict__ tile_loss,
                    long long* __restrict__ tile_pairs, double* __restrict__ cta_gb, long long* __restrict__ cta_pairs,
                    float* __restrict__ scores_g, unsigned* bar, double* loss_out, long long* pairs_out, float* __restrict__ coefA,
                    float* __restrict__ coefB, float* gb_out) {
  extern __shared__ float rsym_smem[];
  float2* sp = reinterpret_cast<float2*>(rsym_smem);  // [n] (score, label)
  float* ss = rsym_smem;                              // reused after the pairs: CTA partials
  __shared__ double wsum[kRsWarps][32];
  __shared__ long long wpairs[kRsWarps];
  __shared__ double red[kRsWarps];
  __shared__ long long redp[kRsWarps];
  __shared__ bool is_last;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const float hb = hbp[0];
  rank_stamp(8);
  rank_cta_stamp(0);
  // ---- every score of the batch, in every CTA (score_of()'s arithmetic: fixed tile order per statement
  // row, then the segment sum); 4 programs' tile partials in flight per thread
  for (long long p0 = t; p0 < n; p0 += 4LL * blockDim.x) {
    float acc[4];
    if (seg == nullptr) {
      float v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
          const long long p = p0 + (long long)u * blockDim.x;
          v[u][tt] = (p < n && tt < ntiles) ? __ldg(part + tt * ld + p) : 0.f;
        }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long long p = p0 + (long long)u * blockDim.x;
        float a = 0.f;
#pragma unroll
        for (int tt = 0; tt < 8; ++tt)
          if (tt < ntiles) a += v[u][tt];
        for (int tt = 8; tt < ntiles; ++tt) a += p < n ? __ldg(part + tt * ld + p) : 0.f;
        acc[u] = a;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long long p = p0 + (long long)u * blockDim.x;
        float a = 0.f;
        if (p < n)
          for (long long r = seg[p]; r < seg[p + 1]; ++r) {
            float d = 0.f;
            for (int tt = 0; tt < ntiles; ++tt) d += __ldg(part + tt * ld + r);
            a += d;
          }
        acc[u] = a;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long p = p0 + (long long)u * blockDim.x;
      if (p < n) {
        sp[p] = make_float2(acc[u] + hb, y[p]);
        if (s_out != nullptr && blockIdx.x == 0) s_out[p] = acc[u] + hb;
      }
    }
  }
  __syncthreads();
  rank_stamp(9);
  rank_cta_stamp(1);

  // ---- pair tiles
  const long long nb = (n + 31) / 32;
  const long long T = nb * (nb + 1) / 2;
  long long my_pairs = 0;
  // CTA c: tiles [c*T/G, (c+1)*T/G) (balanced per SM), its warps round-robin over them
  const long long tb0 = (long long)blockIdx.x * T / gridDim.x, tb1 = (long long)(blockIdx.x + 1) * T / gridDim.x;
  for (long long tile = tb0 + warp; tile < tb1; tile += kRsWarps) {
    const double q = double(2 * nb + 1);
    long long bi = (long long)floor((q - sqrt(q * q - 8.0 * double(tile))) * 0.5);
    bi = max(0LL, min(bi, nb - 1));
    while (bi > 0 && rs_tile_start(bi, nb) > tile) --bi;
    while (bi + 1 < nb && rs_tile_start(bi + 1, nb) <= tile) ++bi;
    const long long bj = bi + (tile - rs_tile_start(bi, nb));
    const int n32 = int(n), i = int(bi) * 32 + lane, jb = int(bj) * 32;
    const bool vi = i < n32;
    const float2 qi = sp[vi ? i : 0];
    const float si = qi.x, yi = qi.y;
    float gr = 0.f, gc = 0.f, ls = 0.f, pcf = 0.f;
    if (bi != bj && jb + 32 <= n32 && bi * 32 + 32 <= n32)
      rs_tile_steps<false, false>(sp, si, yi, true, lane, jb, n32, lane, gr, gc, ls, pcf);
    else if (bi != bj) rs_tile_steps<false, true>(sp, si, yi, vi, lane, jb, n32, lane, gr, gc, ls, pcf);
    else rs_tile_steps<true, true>(sp, si, yi, vi, lane, jb, n32, lane, gr, gc, ls, pcf);
    const int pc = int(pcf);
    rowcol[tile * 64 + lane] = gr;
    rowcol[tile * 64 + 32 + lane] = gc;
    double l = ls;
    long long pcl = pc;
    for (int o = 16; o > 0; o >>= 1) {
      l += __shfl_down_sync(0xffffffffu, l, o);
      pcl += __shfl_down_sync(0xffffffffu, pcl, o);
    }
    if (lane == 0) {
      tile_loss[tile] = l;
      tile_pairs[tile] = pcl;
      my_pairs += pcl;
    }
  }
  if (lane == 0) wpairs[warp] = my_pairs;
  __syncthreads();
  if (t == 0) {
    long long cp = 0;
    for (int w = 0; w < kRsWarps; ++w) cp += wpairs[w];
    cta_pairs[blockIdx.x] = cp;
  }
  rank_stamp(10);
  rank_cta_stamp(2);
  rs_grid_sync(bar);
  rank_stamp(11);
  rank_cta_stamp(3);

  // ---- total pair count (integers: any order), then this CTA's row blocks
  // every CTA's pair count loaded once per thread in parallel (integers: any order), block-reduced
  long long pl = 0;
  for (int b = t; b < int(gridDim.x); b += blockDim.x) pl += __ldcg(cta_pairs + b);
  for (int o = 16; o > 0; o >>= 1) pl += __shfl_down_sync(0xffffffffu, pl, o);
  if (lane == 0) redp[warp] = pl;
  __syncthreads();
  long long P = 0;
  for (int w = 0; w < kRsWarps; ++w) P += redp[w];
  const double inv = P > 0 ? 1.0 / double(P) : 0.0;
  double gb_local = 0.0;  // sum of this CTA's rows' gs (row-block order, then rows)
  for (long long b = blockIdx.x; b < nb; b += gridDim.x) {
    // nb + 1 terms: row parts of tiles (b, bj), bj = b..nb-1, then column parts of (bi, b), bi = 0..b;
    // warp w takes a contiguous run of them, the runs are added in warp order
    const long long terms = nb + 1, per = (terms + kRsWarps - 1) / kRsWarps;
    const long long q0 = warp * per, q1 = min(terms, q0 + per);
    double acc = 0.0;
    const long long rows_n = nb - b;
    for (long long qa = q0; qa < q1; qa += 8) {  // 8 loads in flight, added in term order
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long long qq = qa + u;
        v[u] = qq >= q1 ? 0.f
               : qq < rows_n ? __ldcg(rowcol + (rs_tile_start(b, nb) + qq) * 64 + lane)
                             : __ldcg(rowcol + (rs_tile_start(qq - rows_n, nb) + (b - (qq - rows_n))) * 64 + 32 + lane);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (qa + u < q1) acc += double(v[u]);
    }
    wsum[warp][lane] = acc;
    __syncthreads();
    if (warp == 0) {
      double g = 0.0;
      for (int w = 0; w < kRsWarps; ++w) g += wsum[w][lane];
      const long long i = b * 32 + lane;
      if (i < n) {
        const float a = P > 0 ? float(g * inv) : 0.f;
        if (seg != nullptr) {
          for (long long r = seg[i]; r < seg[i + 1]; ++r) {
            coefA[r] = a;
            coefB[r] = 0.f;
          }
        } else {
          coefA[i] = a;
          coefB[i] = 0.f;
        }
        gb_local += g;
      }
    }
    __syncthreads();
  }
  if (seg != nullptr)  // padding statement rows outside the programs
    for (long long r = (long long)blockIdx.x * blockDim.x + t; r < R; r += (long long)gridDim.x * blockDim.x)
      if (r < seg[0] || r >= seg[n]) {
        coefA[r] = 0.f;
        coefB[r] = 0.f;
      }
  if (warp == 0) {
    for (int o = 16; o > 0; o >>= 1) gb_local += __shfl_down_sync(0xffffffffu, gb_local, o);
    if (lane == 0) cta_gb[blockIdx.x] = gb_local;
  }
  __threadfence();
  __syncthreads();
  rank_stamp(12);
  rank_cta_stamp(4);
  if (t == 0) is_last = atomicAdd(bar + 2, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // loss in tile order (thread-strided, lane tree, warps in order); head-bias gradient in CTA order
  double l_t = 0.0;
  for (long long k = t; k < T; k += blockDim.x) l_t += __ldcg(tile_loss + k);
  for (int o = 16; o > 0; o >>= 1) l_t += __shfl_down_sync(0xffffffffu, l_t, o);
  if (lane == 0) red[warp] = l_t;
  __syncthreads();
  double* sgb = reinterpret_cast<double*>(ss);  // scores no longer needed: CTA partials staged in order
  for (int b = t; b < int(gridDim.x); b += blockDim.x) sgb[b] = __ldcg(cta_gb + b);
  __syncthreads();
  if (t == 0) {
    double L = 0.0, G = 0.0;
    for (int w = 0; w < kRsWarps; ++w) L += red[w];
    for (int b = 0; b < int(gridDim.x); ++b) G += sgb[b];
    *loss_out = P > 0 ? L * inv : 0.0;
    *pairs_out = P;
    if (gb_out != nullptr) *gb_out = P > 0 ? float(G * inv) : 0.f;
    bar[2] = 0u;  // re-arm for the next launch (stream-ordered)
  }
}

template <typename T>
__global__ void head_backward_kernel(const float* __restrict__ coefA, const float* __restrict__ coefB,
                                     const float* __restrict__ wh, const float* __restrict__ u, const T* __restrict__ H,
                                     long long ldh, long long R, int W, T* __restrict__ dz, long long ldz,
                                     T* __restrict__ dz_lo, const float* __restrict__ extra, float extra_scale) {
  ptx::pdl_launch_dependents();
  const long long total = R * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / W;
    const int j = int(i - r * W);
    float v = coefA[r] * wh[j];
    if (u != nullptr) v += coefB[r] * u[j];
    if (extra != nullptr) v += extra_scale * extra[i];  // d(beta * MMD^2)/dH (row-major R x W)
    store_operand(dz, dz_lo, r * ldz + j, to_f(H[r * ldh + j]) > 0.f ? v : 0.f);
  }
}

// bf16 fast path (W % 8 == 0, 16-B aligned rows): 8 columns per thread, one 16-B load of H and one
// 16-B store of dz, no per-element index division. Same per-element arithmetic as above.
__global__ void __launch_bounds__(256) head_backward_bf16x8_kernel(const float* __restrict__ coefA,
                                                                   const float* __restrict__ coefB,
                                                                   const float* __restrict__ wh,
                                                                   const float* __restrict__ u,
                                                                   const __nv_bfloat16* __restrict__ H, long long ldh,
                                                                   long long R, int W, __nv_bfloat16* __restrict__ dz,
                                                                   long long ldz, __nv_bfloat16* __restrict__ dz_lo) {
  ptx::pdl_launch_dependents();
  ptx::pdl_wait();  // programmatic launch behind the ranking step: coefA is its output
  const int groups = W / 8;
  const long long total = R * groups;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / groups;  // one 64-bit division per 8 elements
    const int j0 = int(i - r * groups) * 8;
    const uint4 hv = __ldg(reinterpret_cast<const uint4*>(H + r * ldh + j0));
    const float a = coefA[r];
    const float b = u != nullptr ? coefB[r] : 0.f;
    const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&hv);
    uint4 out, outl;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&out);
    __nv_bfloat16* ol = reinterpret_cast<__nv_bfloat16*>(&outl);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float v = a * __ldg(wh + j0 + k);
      if (u != nullptr) v += b * __ldg(u + j0 + k);
      v = __bfloat162float(hb[k]) > 0.f ? v : 0.f;
      ob[k] = __float2bfloat16_rn(v);
      ol[k] = __float2bfloat16_rn(v - __bfloat162float(ob[k]));  // split bf16: lo = rn(v - hi)
    }
    *reinterpret_cast<uint4*>(dz + r * ldz + j0) = out;
    if (dz_lo != nullptr) *reinterpret_cast<uint4*>(dz_lo + r * ldz + j0) = outl;
  }
}

// g[j] = sum_r coef[r] * H[r][j]; g[W] = sum_r coef[r]. Pass 1: block (32 columns x 8 row-lanes) over a
// 64-row slab -> partial[slab][j]; pass 2 sums the slabs in order. Deterministic.
constexpr int kColSlab = 64;
template <typename T>
__global__ void column_dot_kernel(const float* __restrict__ coef, const T* __restrict__ H, long long ldh, long long R, int W,
                                  float* __restrict__ part, const T* __restrict__ H_lo = nullptr) {
  __shared__ float red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  const long long r0 = (long long)blockIdx.y * kColSlab, r1 = min(R, r0 + kColSlab);
  float acc = 0.f;
  if (j < W)
    for (long long r = r0 + ty; r < r1; r += 8) acc = fmaf(coef[r], load_operand(H, H_lo, r * ldh + j), acc);
  else if (j == W)
    for (long long r = r0 + ty; r < r1; r += 8) acc += coef[r];
  red[ty][tx] = acc;
  __syncthreads();
  if (ty == 0 && j <= W) {
    float s = red[0][tx];
    for (int k = 1; k < 8; ++k) s += red[k][tx];
    part[(long long)blockIdx.y * (W + 1) + j] = s;
  }
}
__global__ void column_sum_kernel(const float* __restrict__ part, int slabs, int W1, float* __restrict__ g,
                                  const float* __restrict__ last_override) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < W1; j += gridDim.x * blockDim.x) {
    if (last_override != nullptr && j == W1 - 1) {
      g[j] = *last_override;
      continue;
    }
    float s = 0.f;
    for (int q = 0; q < slabs; ++q) s += part[(long long)q * W1 + j];
    g[j] = s;
  }
}

// ---------------------------------------------------------------- updates (no FMA contraction: reference
// is built with -ffp-contract=off, so v = mu*v + g and w -= lr*v round after every op)
template <bool MOM, bool MASK, int SHADOW>
__global__ void sgd_kernel(float* __restrict__ w, float* __restrict__ v, const float* __restrict__ g,
                           const uint8_t* __restrict__ mask, long long P, float lr, float mu, void* __restrict__ shadow,
                           long long lo_off) {
  ptx::pdl_launch_dependents();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P; i += (long long)gridDim.x * blockDim.x) {
    float wi = w[i];
    if (!MASK || mask[i]) {
      if (MOM) {
        const float vi = __fadd_rn(__fmul_rn(mu, v[i]), g[i]);
        v[i] = vi;
        wi = __fsub_rn(wi, __fmul_rn(lr, vi));
      } else {
        wi = __fsub_rn(wi, __fmul_rn(lr, g[i]));
      }
      w[i] = wi;
    }
    store_shadow<SHADOW>(shadow, i, wi, lo_off);
  }
}

// Vectorised form of sgd_kernel (same per-element arithmetic): 16-byte lanes for w / v / g, 4-byte mask
// words, 8-byte bf16 shadow stores; two float4 per thread per iteration in flight. Requires 16-byte
// aligned w, v, g (4-byte mask, 8-byte shadow); the P % 4 tail runs scalar.
template <bool MOM, bool MASK, int SHADOW>
__global__ void __launch_bounds__(256) sgd4_kernel(float* __restrict__ w, float* __restrict__ v,
                                                   const float* __restrict__ g, const uint8_t* __restrict__ mask,
                                                   long long P, float lr, float mu, void* __restrict__ shadow,
                                                   long long lo_off) {
  ptx::pdl_launch_dependents();
  const long long n4 = P >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  auto one = [&](float& wi, float& vi, float gi, bool on) {
    if (!on) return;
    if (MOM) {
      vi = __fadd_rn(__fmul_rn(mu, vi), gi);
      wi = __fsub_rn(wi, __fmul_rn(lr, vi));
    } else {
      wi = __fsub_rn(wi, __fmul_rn(lr, gi));
    }
  };
  auto put_shadow4 = [&](long long i4, const float4& x) {
    if constexpr (SHADOW == 1 || SHADOW == 4) {
      const __nv_bfloat162 a = __floats2bfloat162_rn(x.x, x.y), b = __floats2bfloat162_rn(x.z, x.w);
      uint2 u;
      u.x = *reinterpret_cast<const uint32_t*>(&a);
      u.y = *reinterpret_cast<const uint32_t*>(&b);
      reinterpret_cast<uint2*>(shadow)[i4] = u;
      if constexpr (SHADOW == 4) {
        const __nv_bfloat162 la = __floats2bfloat162_rn(x.x - __low2float(a), x.y - __high2float(a));
        const __nv_bfloat162 lb = __floats2bfloat162_rn(x.z - __low2float(b), x.w - __high2float(b));
        uint2 ul;
        ul.x = *reinterpret_cast<const uint32_t*>(&la);
        ul.y = *reinterpret_cast<const uint32_t*>(&lb);
        reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(shadow) + lo_off)[i4] = ul;
      }
    }
    if constexpr (SHADOW == 2)
      reinterpret_cast<float4*>(shadow)[i4] = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
  };
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < n4; base += 2 * stride) {
    float4 wv[2], vv[2], gv[2];
    uchar4 mk[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long i4 = base + u * stride;
      ok[u] = i4 < n4;
      if (!ok[u]) continue;
      wv[u] = reinterpret_cast<const float4*>(w)[i4];
      gv[u] = reinterpret_cast<const float4*>(g)[i4];
      if (MOM) vv[u] = reinterpret_cast<const float4*>(v)[i4];
      mk[u] = MASK ? reinterpret_cast<const uchar4*>(mask)[i4] : make_uchar4(1, 1, 1, 1);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!ok[u]) continue;
      const long long i4 = base + u * stride;
      float4 x = wv[u], y = MOM ? vv[u] : make_float4(0.f, 0.f, 0.f, 0.f);
      one(x.x, y.x, gv[u].x, mk[u].x != 0);
      one(x.y, y.y, gv[u].y, mk[u].y != 0);
      one(x.z, y.z, gv[u].z, mk[u].z != 0);
      one(x.w, y.w, gv[u].w, mk[u].w != 0);
      reinterpret_cast<float4*>(w)[i4] = x;
      if (MOM) reinterpret_cast<float4*>(v)[i4] = y;
      put_shadow4(i4, x);
    }
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P; i += stride) {
    float wi = w[i], vi = MOM ? v[i] : 0.f;
    one(wi, vi, g[i], !MASK || mask[i]);
    w[i] = wi;
    if (MOM) v[i] = vi;
    store_shadow<SHADOW>(shadow, i, wi, lo_off);
  }
}

template <int SHADOW>
__global__ void adam_kernel(float* __restrict__ w, float* __restrict__ m1, float* __restrict__ m2, const float* __restrict__ g,
                            const uint8_t* __restrict__ mask, long long P, float lr, float b1, float b2, float eps,
                            float c1, float c2, void* __restrict__ shadow) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P; i += (long long)gridDim.x * blockDim.x) {
    float wi = w[i];
    if (mask == nullptr || mask[i]) {
      const float gi = g[i];
      const float a = __fadd_rn(__fmul_rn(b1, m1[i]), __fmul_rn(__fsub_rn(1.f, b1), gi));
      const float b = __fadd_rn(__fmul_rn(b2, m2[i]), __fmul_rn(__fsub_rn(1.f, b2), __fmul_rn(gi, gi)));
      m1[i] = a;
      m2[i] = b;
      const float mh = __fdiv_rn(a, c1);
      const float vh = __fdiv_rn(b, c2);
      wi = __fsub_rn(wi, __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), eps)));
      w[i] = wi;
    }
    store_shadow<SHADOW>(shadow, i, wi);
  }
}

template <int SHADOW>
__global__ void decay_kernel(float* __restrict__ w, const uint8_t* __restrict__ mask, long long P, float factor,
                             void* __restrict__ shadow) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P; i += (long long)gridDim.x * blockDim.x) {
    float wi = w[i];
    if (!mask[i]) {
      wi = __fmul_rn(wi, factor);
      w[i] = wi;
    }
    store_shadow<SHADOW>(shadow, i, wi);
  }
}

// ---------------------------------------------------------------- radix select (top `need` keys, ties by index)
// Three MSB-first passes over u32 keys (11, 11, 10 bits). State in device memory.
struct SelState {
  unsigned prefix, pmask;
  unsigned long long need;  // still to take among keys matching the prefix
  unsigned long long gt;    // keys strictly above the current prefix range
  unsigned digit;           // digit chosen in the last pass
  unsigned max_bits;        // threshold mode: max xi bits
  unsigned long long count; // popcount accumulator
};
constexpr int kSelBlock = 256;
constexpr int kBins = 2048;
constexpr int kPassShift[3] = {21, 10, 0};
constexpr int kPassBits[3] = {11, 11, 10};

__device__ __forceinline__ unsigned float_key_desc(float f) {  // orderable: larger float -> larger key
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

struct Chunk {
  long long lo, hi;
};
__device__ __forceinline__ Chunk block_chunk(long long n, long long chunk) {
  const long long lo = (long long)blockIdx.x * chunk;
  return {lo, min(n, lo + chunk)};
}

// MODE 0: keys given; MODE 1: keys = bits(|w*g|) (xi), also atomicMax of bits; MODE 2: keys = float_key_desc(score)
template <int MODE, bool BLOCK_HIST>
__global__ void __launch_bounds__(kSelBlock) radix_hist_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                               unsigned* __restrict__ keys, float* __restrict__ xi_out,
                                                               long long n, long long chunk, SelState* st, int shift,
                                                               int bits, unsigned* __restrict__ hist,
                                                               unsigned* __restrict__ block_hist) {
  __shared__ unsigned sh[kBins];
  const int nb = 1 << bits;
  for (int d = threadIdx.x; d < nb; d += kSelBlock) sh[d] = 0;
  __syncthreads();
  const unsigned prefix = st->prefix, pmask = st->pmask;
  const Chunk ch = block_chunk(n, chunk);
  unsigned local_max = 0;
  for (long long i = ch.lo + threadIdx.x; i < ch.hi; i += kSelBlock) {
    unsigned key;
    if constexpr (MODE == 1) {
      const float x = fabsf(__fmul_rn(a[i], b[i]));
      key = __float_as_uint(x);
      keys[i] = key;
      if (xi_out) xi_out[i] = x;
      local_max = max(local_max, key);
    } else if constexpr (MODE == 2) {
      key = float_key_desc(a[i]);
      keys[i] = key;
    } else {
      key = keys[i];
    }
    if ((key & pmask) == prefix) atomicAdd(&sh[(key >> shift) & (nb - 1)], 1u);
  }
  if constexpr (MODE == 1) {
    for (int o = 16; o; o >>= 1) local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
    if ((threadIdx.x & 31) == 0 && local_max) atomicMax(&st->max_bits, local_max);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nb; d += kSelBlock) {
    const unsigned v = sh[d];
    if (v) atomicAdd(&hist[d], v);
    if (BLOCK_HIST) block_hist[(long long)blockIdx.x * kBins + d] = v;
  }
}

constexpr int kPickBlock = 1024;
__global__ void __launch_bounds__(kPickBlock) radix_pick_kernel(SelState* st, unsigned* hist, int shift, int bits) {
  using Scan = cub::BlockScan<unsigned long long, kPickBlock>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long suffix[kBins + 1];
  const int nb = 1 << bits;
  // suffix[d] = count of digits >= d. Thread t owns digits (nb-1-2t, nb-2-2t) in descending order.
  const int per = (nb + kPickBlock - 1) / kPickBlock;
  unsigned long long vals[2] = {0, 0};
  unsigned long long local = 0;
  for (int q = 0; q < per; ++q) {
    const int d = nb - 1 - (threadIdx.x * per + q);
    vals[q] = d >= 0 ? hist[d] : 0;
    local += vals[q];
  }
  unsigned long long excl;
  Scan(tmp).ExclusiveSum(local, excl);
  unsigned long long run = excl;
  for (int q = 0; q < per; ++q) {
    const int d = nb - 1 - (threadIdx.x * per + q);
    run += vals[q];
    if (d >= 0) suffix[d] = run;
  }
  if (threadIdx.x == 0) suffix[nb] = 0;
  __syncthreads();
  const unsigned long long need = st->need;
  // the chosen digit d* is the largest d with suffix[d] >= need (suffix is non-increasing in d)
  for (int d = threadIdx.x; d < nb; d += kPickBlock) {
    if (suffix[d] >= need && suffix[d + 1] < need) {
      st->digit = unsigned(d);
      st->need = need - suffix[d + 1];
      st->gt += suffix[d + 1];
      st->prefix |= unsigned(d) << shift;
      st->pmask |= unsigned(nb - 1) << shift;
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nb; d += kPickBlock) hist[d] = 0;
}

__global__ void sel_init_kernel(SelState* st, unsigned long long need, unsigned* hist) {
  if (threadIdx.x == 0) {
    st->prefix = 0;
    st->pmask = 0;
    st->need = need;
    st->gt = 0;
    st->digit = 0;
    st->max_bits = 0;
    st->count = 0;
  }
  for (int d = threadIdx.x; d < kBins; d += blockDim.x) hist[d] = 0;
}

// Block-contiguous final pass: kept = key > T || (key == T && rank_among_equal < need).
// ACTION 0: write mask byte; 1: compact (key, idx) for top-k.
template <int ACTION>
__global__ void __launch_bounds__(kSelBlock) radix_apply_kernel(const unsigned* __restrict__ keys, long long n,
                                                                long long chunk, const SelState* st,
                                                                const unsigned* __restrict__ block_hist,
                                                                uint8_t* __restrict__ mask, unsigned* out_key,
                                                                long long* out_idx, unsigned long long* counter) {
  using Scan = cub::BlockScan<unsigned, kSelBlock>;
  using Red = cub::BlockReduce<unsigned long long, kSelBlock>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ typename Red::TempStorage rtmp;
  __shared__ unsigned long long sh_base;
  const unsigned T = st->prefix;
  const unsigned long long need = st->need;
  const unsigned digit = st->digit;
  // equal keys in earlier blocks (last pass histogram of block b' at digit d* counts keys == T)
  unsigned long long before = 0;
  for (int b = threadIdx.x; b < blockIdx.x; b += kSelBlock) before += block_hist[(long long)b * kBins + digit];
  before = Red(rtmp).Sum(before);
  if (threadIdx.x == 0) sh_base = before;
  __syncthreads();
  unsigned long long base = sh_base;
  const Chunk ch = block_chunk(n, chunk);
  for (long long t0 = ch.lo; t0 < ch.hi; t0 += kSelBlock) {
    const long long i = t0 + threadIdx.x;
    const bool valid = i < ch.hi;
    const unsigned key = valid ? keys[i] : 0u;
    const unsigned eq = (valid && key == T) ? 1u : 0u;
    unsigned rank, tot;
    Scan(tmp).ExclusiveSum(eq, rank, tot);
    __syncthreads();
    const bool kept = valid && (key > T || (eq && base + rank < need));
    if (valid) {
      if constexpr (ACTION == 0) {
        mask[i] = kept ? 1 : 0;
      } else {
        if (kept) {
          const unsigned long long pos = atomicAdd(counter, 1ull);
          out_key[pos] = key;
          out_idx[pos] = i;
        }
      }
    }
    base += tot;
  }
}

// Threshold mode (normalised xi strictly above theta, lottery.cpp:152-157); also counts kept scalars.
__global__ void __launch_bounds__(kSelBlock) threshold_mask_kernel(const unsigned* __restrict__ keys, long long n,
                                                                   SelState* st, float theta, bool normalize,
                                                                   uint8_t* __restrict__ mask, float* xi_norm) {
  using Red = cub::BlockReduce<unsigned long long, kSelBlock>;
  __shared__ typename Red::TempStorage rtmp;
  const float top = __uint_as_float(st->max_bits);
  unsigned long long cnt = 0;
  for (long long i = blockIdx.x * (long long)kSelBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kSelBlock) {
    float x = __uint_as_float(keys[i]);
    if (normalize && top > 0.f) x = __fdiv_rn(x, top);
    if (xi_norm) xi_norm[i] = x;
    const bool kept = x > theta;
    if (mask) mask[i] = kept;
    cnt += kept;
  }
  cnt = Red(rtmp).Sum(cnt);
  if (threadIdx.x == 0 && cnt) atomicAdd(&st->count, cnt);
}

__global__ void xi_normalize_kernel(float* xi, long long n, const SelState* st) {
  const float top = __uint_as_float(st->max_bits);
  if (!(top > 0.f)) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    xi[i] = __fdiv_rn(xi[i], top);
}

// Fused transferable step + variant decay on the mask (lottery.cpp:92-120):
//   kept:   w -= alpha * g     (apply_update, no momentum)
//   else:   w *= (1 - alpha*lambda)
template <int SHADOW>
__global__ void lottery_apply_kernel(float* __restrict__ w, const float* __restrict__ g, const uint8_t* __restrict__ mask,
                                     long long n, float alpha, float factor, bool step, bool decay,
                                     void* __restrict__ shadow) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float wi = w[i];
    if (mask[i]) {
      if (step) wi = __fsub_rn(wi, __fmul_rn(alpha, g[i]));
    } else if (decay) {
      wi = __fmul_rn(wi, factor);
    }
    w[i] = wi;
    store_shadow<SHADOW>(shadow, i, wi);
  }
}

__global__ void shadow_kernel1(const float* w, long long n, void* sh) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    store_shadow<1>(sh, i, w[i]);
}
__global__ void shadow_kernel2(const float* w, long long n, void* sh) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    store_shadow<2>(sh, i, w[i]);
}
// kind 3 (3xTF32): hi at sh[i], lo at sh[shadow_lo_offset(n) + i]
__global__ void shadow_kernel3(const float* w, long long n, float* sh) {
  float* lo = sh + shadow_lo_offset(n);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    store_operand(sh, lo, i, w[i]);
}

// kind 4 (split bf16): hi at sh[i], lo at sh[i + lo_off]
__global__ void shadow_kernel4(const float* w, long long n, __nv_bfloat16* sh, long long lo_off) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    store_shadow<4>(sh, i, w[i], lo_off);
}

__global__ void popcount_kernel(const uint8_t* __restrict__ mask, long long n, unsigned long long* out) {
  using Red = cub::BlockReduce<unsigned long long, kSelBlock>;
  __shared__ typename Red::TempStorage rtmp;
  unsigned long long c = 0;
  for (long long i = blockIdx.x * (long long)kSelBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kSelBlock) c += mask[i] != 0;
  c = Red(rtmp).Sum(c);
  if (threadIdx.x == 0 && c) atomicAdd(out, c);
}

// Top-k: bitonic sort of the compacted winners by (key desc, index asc), one block.
constexpr int kSortBlock = 1024;
__global__ void __launch_bounds__(kSortBlock) topk_sort_kernel(unsigned* keys, long long* idx, const unsigned long long* count,
                                                               long long k) {
  __shared__ unsigned sk[kTopkMax];
  __shared__ long long si[kTopkMax];
  const int cnt = int(*count);
  int np = 1;
  while (np < cnt) np <<= 1;
  for (int t = threadIdx.x; t < np; t += kSortBlock) {
    sk[t] = t < cnt ? keys[t] : 0u;
    si[t] = t < cnt ? idx[t] : 0x7fffffffffffffffll;
  }
  __syncthreads();
  for (int size = 2; size <= np; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < np; t += kSortBlock) {
        const int o = t ^ stride;
        if (o > t) {
          const bool desc_block = (t & size) == 0;  // first half ordered "before"
          const bool t_before_o = sk[t] > sk[o] || (sk[t] == sk[o] && si[t] < si[o]);
          if (t_before_o != desc_block) {
            const unsigned a = sk[t]; sk[t] = sk[o]; sk[o] = a;
            const long long b = si[t]; si[t] = si[o]; si[o] = b;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < k && t < cnt; t += kSortBlock) {
    keys[t] = sk[t];
    idx[t] = si[t];
  }
}

// ---------------------------------------------------------------- accuracy (model.cpp:298-312)
__global__ void accuracy_kernel(const float* __restrict__ s, const float* __restrict__ y, const long long* __restrict__ seg_of_row,
                                const long long* __restrict__ seg_off, long long n, unsigned long long* totals) {
  using Red = cub::BlockReduce<unsigned long long, 256>;
  __shared__ typename Red::TempStorage rtmp;
  unsigned long long p = 0, c = 0;
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const long long sg = seg_of_row[i];
    const long long lo = seg_off[sg], hi = seg_off[sg + 1];
    const float yi = y[i], si = s[i];
    for (long long j = lo; j < hi; ++j) {
      if (yi <= y[j]) continue;
      ++p;
      if (si > s[j]) ++c;
    }
  }
  p = Red(rtmp).Sum(p);
  __syncthreads();
  c = Red(rtmp).Sum(c);
  if (threadIdx.x == 0) {
    if (p) atomicAdd(&totals[0], p);
    if (c) atomicAdd(&totals[1], c);
  }
}

// ---------------------------------------------------------------- adversary (lottery.cpp:135-164)
__global__ void __launch_bounds__(kFinBlock) adv_logits_kernel(const float* part2, int ntiles, long long ld2, long long m,
                                                               long long n, const float* c, float* dz, double* loss_out,
                                                               double* dc_out) {
  using BR = cub::BlockReduce<double, kFinBlock>;
  __shared__ typename BR::TempStorage tmp;
  const long long R = m + n;
  double ls = 0.0, lt = 0.0, dcs = 0.0, dct = 0.0;
  for (long long r = threadIdx.x; r < R; r += kFinBlock) {
    float z = 0.f;
    for (int t = 0; t < ntiles; ++t) z += part2[t * ld2 + r];
    z += c[0];
    float d;
    if (r < m) {
      d = float(-0.5 * double(stable_sigmoid(-z)) / double(m));
      ls += softplus_d(-double(z));
      dcs += d;
    } else {
      d = float(0.5 * double(stable_sigmoid(z)) / double(n));
      lt += softplus_d(double(z));
      dct += d;
    }
    dz[r] = d;
  }
  const double a = BR(tmp).Sum(ls);
  __syncthreads();
  const double b = BR(tmp).Sum(lt);
  __syncthreads();
  const double e = BR(tmp).Sum(dcs);
  __syncthreads();
  const double f = BR(tmp).Sum(dct);
  if (threadIdx.x == 0) {
    *loss_out = 0.5 * (a / double(m) + b / double(n));
    *dc_out = e + f;
  }
}
__global__ void __launch_bounds__(kFinBlock) disc_ce_kernel(const double* z, long long m, long long n, double* out) {
  using BR = cub::BlockReduce<double, kFinBlock>;
  __shared__ typename BR::TempStorage tmp;
  double ls = 0.0, lt = 0.0;
  for (long long r = threadIdx.x; r < m + n; r += kFinBlock) {
    if (r < m) ls += softplus_d(-z[r]);
    else lt += softplus_d(z[r]);
  }
  const double a = BR(tmp).Sum(ls);
  __syncthreads();
  const double b = BR(tmp).Sum(lt);
  if (threadIdx.x == 0) *out = 0.5 * (a / double(m) + b / double(n));
}
__global__ void adv_update_kernel(float* u, float* c, const float* du, int W, float eta, const double* dc) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < W; j += gridDim.x * blockDim.x)
    u[j] = __fsub_rn(u[j], __fmul_rn(eta, du[j]));
  if (blockIdx.x == 0 && threadIdx.x == 0) c[0] = __fsub_rn(c[0], __fmul_rn(eta, float(*dc)));
}

// ---------------------------------------------------------------- segment-sum pooling (CSR), one warp per program
template <typename T>
__global__ void segment_sum_kernel(const T* __restrict__ H, long long ldh, int W, const long long* __restrict__ off,
                                   long long programs, float* __restrict__ out, long long ldo) {
  constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
  const long long warp_global = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long p = warp_global; p < programs; p += nwarps) {
    const long long lo = off[p], hi = off[p + 1];
    for (int j0 = lane * V; j0 < W; j0 += 32 * V) {
      float acc[V];
#pragma unroll
      for (int q = 0; q < V; ++q) acc[q] = 0.f;
      for (long long r = lo; r < hi; ++r) {
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(H + r * ldh + j0));
        const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] += to_f(e[q]);
      }
      float* o = out + p * ldo + j0;
#pragma unroll
      for (int q = 0; q < V; q += 4) *reinterpret_cast<float4*>(o + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
    }
  }
}
__global__ void segment_sum_scalar_kernel(const float* __restrict__ v, const long long* __restrict__ off, long long programs,
                                          float bias, float* __restrict__ out) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < programs; p += (long long)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (long long r = off[p]; r < off[p + 1]; ++r) acc += v[r];
    out[p] = acc + bias;
  }
}


// ---------------------------------------------------------------- synthetic data
__device__ __forceinline__ unsigned long long fnv_u64(unsigned long long h, unsigned long long v) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xffull;
    h *= 0x100000001b3ull;
  }
  return h;
}
template <int N>
__device__ __forceinline__ unsigned long long fnv_str(unsigned long long h, const char (&s)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {  // includes the terminating NUL, like KeyBuilder::add(string_view)
    h ^= (unsigned char)s[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
__device__ __forceinline__ unsigned long long splitmix_at(unsigned long long key, unsigned long long k) {
  unsigned long long z = key + k * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u01(unsigned long long bits) { return double(bits >> 11) * 0x1.0p-53; }

template <typename T>
__global__ void synth_features_kernel(unsigned long long seed, long long row0, long long n, int D, T* dst, long long ld) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    unsigned long long key = fnv_u64(0xcbf29ce484222325ull, seed);
    key = fnv_str(key, "feat");
    key = fnv_u64(key, (unsigned long long)(row0 + r));
    T* row = dst + r * ld;
    for (int c = 0; c < ld; ++c) {
      const float v = c < D ? float(u01(splitmix_at(key, (unsigned long long)c + 1))) : (c == D ? 1.f : 0.f);
      if constexpr (sizeof(T) == 4) row[c] = v;  // bit-identical to the oracle generator
      else row[c] = from_f<T>(v);
    }
  }
}
__global__ void synth_labels_kernel(unsigned long long seed, long long row0, long long n, float* dst) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    unsigned long long key = fnv_u64(0xcbf29ce484222325ull, seed);
    key = fnv_str(key, "label");
    key = fnv_u64(key, (unsigned long long)(row0 + r));
    dst[r] = float(0.1 + u01(splitmix_at(key, 1)));
  }
}

}  // namespace

// ====================================================================== host wrappers
template <typename T>
void pack_rows(const double* src, long long n, int D, T* dst, long long ld, cudaStream_t s, T* lo) {
  if (n <= 0) return;
  pack_rows_kernel<T><<<grid_for(n * ld, 256), 256, 0, s>>>(src, n, D, dst, ld, lo);
  MOSES_CUDA(cudaGetLastError());
}
template <typename T>
void pack_rows_f32(const float* src, long long n, int D, long long lds, T* dst, long long ld, cudaStream_t s, T* lo) {
  if (n <= 0) return;
  pack_rows_f32_kernel<T><<<grid_for(n * ld, 256), 256, 0, s>>>(src, n, D, lds, dst, ld, lo);
  MOSES_CUDA(cudaGetLastError());
}
template <typename T>
void set_ones_column(T* act, long long rows, int col, long long ld, cudaStream_t s) {
  if (rows <= 0) return;
  set_col_kernel<T><<<grid_for(rows, 256), 256, 0, s>>>(act, rows, col, ld);
  MOSES_CUDA(cudaGetLastError());
}
template <typename T>
void unpack_rows(const T* src, long long n, int W, long long ld, double* dst, cudaStream_t s, const T* lo) {
  if (n <= 0) return;
  unpack_rows_kernel<T><<<grid_for(n * W, 256), 256, 0, s>>>(src, n, W, ld, dst, lo);
  MOSES_CUDA(cudaGetLastError());
}
void f32_to_f64(const float* src, long long n, double* dst, cudaStream_t s) {
  if (n <= 0) return;
  f32_to_f64_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, n, dst);
  MOSES_CUDA(cudaGetLastError());
}
void f64_to_f32(const double* src, long long n, float* dst, cudaStream_t s) {
  if (n <= 0) return;
  f64_to_f32_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, n, dst);
  MOSES_CUDA(cudaGetLastError());
}
void refresh_shadow(const float* w, long long n, Shadow sh, cudaStream_t s) {
  if (n <= 0 || sh.kind == 0) return;
  if (sh.kind == 1) shadow_kernel1<<<grid_for(n, 256), 256, 0, s>>>(w, n, sh.ptr);
  else if (sh.kind == 2) shadow_kernel2<<<grid_for(n, 256), 256, 0, s>>>(w, n, sh.ptr);
  else if (sh.kind == 4)
    shadow_kernel4<<<grid_for(n, 256), 256, 0, s>>>(w, n, static_cast<__nv_bfloat16*>(sh.ptr), sh.lo_off);
  else shadow_kernel3<<<grid_for(n, 256), 256, 0, s>>>(w, n, static_cast<float*>(sh.ptr));
  MOSES_CUDA(cudaGetLastError());
}
void f32_to_bf16(const float* src, long long n, __nv_bfloat16* dst, cudaStream_t s) {
  if (n <= 0) return;
  f32_to_bf16_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, n, dst);
  MOSES_CUDA(cudaGetLastError());
}

void gather_batch(const void* x_base, long long row_bytes, const float* y_base, const long long* counter, long long nb,
                  long long batch, void* dst, float* ydst, cudaStream_t s, void* dst_lo) {
  if ((row_bytes % 16) != 0) fail(MOSES_ERR_INVALID_ARG, "packed rows must be 16-byte multiples");
  gather_batch_kernel<<<grid_for(batch * row_bytes / 16, 256), 256, 0, s>>>(
      static_cast<const uint8_t*>(x_base), row_bytes, y_base, counter, nb, batch, static_cast<uint8_t*>(dst), ydst,
      static_cast<uint8_t*>(dst_lo));
  MOSES_CUDA(cudaGetLastError());
}
void gather_plan(const void* x_base, long long row_bytes, const float* y_base, const long long* rows, const long long* off,
                 const long long* counter, long long n, void* dst, float* ydst, cudaStream_t s, void* dst_lo) {
  if ((row_bytes % 16) != 0) fail(MOSES_ERR_INVALID_ARG, "packed rows must be 16-byte multiples");
  gather_plan_kernel<<<std::max(1, ceil_div(n * 32, 256)), 256, 0, s>>>(static_cast<const uint8_t*>(x_base), row_bytes,
                                                                         y_base, rows, off, counter, n,
                                                                         static_cast<uint8_t*>(dst), ydst,
                                                                         static_cast<uint8_t*>(dst_lo));
  MOSES_CUDA(cudaGetLastError());
}
void accum_f64(const double* src, double* dst, cudaStream_t s) {
  accum_f64_kernel<<<1, 1, 0, s>>>(src, dst);
  MOSES_CUDA(cudaGetLastError());
}
void gather_pooled(const void* x_base, long long row_bytes, const float* y_base, const long long* prog_off,
                   const long long* counter, long long nb, long long B, long long rows_pad, void* dst, float* ydst,
                   long long* seg_off, int* seg_rows, cudaStream_t s, void* dst_lo) {
  if ((row_bytes % 16) != 0) fail(MOSES_ERR_INVALID_ARG, "packed rows must be 16-byte multiples");
  gather_pooled_kernel<<<grid_for(rows_pad * row_bytes / 16, 256), 256, 0, s>>>(
      static_cast<const uint8_t*>(x_base), row_bytes, y_base, prog_off, counter, nb, B, rows_pad,
      static_cast<uint8_t*>(dst), ydst, seg_off, seg_rows, static_cast<uint8_t*>(dst_lo));
  MOSES_CUDA(cudaGetLastError());
}
template <typename T>
void pack_pooled(const double* xs, const double* ys, const long long* offs, const long long* dims_dev, int D,
                 long long rows_pad, T* act0, long long ld, float* ydst, long long* seg_off, int* seg_rows,
                 cudaStream_t s, T* lo) {
  pack_pooled_kernel<T><<<grid_for(rows_pad * ld, 256), 256, 0, s>>>(xs, ys, offs, dims_dev, D, rows_pad, act0, ld, ydst,
                                                                     seg_off, seg_rows, lo);
  MOSES_CUDA(cudaGetLastError());
}
template void pack_pooled<__nv_bfloat16>(const double*, const double*, const long long*, const long long*, int,
                                         long long, __nv_bfloat16*, long long, float*, long long*, int*, cudaStream_t,
                                         __nv_bfloat16*);
void store_scalar_f64(const double* src, double* dst, cudaStream_t s) {
  store_scalar_f64_kernel<<<1, 1, 0, s>>>(src, dst);
  MOSES_CUDA(cudaGetLastError());
}
void advance_counter(long long* c, cudaStream_t s) {
  advance_counter_kernel<<<1, 32, 0, s>>>(c);
  MOSES_CUDA(cudaGetLastError());
}

void strided_f64_to_f32(const double* src, long long rows, int W, float* dst, long long ldd, cudaStream_t s) {
  if (rows <= 0) return;
  strided_f64_to_f32_kernel<<<grid_for(rows * W, 256), 256, 0, s>>>(src, rows, W, dst, ldd);
  MOSES_CUDA(cudaGetLastError());
}
void row_dot(const float* H, long long ldh, long long R, int W, const float* u, float* out, cudaStream_t s) {
  if (R <= 0) return;
  row_dot_kernel<<<grid_for(R * 32, 256), 256, 0, s>>>(H, ldh, R, W, u, out);
  MOSES_CUDA(cudaGetLastError());
}
void disc_ce(const double* z, long long m, long long n, double* out, cudaStream_t s) {
  disc_ce_kernel<<<1, kFinBlock, 0, s>>>(z, m, n, out);
  MOSES_CUDA(cudaGetLastError());
}

void head_scores(const float* part, int ntiles, long long ld, const float* hb, long long rows, float* s, cudaStream_t st) {
  if (rows <= 0) return;
  head_scores_kernel<<<grid_for(rows, 256), 256, 0, st>>>(part, ntiles, ld, hb, rows, s);
  MOSES_CUDA(cudaGetLastError());
}

int rank_splits(long long n) { return n <= 0 ? 1 : ceil_div(n, kRankChunk); }

void rank_pairs(const float* s, const float* y, long long n, const RankWs& ws, cudaStream_t st) {
  if (n <= 0) return;
  dim3 grid(ceil_div(n, kRankBlock), ceil_div(n, kRankChunk));
  rank_pairs_kernel<<<grid, kRankBlock, 0, st>>>(s, nullptr, 0, 0, nullptr, nullptr, y, n, ws.gs_part, ws.loss_part,
                                                 ws.pairs_part, nullptr, 0, n);
  MOSES_CUDA(cudaGetLastError());
}
void rank_pairs_rows(const float* s, const float* y, long long n, long long r0, long long nr, const RankWs& ws,
                     cudaStream_t st) {
  if (nr <= 0 || n <= 0) return;
  dim3 grid(ceil_div(nr, kRankBlock), ceil_div(n, kRankChunk));
  rank_pairs_kernel<<<grid, kRankBlock, 0, st>>>(s, nullptr, 0, 0, nullptr, nullptr, y, n, ws.gs_part, ws.loss_part,
                                                 ws.pairs_part, nullptr, r0, nr);
  MOSES_CUDA(cudaGetLastError());
}
// (loss sum, pair count) of the partials of nr rows -> out[0..1] (fixed order, one block)
__global__ void __launch_bounds__(kFinBlock) rank_totals_kernel(const double* loss_part, const long long* pairs_part,
                                                                int nsplit, long long nr, double* out) {
  using BR = cub::BlockReduce<double, kFinBlock>;
  using BRL = cub::BlockReduce<long long, kFinBlock>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ typename BRL::TempStorage tmpl;
  long long p = 0;
  double l = 0.0;
  for (long long i = threadIdx.x; i < nr; i += kFinBlock)
    for (int sp = 0; sp < nsplit; ++sp) {
      p += pairs_part[sp * nr + i];
      l += loss_part[sp * nr + i];
    }
  const long long pt = BRL(tmpl).Sum(p);
  __syncthreads();
  const double lt = BR(tmp).Sum(l);
  if (threadIdx.x == 0) {
    out[0] = lt;
    out[1] = double(pt);
  }
}
void rank_local_totals(const RankWs& ws, long long nr, double* out, cudaStream_t st) {
  rank_totals_kernel<<<1, kFinBlock, 0, st>>>(ws.loss_part, ws.pairs_part, ws.nsplit, nr, out);
  MOSES_CUDA(cudaGetLastError());
}
void rank_pairs_fused(const float* part, int ntiles, long long ld, const float* hb, const long long* seg, const float* y,
                      long long n, const RankWs& ws, float* s_out, cudaStream_t st) {
  if (n <= 0) return;
  dim3 grid(ceil_div(n, kRankBlock), ceil_div(n, kRankChunk));
  rank_pairs_kernel<<<grid, kRankBlock, 0, st>>>(nullptr, part, ntiles, ld, hb, seg, y, n, ws.gs_part, ws.loss_part,
                                                 ws.pairs_part, s_out, 0, n);
  MOSES_CUDA(cudaGetLastError());
}

void rank_finalize(const RankWs& ws, long long n, long long roff, const float* part2, int ntiles2, long long ld2,
                   const float* adv_bias, double beta, const FinalizeOut& out, cudaStream_t st, const double* totals) {
  rank_finalize_kernel<<<1, kFinBlock, 0, st>>>(ws.gs_part, ws.loss_part, ws.pairs_part, ws.nsplit, n, roff, part2,
                                                ntiles2, ld2, adv_bias, beta, out.loss, out.pairs, out.coefA, out.coefB,
                                                out.ce, out.seg_of_row, out.R_rows, out.gb, totals);
  MOSES_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- MMD^2 as a differentiable loss
// Biased MMD^2 with k(a,b) = exp(-c |a-b|^2), c = 1/(2 sigma^2), over rows a of X = [S; T] (m source
// rows, then n target rows) with alpha_a = 1/m (source) or -1/n (target):
//   MMD^2 = sum_a alpha_a r_a,   r_a = sum_b alpha_b k_ab
//   dMMD^2/dx_a = -4 c alpha_a (x_a r_a - O_a),   O_a = sum_b alpha_b k_ab x_b
// Register-tiled passes on the CUDA cores (fp32; the O(R^2 W) work is two GEMM-shaped products,
// ~0.3 G FMA each at the fine-tune shape R = 768, W = 512):
//   mmd_prep_kernel  X_a = hi + lo in fp32 and |x_a|^2 (features in order)
//   mmd_kmat_kernel  K_ab = alpha_b exp(-c max(|x_a|^2 + |x_b|^2 - 2 x_a.x_b, 0)) for a 64 x 64 tile per
//                    block; the dot products accumulate over the features in the same order as |x_a|^2,
//                    so d_aa is exactly 0 (an fp32 distance error of ~1e-4 moves k by ~1e-6 relative)
//   mmd_rows_kernel  r_a = sum_b K_ab (b in order) and the MMD^2 partial alpha_a r_a
//   mmd_out_kernel   G_a = -4 c alpha_a (x_a r_a - sum_b K_ab x_b) for a 64 x 64 (rows x features) tile
// Operand tiles are double-buffered through registers. Rows are taken in chunks of kMmdChunk so the K
// block stays L2-sized. Deterministic.
constexpr int kMmdT = 64, kMmdF = 32, kMmdChunk = 2048;
template <typename T>
__global__ void mmd_prep_kernel(const T* __restrict__ H, const T* __restrict__ H_lo, long long ld, long long R, int W,
                                float* __restrict__ X, float* __restrict__ nrm) {
  // a warp per row: lanes write the fp32 row; lane 0 then forms |x|^2 in feature order from it
  const long long a = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= R) return;
  for (int f = lane; f < W; f += 32) X[a * W + f] = load_operand(H, H_lo, a * ld + f);
  __syncwarp();
  if (lane == 0) {
    float n = 0.f;
    for (int f = 0; f < W; ++f) {
      const float v = X[a * W + f];
      n = fmaf(v, v, n);
    }
    nrm[a] = n;
  }
}
// acc[i][j] += sum_k A(row i, k) B(k, col j) over a 64 x 64 tile, k in chunks of 32, double-buffered
// through registers. An operand is either row-major with k contiguous (ROWK: X rows, K rows; a thread
// fetches 4 consecutive k of one row and they are transposed into the [k][row] smem tile) or k-major
// with the tile's columns contiguous (X rows indexed by k = b). get(row_or_k, col_or_k, ...) -> float4.
template <bool A_ROWK, bool B_ROWK, typename FA, typename FB>
__device__ __forceinline__ void mmd_tile_mac(int kdim, FA fa, FB fb, float (&acc)[4][4]) {
  __shared__ __align__(16) float at[2][kMmdF][kMmdT + 4];
  __shared__ __align__(16) float bt[2][kMmdF][kMmdT + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float4 ra[2], rb[2];
  // 512 float4 per 64 x 32 tile: ROWK -> (row e / 8, k 4 (e % 8)); k-major -> (k e / 16, col 4 (e % 16))
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = threadIdx.x + u * 256;
      ra[u] = A_ROWK ? fa(e >> 3, k0 + (e & 7) * 4) : fa(k0 + (e >> 4), (e & 15) * 4);
      rb[u] = B_ROWK ? fb(e >> 3, k0 + (e & 7) * 4) : fb(k0 + (e >> 4), (e & 15) * 4);
    }
  };
  auto put = [&](float (*t)[kMmdT + 4], bool rowk, int e, float4 v) {
    if (rowk) {
      const int row = e >> 3, k4 = (e & 7) * 4;
      t[k4 + 0][row] = v.x;
      t[k4 + 1][row] = v.y;
      t[k4 + 2][row] = v.z;
      t[k4 + 3][row] = v.w;
    } else {
      *reinterpret_cast<float4*>(&t[e >> 4][(e & 15) * 4]) = v;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = threadIdx.x + u * 256;
      put(at[buf], A_ROWK, e, ra[u]);
      put(bt[buf], B_ROWK, e, rb[u]);
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < kdim; k0 += kMmdF) {
    const bool more = k0 + kMmdF < kdim;
    if (more) fetch(k0 + kMmdF);
#pragma unroll 8
    for (int k = 0; k < kMmdF; ++k) {
      const float4 va = *reinterpret_cast<const float4*>(&at[buf][k][ty * 4]);
      const float4 vb = *reinterpret_cast<const float4*>(&bt[buf][k][tx * 4]);
      const float pa[4] = {va.x, va.y, va.z, va.w}, pb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(pa[i], pb[j], acc[i][j]);
    }
    if (more) {
      stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
}
__global__ void __launch_bounds__(256) mmd_kmat_kernel(const float* __restrict__ X, const float* __restrict__ nrm,
                                                       long long R, long long m, int W, float c, long long a_base,
                                                       long long na, float* __restrict__ K, long long Rk) {
  const long long a0 = a_base + (long long)blockIdx.y * kMmdT, b0 = (long long)blockIdx.x * kMmdT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  auto quad = [&](long long row, long long lim, int f) -> float4 {  // X[row][f..f+3], W % 4 == 0
    return (row < lim && f < W) ? *reinterpret_cast<const float4*>(X + row * W + f) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  mmd_tile_mac<true, true>(W, [&](int r, int f) { return quad(a0 + r, a_base + na, f); },
                           [&](int r, int f) { return quad(b0 + r, R, f); }, acc);
  const float as = 1.f / float(m), at = -1.f / float(R - m);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long a = a0 + ty * 4 + i;
    if (a >= a_base + na) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long b = b0 + tx * 4 + j;
      if (b >= R) continue;
      const float d = fmaxf(fmaf(-2.f, acc[i][j], nrm[a] + nrm[b]), 0.f);
      K[(a - a_base) * Rk + b] = (b < m ? as : at) * expf(-c * d);
    }
  }
}
// r_a = sum_b K_ab in b order (a warp per row: lane-strided partial sums, fixed shuffle tree)
__global__ void mmd_rows_kernel(const float* __restrict__ K, long long R, long long Rk, long long m, long long a_base,
                                long long na, float* __restrict__ r, double* __restrict__ vpart) {
  const long long a = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= na) return;
  float s = 0.f;
  for (long long b = lane; b < R; b += 32) s += K[a * Rk + b];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const long long ga = a_base + a;
    r[a] = s;
    vpart[ga] = double(ga < m ? 1.f / float(m) : -1.f / float(R - m)) * double(s);
  }
}
// G_a,f = -4 c alpha_a (x_a,f r_a - sum_b K_ab x_b,f): rows a x features f tiles of 64 x 64
__global__ void __launch_bounds__(256) mmd_out_kernel(const float* __restrict__ X, const float* __restrict__ K,
                                                      const float* __restrict__ r, long long R, long long m, int W,
                                                      float c, long long a_base, long long na, float* __restrict__ G) {
  const long long a0 = (long long)blockIdx.y * kMmdT;  // chunk-local row
  const int f0 = blockIdx.x * kMmdT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  const long long Rk = (R + 3) / 4 * 4;  // K rows are padded to 4 columns (host)
  mmd_tile_mac<true, false>(
      int(Rk),
      [&](int i, int b) {  // K[a0 + i][b..b+3]
        return (a0 + i < na && b < Rk) ? *reinterpret_cast<const float4*>(K + (a0 + i) * Rk + b)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
      },
      [&](int b, int f) {  // X[b][f0 + f..+3]
        return (b < R && f0 + f < W) ? *reinterpret_cast<const float4*>(X + (long long)b * W + f0 + f)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
      },
      acc);
  const float as = 1.f / float(m), at = -1.f / float(R - m);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long al = a0 + ty * 4 + i;
    if (al >= na) continue;
    const long long a = a_base + al;
    const float s = -4.f * c * (a < m ? as : at);
    const float ra = r[al];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int f = f0 + tx * 4 + j;
      if (f < W) G[a * W + f] = s * fmaf(X[a * W + f], ra, -acc[i][j]);
    }
  }
}
__global__ void sum_f64_kernel(const double* __restrict__ v, long long n, double scale, double* out, int accumulate) {
  using BR = cub::BlockReduce<double, 1024>;
  __shared__ typename BR::TempStorage tmp;
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += 1024) acc += v[i];
  const double t = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) {
    out[0] = accumulate ? out[0] + scale * t : scale * t;
  }
}
// The stream-ordered allocations of the per-call workspaces come from the device's default memory pool,
// whose release threshold is 0: every synchronisation hands its memory back to the driver and the next
// call maps it again (~0.3 ms per call, measured in the fine-tune step). Keep it mapped.
void keep_async_pool() {
  static thread_local int done_dev = -1;
  int dev = 0;
  MOSES_CUDA(cudaGetDevice(&dev));
  if (done_dev == dev) return;
  cudaMemPool_t pool;
  MOSES_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = ~uint64_t(0);
  MOSES_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  done_dev = dev;
}
template <typename T>
void mmd_grad(const T* H, const T* H_lo, long long ld, long long R, long long m, int W, float sigma, float* G,
              double* vpart, double* value_out, double scale, bool accumulate, cudaStream_t st) {
  if (m <= 0 || R - m <= 0) fail(MOSES_ERR_ADVERSARY_DISABLED, "MMD needs source and target rows");
  if (W % 4 != 0) fail(MOSES_ERR_INVALID_ARG, "MMD loss needs a representation width divisible by 4");
  const float c = 1.f / (2.f * sigma * sigma);
  keep_async_pool();
  const long long chunk = std::min<long long>(R, kMmdChunk);
  const long long Rk = (R + 3) / 4 * 4;  // K rows padded to 4 columns (float4 loads), pad columns zero
  float *X = nullptr, *nrm = nullptr, *K = nullptr, *r = nullptr;
  MOSES_CUDA(cudaMallocAsync(&X, sizeof(float) * size_t(R) * size_t(W), st));
  MOSES_CUDA(cudaMallocAsync(&nrm, sizeof(float) * size_t(R), st));
  MOSES_CUDA(cudaMallocAsync(&K, sizeof(float) * size_t(chunk) * size_t(Rk), st));
  MOSES_CUDA(cudaMallocAsync(&r, sizeof(float) * size_t(chunk), st));
  if (Rk != R) MOSES_CUDA(cudaMemsetAsync(K, 0, sizeof(float) * size_t(chunk) * size_t(Rk), st));
  mmd_prep_kernel<T><<<unsigned(ceil_div(R, 8)), 256, 0, st>>>(H, H_lo, ld, R, W, X, nrm);
  for (long long a0 = 0; a0 < R; a0 += chunk) {
    const long long na = std::min(chunk, R - a0);
    const dim3 gk(unsigned(ceil_div(R, kMmdT)), unsigned(ceil_div(na, kMmdT)));
    mmd_kmat_kernel<<<gk, 256, 0, st>>>(X, nrm, R, m, W, c, a0, na, K, Rk);
    mmd_rows_kernel<<<unsigned(ceil_div(na, 8)), 256, 0, st>>>(K, R, Rk, m, a0, na, r, vpart);
    const dim3 go(unsigned(ceil_div(W, kMmdT)), unsigned(ceil_div(na, kMmdT)));
    mmd_out_kernel<<<go, 256, 0, st>>>(X, K, r, R, m, W, c, a0, na, G);
  }
  MOSES_CUDA(cudaFreeAsync(X, st));
  MOSES_CUDA(cudaFreeAsync(nrm, st));
  MOSES_CUDA(cudaFreeAsync(K, st));
  MOSES_CUDA(cudaFreeAsync(r, st));
  sum_f64_kernel<<<1, 1024, 0, st>>>(vpart, R, scale, value_out, accumulate ? 1 : 0);
  MOSES_CUDA(cudaGetLastError());
}
template void mmd_grad<float>(const float*, const float*, long long, long long, long long, int, float, float*, double*,
                              double*, double, bool, cudaStream_t);
template void mmd_grad<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, long long, long long, long long, int,
                                      float, float*, double*, double*, double, bool, cudaStream_t);

// sharded top-k: the k local winners (score, global index); slots past k_valid padded (-inf, -1)
__global__ void topk_winners_kernel(const float* __restrict__ s, const long long* __restrict__ idx, long long k_valid,
                                    long long k, long long row0, float* __restrict__ out_s, long long* __restrict__ out_i) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < k; i += (long long)gridDim.x * blockDim.x) {
    if (i < k_valid) {
      out_s[i] = s[idx[i]];
      out_i[i] = idx[i] + row0;
    } else {
      out_s[i] = -INFINITY;
      out_i[i] = -1;
    }
  }
}
void topk_winners(const float* s, const long long* idx, long long k_valid, long long k, long long row0, float* out_s,
                  long long* out_i, cudaStream_t st) {
  topk_winners_kernel<<<ceil_div(k, 256), 256, 0, st>>>(s, idx, k_valid, k, row0, out_s, out_i);
  MOSES_CUDA(cudaGetLastError());
}

void rank_trace_read(unsigned long long* out) {
  MOSES_CUDA(cudaMemcpyFromSymbol(out, g_rank_trace, sizeof(unsigned long long) * 16));
}
void rank_cta_trace_read(unsigned long long* out) {
  MOSES_CUDA(cudaMemcpyFromSymbol(out, g_rank_cta_trace, sizeof(unsigned long long) * 512 * 5));
}
// Policy: the 16-CTA cluster form when the batch fits it (at n = 512 it is faster: the grid form's
// 128 CTAs all read the same head partials, and its last-CTA tail adds ~3 us), else the grid form,
// else (false) the two-kernel path. The test hook forces the grid form.
static bool g_rank_grid = false;
static bool g_rank_sym = true;
void debug_set_rank_grid(bool on) { g_rank_grid = on; }
void debug_set_rank_sym(bool on) { g_rank_sym = on; }
bool rank_step(const float* part, int ntiles, long long ld, const float* hb, const long long* seg, const float* y,
               long long n, const RankWs& ws, unsigned int* ticket, float* s_out, const int* seg_of_row, long long R,
               const FinalizeOut& out, cudaStream_t st) {
  const int nsplit = rank_splits(n);
  if (n <= 0) return false;
  const int cl_rows = ceil_div(n, kRankCluster);
  const bool cluster_fits = cl_rows * nsplit <= kRankMaxItems && cl_rows <= kRankMaxRows &&
                            size_t(2 * n + 3 * kRankMaxItems + (seg ? R : 0)) * 4 <= 160 * 1024;
  // symmetric form (each pair once) for batches past the cluster form; the grid form stays reachable
  // through the test hook (g_rank_grid) and when the symmetric workspace does not fit
  if (!cluster_fits && !g_rank_grid && g_rank_sym && ticket != nullptr) {
    const long long nb = ceil_div(n, 32), T = nb * (nb + 1) / 2;
    const size_t smem = size_t(n) * 8;  // (score, label) pairs
    const long long ws_entries = (long long)nsplit * n;  // gs_part / loss_part / pairs_part entries
    static int sms = 0;
    if (sms == 0) {
      MOSES_CUDA(cudaFuncSetAttribute(rank_sym_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      int dev = 0;
      MOSES_CUDA(cudaGetDevice(&dev));
      MOSES_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    int per_sm = 0;  // co-resident CTAs at this batch's shared memory (cooperative launch bound)
    MOSES_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rank_sym_kernel, kRsThreads, smem));
    const int sym_grid = sms;  // one 1024-thread CTA per SM
    if (per_sm >= 1 && smem <= 100 * 1024 && T * 64 <= 2 * ws_entries && T + sym_grid + n <= ws_entries) {
      float* rowcol = reinterpret_cast<float*>(ws.gs_part);
      double* tl = ws.loss_part;
      long long* tp = ws.pairs_part;
      double* cgb = ws.loss_part + T;
      long long* cpp = ws.pairs_part + T;
      float* sg = reinterpret_cast<float*>(ws.loss_part + T + sym_grid);
      unsigned* bar = ticket + 1;  // [count, generation, final ticket]
      const long long Rk = seg ? R : n;
      void* args[] = {(void*)&part, (void*)&ntiles, (void*)&ld, (void*)&hb, (void*)&seg, (void*)&y, (void*)&n,
                      (void*)&s_out, (void*)&Rk, (void*)&rowcol, (void*)&tl, (void*)&tp, (void*)&cgb, (void*)&cpp,
                      (void*)&sg, (void*)&bar, (void*)&out.loss, (void*)&out.pairs, (void*)&out.coefA, (void*)&out.coefB,
                      (void*)&out.gb};
      MOSES_CUDA(cudaLaunchCooperativeKernel((const void*)rank_sym_kernel, dim3(sym_grid), dim3(kRsThreads), args,
                                             smem, st));
      MOSES_CUDA(cudaGetLastError());
      return true;
    }
  }
  if ((g_rank_grid || !cluster_fits) && ticket != nullptr) {
    const int rows_per_cta = std::max<int>(4, ceil_div(n, 148));
    const int grid = ceil_div(n, rows_per_cta);
    const int items = rows_per_cta * nsplit;
    const size_t smem = size_t(2 * n + 3 * items + (seg ? R : 0)) * 4 + 8 + (seg ? size_t(n + 1) * 8 : 0) + size_t(n) * 8;
    if (smem <= 200 * 1024) {
      static bool configured = false;
      if (!configured) {
        MOSES_CUDA(cudaFuncSetAttribute(rank_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
      }
      rank_grid_kernel<<<grid, kRgThreads, smem, st>>>(part, ntiles, ld, hb, seg, seg ? seg_of_row : nullptr, y, n,
                                                       nsplit, rows_per_cta, s_out, seg ? R : n, ws.gs_part,
                                                       ws.loss_part, ws.pairs_part, ticket, out.loss, out.pairs,
                                                       out.coefA, out.coefB, out.gb);
      MOSES_CUDA(cudaGetLastError());
      return true;
    }
  }
  const int rows_per_cta = ceil_div(n, kRankCluster);
  if (rows_per_cta * nsplit > kRankMaxItems || rows_per_cta > kRankMaxRows) return false;
  const size_t smem = size_t(2 * n + 3 * kRankMaxItems + (seg ? R : 0)) * 4;
  if (smem > 160 * 1024) return false;
  static bool configured = false;
  if (!configured) {
    MOSES_CUDA(cudaFuncSetAttribute(rank_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    MOSES_CUDA(cudaFuncSetAttribute(rank_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kRankCluster);
  cfg.blockDim = dim3(kRankThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kRankCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // prologue overlaps the forward's tail
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const long long Rk = seg ? R : n;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, rank_cluster_kernel, part, ntiles, ld, hb, seg, y, n, nsplit, rows_per_cta, s_out,
                                Rk, out.loss, out.pairs, out.coefA, out.coefB, out.gb));
  MOSES_CUDA(cudaGetLastError());
  return true;
}

template <typename T>
void head_backward(const float* coefA, const float* coefB, const float* wh, const float* u, const T* H, long long ldh,
                   long long R, int W, T* dz, long long ldz, cudaStream_t st, T* dz_lo, const float* extra,
                   float extra_scale) {
  if (R <= 0) return;
  if constexpr (sizeof(T) == 2) {
    if (extra == nullptr && W % 8 == 0 && ldh % 8 == 0 && ldz % 8 == 0 &&
        ((reinterpret_cast<uintptr_t>(H) | reinterpret_cast<uintptr_t>(dz) | reinterpret_cast<uintptr_t>(dz_lo)) & 15) ==
            0) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid_for(R * (W / 8), 256));
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      MOSES_CUDA(cudaLaunchKernelEx(&cfg, head_backward_bf16x8_kernel, coefA, coefB, wh, u,
                                    reinterpret_cast<const __nv_bfloat16*>(H), ldh, R, W,
                                    reinterpret_cast<__nv_bfloat16*>(dz), ldz,
                                    reinterpret_cast<__nv_bfloat16*>(dz_lo)));
      return;
    }
  }
  head_backward_kernel<T><<<grid_for(R * W, 256), 256, 0, st>>>(coefA, coefB, wh, u, H, ldh, R, W, dz, ldz, dz_lo,
                                                                 extra, extra_scale);
  MOSES_CUDA(cudaGetLastError());
}

template <typename T>
void column_dot(const float* coef, const T* H, long long ldh, long long R, int W, float* g, float* ws, cudaStream_t st,
                const float* bias_override, const T* H_lo) {
  const int slabs = R > 0 ? ceil_div(R, kColSlab) : 1;
  if (R <= 0) {
    MOSES_CUDA(cudaMemsetAsync(g, 0, sizeof(float) * (W + 1), st));
    return;
  }
  column_dot_kernel<T><<<dim3(ceil_div(W + 1, 32), slabs), 256, 0, st>>>(coef, H, ldh, R, W, ws, H_lo);
  column_sum_kernel<<<ceil_div(W + 1, 256), 256, 0, st>>>(ws, slabs, W + 1, g, bias_override);
  MOSES_CUDA(cudaGetLastError());
}
size_t column_dot_ws_floats(long long R, int W) { return size_t(R > 0 ? ceil_div(R, kColSlab) : 1) * (W + 1); }

void sgd_update(float* w, float* v, const float* g, const uint8_t* mask, long long P, float lr, float mu, bool momentum,
                Shadow sh, cudaStream_t st) {
  const int grid = grid_for(P, 256);
  // 16-byte lanes when every array allows it (the whole-model buffers do; offset sub-blocks may not)
  const uintptr_t al16 = reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g) |
                         (momentum ? reinterpret_cast<uintptr_t>(v) : 0);
  const uintptr_t sh_al = sh.kind == 2 ? 15 : 7;
  const bool vec = P >= 1024 && (al16 & 15) == 0 && (reinterpret_cast<uintptr_t>(mask) & 3) == 0 &&
                   (sh.ptr == nullptr || ((reinterpret_cast<uintptr_t>(sh.ptr) & sh_al) == 0 &&
                                          (sh.kind != 4 || (sh.lo_off & 3) == 0)));
  const int grid4 = grid_for((P / 4 + 1) / 2, 256, 4);
#define SGD_LAUNCH(M, K, S)                                                                                   \
  if (vec) sgd4_kernel<M, K, S><<<grid4, 256, 0, st>>>(w, v, g, mask, P, lr, mu, sh.ptr, sh.lo_off);           \
  else sgd_kernel<M, K, S><<<grid, 256, 0, st>>>(w, v, g, mask, P, lr, mu, sh.ptr, sh.lo_off)
#define SGD_K(M, K)                                            \
  if (sh.kind == 1) { SGD_LAUNCH(M, K, 1); }                   \
  else if (sh.kind == 2) { SGD_LAUNCH(M, K, 2); }              \
  else if (sh.kind == 4) { SGD_LAUNCH(M, K, 4); }              \
  else { SGD_LAUNCH(M, K, 0); }
  const bool k = mask != nullptr;
  if (momentum) {
    if (k) { SGD_K(true, true); } else { SGD_K(true, false); }
  } else {
    if (k) { SGD_K(false, true); } else { SGD_K(false, false); }
  }
#undef SGD_K
#undef SGD_LAUNCH
  MOSES_CUDA(cudaGetLastError());
}

void adam_update(float* w, float* m1, float* m2, const float* g, const uint8_t* mask, long long P, float lr, float b1,
                 float b2, float eps, float c1, float c2, Shadow sh, cudaStream_t st) {
  const int grid = grid_for(P, 256);
  if (sh.kind == 1) adam_kernel<1><<<grid, 256, 0, st>>>(w, m1, m2, g, mask, P, lr, b1, b2, eps, c1, c2, sh.ptr);
  else if (sh.kind == 2) adam_kernel<2><<<grid, 256, 0, st>>>(w, m1, m2, g, mask, P, lr, b1, b2, eps, c1, c2, sh.ptr);
  else adam_kernel<0><<<grid, 256, 0, st>>>(w, m1, m2, g, mask, P, lr, b1, b2, eps, c1, c2, sh.ptr);
  MOSES_CUDA(cudaGetLastError());
}

void variant_decay(float* w, const uint8_t* mask, long long P, float factor, Shadow sh, cudaStream_t st) {
  const int grid = grid_for(P, 256);
  if (sh.kind == 1) decay_kernel<1><<<grid, 256, 0, st>>>(w, mask, P, factor, sh.ptr);
  else if (sh.kind == 2) decay_kernel<2><<<grid, 256, 0, st>>>(w, mask, P, factor, sh.ptr);
  else decay_kernel<0><<<grid, 256, 0, st>>>(w, mask, P, factor, sh.ptr);
  MOSES_CUDA(cudaGetLastError());
}

// ---- select workspace
static long long sel_chunk(long long n, int* grid) {
  const long long target = kSMs * 4;
  long long chunk = (n + target - 1) / target;
  chunk = round_up(chunk < 1 ? 1 : chunk, kSelBlock * 4);
  *grid = int((n + chunk - 1) / chunk);
  if (*grid < 1) *grid = 1;
  return chunk;
}
size_t select_ws_bytes(long long n, int* grid_out) {
  int grid;
  sel_chunk(n, &grid);
  if (grid_out) *grid_out = grid;
  return size_t(n) * 4 + kBins * 4 + size_t(grid) * kBins * 4 + 256 + 64 + 1024;
}
void select_ws_carve(void* base, long long n, SelectWs* ws) {
  int grid;
  sel_chunk(n, &grid);
  uint8_t* p = static_cast<uint8_t*>(base);
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += round_up(bytes, 256);
    return r;
  };
  ws->state = reinterpret_cast<unsigned*>(take(sizeof(SelState)));
  ws->counter = reinterpret_cast<unsigned long long*>(take(64));
  ws->hist = reinterpret_cast<unsigned*>(take(kBins * 4));
  ws->block_hist = reinterpret_cast<unsigned*>(take(size_t(grid) * kBins * 4));
  ws->keys = reinterpret_cast<unsigned*>(take(size_t(n) * 4));
  ws->grid = grid;
}

// Runs the three histogram passes; the first one is fused with key production (MODE).
template <int MODE>
static void radix_select_passes(const float* a, const float* b, long long n, unsigned long long need, const SelectWs& ws,
                                float* xi_out, cudaStream_t st) {
  int grid;
  const long long chunk = sel_chunk(n, &grid);
  SelState* S = reinterpret_cast<SelState*>(ws.state);
  sel_init_kernel<<<1, 256, 0, st>>>(S, need, ws.hist);
  for (int p = 0; p < 3; ++p) {
    const bool last = p == 2;
    if (p == 0) {
      radix_hist_kernel<MODE, false><<<grid, kSelBlock, 0, st>>>(a, b, ws.keys, xi_out, n, chunk, S, kPassShift[p],
                                                                 kPassBits[p], ws.hist, ws.block_hist);
    } else if (last) {
      radix_hist_kernel<0, true><<<grid, kSelBlock, 0, st>>>(a, b, ws.keys, nullptr, n, chunk, S, kPassShift[p],
                                                             kPassBits[p], ws.hist, ws.block_hist);
    } else {
      radix_hist_kernel<0, false><<<grid, kSelBlock, 0, st>>>(a, b, ws.keys, nullptr, n, chunk, S, kPassShift[p],
                                                              kPassBits[p], ws.hist, ws.block_hist);
    }
    radix_pick_kernel<<<1, kPickBlock, 0, st>>>(S, ws.hist, kPassShift[p], kPassBits[p]);
  }
  MOSES_CUDA(cudaGetLastError());
}

// exact key of descending rank `need` among ws.keys[0, n) -> SelState::prefix (sel_result_key)
void select_kth_key(long long n, unsigned long long need, const SelectWs& ws, cudaStream_t st) {
  radix_select_passes<0>(nullptr, nullptr, n, need, ws, nullptr, st);
}
const unsigned* sel_result_key(const SelectWs& ws) { return &reinterpret_cast<const SelState*>(ws.state)->prefix; }

void lottery_select(const float* w, const float* g, long long n, int mode, float theta, long long keep, const SelectWs& ws,
                    uint8_t* mask_out, float* xi_out, bool normalize_xi, cudaStream_t st) {
  int grid;
  const long long chunk = sel_chunk(n, &grid);
  SelState* S = reinterpret_cast<SelState*>(ws.state);
  if (mode == 1) {
    // threshold: xi + max in one pass, then the strict comparison on xi/max
    sel_init_kernel<<<1, 256, 0, st>>>(S, 0, ws.hist);
    radix_hist_kernel<1, false><<<grid, kSelBlock, 0, st>>>(w, g, ws.keys, nullptr, n, chunk, S, 31, 1, ws.hist,
                                                            ws.block_hist);
    threshold_mask_kernel<<<grid_for(n, kSelBlock), kSelBlock, 0, st>>>(ws.keys, n, S, theta, true, mask_out, xi_out);
  } else {
    radix_select_passes<1>(w, g, n, (unsigned long long)keep, ws, xi_out, st);
    radix_apply_kernel<0><<<grid, kSelBlock, 0, st>>>(ws.keys, n, chunk, S, ws.block_hist, mask_out, nullptr, nullptr,
                                                      nullptr);
    if (xi_out && normalize_xi) xi_normalize_kernel<<<grid_for(n, 256), 256, 0, st>>>(xi_out, n, S);
  }
  MOSES_CUDA(cudaGetLastError());
}

void xi_scores(const float* w, const float* g, long long n, bool normalize, const SelectWs& ws, float* xi_out,
               cudaStream_t st) {
  int grid;
  const long long chunk = sel_chunk(n, &grid);
  SelState* S = reinterpret_cast<SelState*>(ws.state);
  sel_init_kernel<<<1, 256, 0, st>>>(S, 0, ws.hist);
  radix_hist_kernel<1, false><<<grid, kSelBlock, 0, st>>>(w, g, ws.keys, xi_out, n, chunk, S, 31, 1, ws.hist,
                                                          ws.block_hist);
  if (normalize) xi_normalize_kernel<<<grid_for(n, 256), 256, 0, st>>>(xi_out, n, S);
  MOSES_CUDA(cudaGetLastError());
}

__global__ void keys_from_xi_kernel(const float* xi, long long n, unsigned* keys) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    keys[i] = __float_as_uint(xi[i]);
}

void partition_from_xi(const float* xi, long long n, int mode, float theta, long long keep, const SelectWs& ws,
                       uint8_t* mask_out, cudaStream_t st) {
  int grid;
  const long long chunk = sel_chunk(n, &grid);
  SelState* S = reinterpret_cast<SelState*>(ws.state);
  if (mode == 1) {
    sel_init_kernel<<<1, 256, 0, st>>>(S, 0, ws.hist);
    keys_from_xi_kernel<<<grid_for(n, 256), 256, 0, st>>>(xi, n, ws.keys);
    threshold_mask_kernel<<<grid_for(n, kSelBlock), kSelBlock, 0, st>>>(ws.keys, n, S, theta, false, mask_out, nullptr);
  } else {
    keys_from_xi_kernel<<<grid_for(n, 256), 256, 0, st>>>(xi, n, ws.keys);
    radix_select_passes<0>(nullptr, nullptr, n, (unsigned long long)keep, ws, nullptr, st);
    radix_apply_kernel<0><<<grid, kSelBlock, 0, st>>>(ws.keys, n, chunk, S, ws.block_hist, mask_out, nullptr, nullptr,
                                                      nullptr);
  }
  MOSES_CUDA(cudaGetLastError());
}

void lottery_apply(float* w, const float* g, const uint8_t* mask, long long n, float alpha, float factor, bool step,
                   bool decay, Shadow sh, cudaStream_t st) {
  const int grid = grid_for(n, 256);
  if (sh.kind == 1) lottery_apply_kernel<1><<<grid, 256, 0, st>>>(w, g, mask, n, alpha, factor, step, decay, sh.ptr);
  else if (sh.kind == 2) lottery_apply_kernel<2><<<grid, 256, 0, st>>>(w, g, mask, n, alpha, factor, step, decay, sh.ptr);
  else lottery_apply_kernel<0><<<grid, 256, 0, st>>>(w, g, mask, n, alpha, factor, step, decay, sh.ptr);
  MOSES_CUDA(cudaGetLastError());
}

long long popcount_mask(const uint8_t* mask, long long n, unsigned long long* dcount, cudaStream_t st) {
  MOSES_CUDA(cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), st));
  popcount_kernel<<<grid_for(n, kSelBlock), kSelBlock, 0, st>>>(mask, n, dcount);
  MOSES_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  MOSES_CUDA(cudaMemcpyAsync(&h, dcount, sizeof(h), cudaMemcpyDeviceToHost, st));
  MOSES_CUDA(cudaStreamSynchronize(st));
  return (long long)h;
}

void topk_select(const float* scores, long long n, long long k, const SelectWs& ws, unsigned* out_key, long long* out_idx,
                 cudaStream_t st) {
  if (k > kTopkMax) fail(MOSES_ERR_INVALID_ARG, "top-k supports k <= 4096");
  int grid;
  const long long chunk = sel_chunk(n, &grid);
  SelState* S = reinterpret_cast<SelState*>(ws.state);
  radix_select_passes<2>(scores, nullptr, n, (unsigned long long)k, ws, nullptr, st);
  MOSES_CUDA(cudaMemsetAsync(ws.counter, 0, sizeof(unsigned long long), st));
  radix_apply_kernel<1><<<grid, kSelBlock, 0, st>>>(ws.keys, n, chunk, S, ws.block_hist, nullptr, out_key, out_idx,
                                                    ws.counter);
  topk_sort_kernel<<<1, kSortBlock, 0, st>>>(out_key, out_idx, ws.counter, k);
  MOSES_CUDA(cudaGetLastError());
}

void accuracy_counts(const float* s, const float* y, const long long* seg_of_row, const long long* seg_off, long long n,
                     long long*, long long*, unsigned long long* totals, cudaStream_t st) {
  MOSES_CUDA(cudaMemsetAsync(totals, 0, 2 * sizeof(unsigned long long), st));
  if (n <= 0) return;
  accuracy_kernel<<<grid_for(n, 256), 256, 0, st>>>(s, y, seg_of_row, seg_off, n, totals);
  MOSES_CUDA(cudaGetLastError());
}

template <typename T>
void adversary_step(const float* part2, int ntiles, long long ld2, const T* H, long long ldh, long long m, long long n,
                    int W, float* u, float* c, float eta, double* loss_out, float* ws, cudaStream_t st,
                    const T* H_lo) {
  float* dz = ws;                                   // [m+n]
  float* du = ws + round_up(m + n, 64);             // [W+1]
  double* dc = reinterpret_cast<double*>(du + round_up(W + 1, 64));
  adv_logits_kernel<<<1, kFinBlock, 0, st>>>(part2, ntiles, ld2, m, n, c, dz, loss_out, dc);
  {
    const long long R = m + n;
    const int slabs = ceil_div(R, kColSlab);
    float* part = reinterpret_cast<float*>(dc + 8);
    column_dot_kernel<T><<<dim3(ceil_div(W + 1, 32), slabs), 256, 0, st>>>(dz, H, ldh, R, W, part, H_lo);
    column_sum_kernel<<<ceil_div(W + 1, 256), 256, 0, st>>>(part, slabs, W + 1, du, nullptr);
  }
  adv_update_kernel<<<ceil_div(W, 256), 256, 0, st>>>(u, c, du, W, eta, dc);
  MOSES_CUDA(cudaGetLastError());
}

template <typename T>
void segment_sum(const T* H, long long ldh, int W, const long long* offsets, long long programs, float* out, long long ldo,
                 cudaStream_t st) {
  if (programs <= 0) return;
  if ((W * sizeof(T)) % 16 != 0 || (ldh * sizeof(T)) % 16 != 0) fail(MOSES_ERR_INVALID_ARG, "segment_sum needs 16-byte rows");
  const int warps_per_block = 8;
  long long blocks = (programs + warps_per_block - 1) / warps_per_block;
  if (blocks > kSMs * 16) blocks = kSMs * 16;
  segment_sum_kernel<T><<<int(blocks), warps_per_block * 32, 0, st>>>(H, ldh, W, offsets, programs, out, ldo);
  MOSES_CUDA(cudaGetLastError());
}
void segment_sum_scalar(const float* v, const long long* offsets, long long programs, float bias, float* out,
                        cudaStream_t st) {
  if (programs <= 0) return;
  segment_sum_scalar_kernel<<<grid_for(programs, 256), 256, 0, st>>>(v, offsets, programs, bias, out);
  MOSES_CUDA(cudaGetLastError());
}


template <typename T>
void synth_features(unsigned long long seed, long long row0, long long n, int D, T* dst, long long ld, cudaStream_t st) {
  if (n <= 0) return;
  synth_features_kernel<T><<<grid_for(n, 128, 32), 128, 0, st>>>(seed, row0, n, D, dst, ld);
  MOSES_CUDA(cudaGetLastError());
}
void synth_labels(unsigned long long seed, long long row0, long long n, float* dst, cudaStream_t st) {
  if (n <= 0) return;
  synth_labels_kernel<<<grid_for(n, 256), 256, 0, st>>>(seed, row0, n, dst);
  MOSES_CUDA(cudaGetLastError());
}

#define INST(T)                                                                                                   \
  template void pack_rows<T>(const double*, long long, int, T*, long long, cudaStream_t, T*);                         \
  template void pack_rows_f32<T>(const float*, long long, int, long long, T*, long long, cudaStream_t, T*);           \
  template void set_ones_column<T>(T*, long long, int, long long, cudaStream_t);                                  \
  template void unpack_rows<T>(const T*, long long, int, long long, double*, cudaStream_t, const T*);             \
  template void head_backward<T>(const float*, const float*, const float*, const float*, const T*, long long,     \
                                 long long, int, T*, long long, cudaStream_t, T*, const float*, float);          \
  template void column_dot<T>(const float*, const T*, long long, long long, int, float*, float*, cudaStream_t,     \
                              const float*, const T*);                                                            \
  template void adversary_step<T>(const float*, int, long long, const T*, long long, long long, long long, int,   \
                                  float*, float*, float, double*, float*, cudaStream_t, const T*);                \
  template void segment_sum<T>(const T*, long long, int, const long long*, long long, float*, long long,          \
                               cudaStream_t);                                                                     \
  template void synth_features<T>(unsigned long long, long long, long long, int, T*, long long, cudaStream_t);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace moses
