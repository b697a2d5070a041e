// lottery.cu — the Moses adaptation step (tuner.cpp:258-262) as few HBM passes as the exact
// selection allows: xi = |w*g| is never materialised, every pass recomputes it from (w, g).
//
//   threshold (lottery.cpp:152-157, normalised):  pass 1 max(xi)  ->  pass 2 fused apply       23 B/param
//   ratio     (lottery.cpp:158-175, top ceil(rho*N), ties by index):
//     pass 1  15-bit histogram of xi bits [30:16] (xi >= 0, so the bit pattern orders like the value)
//     pass 2  16-bit histogram of bits [15:0] within the chosen bucket  -> exact threshold key T
//     pass 3  only if some keys equal to T must be dropped: per-block counts of key == T, then the
//             index of the last kept equal key (ascending-index tie-break, lottery.cpp:169-172)
//     pass 4  fused apply: kept = key > T || (key == T && i <= cut);  w -= alpha*g (kept) /
//             w *= 1 - alpha*lambda (others); operand shadow + mask byte written      31-39 B/param
// vs the algorithmic 15 B/param (read w, g; write w, bf16 shadow, mask byte).
// The passes only count and compare integers, so the mask is bit-identical to nth_element's.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "kernels.cuh"
#include "ptx.cuh"

namespace moses {
namespace {

constexpr int kB1 = 15, kB2 = 16;                 // digit widths (bit 31 of xi is always 0)
constexpr int kBins1 = 1 << kB1, kBins2 = 1 << kB2;
constexpr int kPassBlock = 1024;

struct LotState {
  unsigned long long need;   // scalars still to take among keys matching the prefix
  unsigned long long gt;     // scalars strictly above the current prefix range
  unsigned long long eq;     // scalars equal to T (after pass 2)
  unsigned prefix;           // b1 after pick 1; T after pick 2
  unsigned max_bits;         // threshold mode: max xi bits
  long long cut;             // last kept index among keys == T (LLONG_MAX: keep all equal keys)
  unsigned long long count;  // threshold mode popcount
};

__device__ __forceinline__ unsigned xi_key(const float* __restrict__ w, const float* __restrict__ g, long long i) {
  return __float_as_uint(fabsf(__fmul_rn(w[i], g[i])));
}

// Shared-memory histogram increment. Ties (e.g. the many xi == 0, README.md:106-113) make a whole
// warp hit one bin: that case is detected with one vote and added once; otherwise each lane adds
// to its own (mostly distinct) bin.
__device__ __forceinline__ void hist_add(unsigned* sh, unsigned bin, bool valid) {
  const unsigned b0 = __shfl_sync(0xffffffffu, bin, 0);
  const unsigned v0 = __shfl_sync(0xffffffffu, valid ? 1u : 0u, 0);
  if (__all_sync(0xffffffffu, valid && bin == b0)) {
    if ((threadIdx.x & 31) == 0) atomicAdd(&sh[b0], 32u);
    return;
  }
  (void)v0;
  if (valid) atomicAdd(&sh[bin], 1u);
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ unsigned key_of(float w, float g) { return __float_as_uint(fabsf(__fmul_rn(w, g))); }

__global__ void __launch_bounds__(kPassBlock) lot_hist1_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                                               long long n, unsigned* __restrict__ hist) {
  extern __shared__ unsigned sh[];
  for (int d = threadIdx.x; d < kBins1; d += kPassBlock) sh[d] = 0;
  __syncthreads();
  const long long n4 = n / 4;
  const long long stride = (long long)gridDim.x * kPassBlock;
  for (long long base = blockIdx.x * (long long)kPassBlock; base < n4; base += stride) {  // 4 scalars / thread
    const long long q = base + threadIdx.x;
    const bool ok = q < n4;
    float4 a = make_float4(0, 0, 0, 0), b = a;
    if (ok) {
      a = ld4(w + 4 * q);
      b = ld4(g + 4 * q);
    }
    hist_add(sh, key_of(a.x, b.x) >> 16, ok);
    hist_add(sh, key_of(a.y, b.y) >> 16, ok);
    hist_add(sh, key_of(a.z, b.z) >> 16, ok);
    hist_add(sh, key_of(a.w, b.w) >> 16, ok);
  }
  if (blockIdx.x == 0)  // scalar tail
    for (long long i = 4 * n4 + threadIdx.x; i < n; i += kPassBlock) atomicAdd(&sh[xi_key(w, g, i) >> 16], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < kBins1; d += kPassBlock)
    if (sh[d]) atomicAdd(&hist[d], sh[d]);
}

// Pass 2: 16-bit digits of the keys in bucket b1. 65536 u32 bins do not fit in shared memory, so
// the block keeps u16 counters and flushes its non-zero bins to the global histogram every
// 32768 elements (a bin can gain at most 32768 per round: no u16 overflow).
constexpr int kRound = 32 * kPassBlock;  // multiple of 4 (float4 loads stay aligned)
__global__ void __launch_bounds__(kPassBlock) lot_hist2_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                                               long long n, const LotState* st,
                                                               unsigned* __restrict__ hist) {
  extern __shared__ unsigned short sh16[];
  __shared__ int s_any;
  const unsigned b1 = st->prefix;
  for (int d = threadIdx.x; d < kBins2; d += kPassBlock) sh16[d] = 0;
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  long long per = (n + gridDim.x - 1) / gridDim.x;
  per = (per + 3) / 4 * 4;  // keep every block's range 16-byte aligned for the float4 loads
  const long long lo = blockIdx.x * per, hi = min(n, lo + per);
  for (long long r0 = lo; r0 < hi; r0 += kRound) {
    const long long r1 = min(hi, r0 + kRound);
    int any = 0;
    auto add = [&](unsigned key, bool ok) {
      const bool in = ok && (key >> kB2) == b1;
      const unsigned d = key & (kBins2 - 1);
      const unsigned d0 = __shfl_sync(0xffffffffu, d, 0);
      if (__all_sync(0xffffffffu, in && d == d0)) {
        if ((threadIdx.x & 31) == 0)
          atomicAdd(reinterpret_cast<unsigned*>(sh16 + (d0 & ~1u)), 32u << (16 * (d0 & 1u)));
        any = 1;
      } else if (in) {
        atomicAdd(reinterpret_cast<unsigned*>(sh16 + (d & ~1u)), 1u << (16 * (d & 1u)));
        any = 1;
      }
    };
    for (long long base = r0; base < r1; base += 4 * kPassBlock) {  // r0, r1 are multiples of 4 except the end
      const long long i = base + 4 * threadIdx.x;
      unsigned k0 = 0xffffffffu, k1 = k0, k2 = k0, k3 = k0;
      if (i + 3 < r1) {
        const float4 a = ld4(w + i), b = ld4(g + i);
        k0 = key_of(a.x, b.x);
        k1 = key_of(a.y, b.y);
        k2 = key_of(a.z, b.z);
        k3 = key_of(a.w, b.w);
      } else {
        if (i < r1) k0 = xi_key(w, g, i);
        if (i + 1 < r1) k1 = xi_key(w, g, i + 1);
        if (i + 2 < r1) k2 = xi_key(w, g, i + 2);
      }
      // warp-collective adds: every lane takes part (out-of-range lanes with ok = false)
      add(k0, i < r1);
      add(k1, i + 1 < r1);
      add(k2, i + 2 < r1);
      add(k3, i + 3 < r1);
    }
    if (any) s_any = 1;
    __syncthreads();
    if (s_any) {  // flush (block-uniform)
      for (int d = threadIdx.x; d < kBins2; d += kPassBlock) {
        const unsigned v = sh16[d];
        if (v) {
          atomicAdd(&hist[d], v);
          sh16[d] = 0;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
  }
}

// Single block: choose the digit where the descending cumulative count reaches `need`.
template <int BINS>
__global__ void __launch_bounds__(1024) lot_pick_kernel(LotState* st, unsigned* hist, int shift, bool last) {
  using Scan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr int PER = BINS / 1024;
  const unsigned long long need = st->need;  // read before any thread updates the state
  unsigned long long vals[PER];
  unsigned long long local = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {  // thread t owns digits BINS-1-(t*PER+q): descending order
    vals[q] = hist[BINS - 1 - (threadIdx.x * PER + q)];
    local += vals[q];
  }
  unsigned long long before;
  Scan(tmp).ExclusiveSum(local, before);
  unsigned long long run = before;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int d = BINS - 1 - (threadIdx.x * PER + q);
    if (run < need && run + vals[q] >= need) {  // unique digit d*
      st->need = need - run;
      st->gt += run;
      st->prefix = shift ? unsigned(d) : ((st->prefix << kB2) | unsigned(d));
      if (last) {
        st->eq = vals[q];
        st->cut = 0x7fffffffffffffffll;
      }
    }
    run += vals[q];
  }
  __syncthreads();
  for (int d = threadIdx.x; d < BINS; d += 1024) hist[d] = 0;  // ready for the next pass / call
}

// pass 3 (only when ties at T straddle the cut): per-block counts of key == T over fixed chunks
__global__ void __launch_bounds__(kPassBlock) lot_eq_count_kernel(const float* __restrict__ w,
                                                                  const float* __restrict__ g, long long n,
                                                                  long long chunk, const LotState* st,
                                                                  unsigned long long* __restrict__ block_eq) {
  using Red = cub::BlockReduce<unsigned long long, kPassBlock>;
  __shared__ typename Red::TempStorage tmp;
  if (st->need >= st->eq) return;  // every key equal to T is kept: no index cut needed
  const unsigned T = st->prefix;
  const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  unsigned long long c = 0;
  for (long long i = lo + threadIdx.x; i < hi; i += kPassBlock) c += xi_key(w, g, i) == T;
  c = Red(tmp).Sum(c);
  if (threadIdx.x == 0) block_eq[blockIdx.x] = c;
}

// one block: find the chunk holding the need-th key == T (ascending index), then its exact index
__global__ void __launch_bounds__(kPassBlock) lot_cut_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                                             long long n, long long chunk, int nblocks, LotState* st,
                                                             const unsigned long long* __restrict__ block_eq) {
  using Scan = cub::BlockScan<unsigned, kPassBlock>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long s_blk;
  __shared__ unsigned long long s_before;
  __shared__ long long s_cut;
  if (st->need >= st->eq) return;
  const unsigned long long need = st->need;
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    long long b = 0;
    for (; b < nblocks; ++b) {
      if (run + block_eq[b] >= need) break;
      run += block_eq[b];
    }
    s_blk = b;
    s_before = run;
    s_cut = -1;
  }
  __syncthreads();
  const unsigned T = st->prefix;
  const long long lo = s_blk * chunk, hi = min(n, lo + chunk);
  unsigned long long base = s_before;
  for (long long t0 = lo; t0 < hi; t0 += kPassBlock) {
    const long long i = t0 + threadIdx.x;
    const unsigned eq = (i < hi && xi_key(w, g, i) == T) ? 1u : 0u;
    unsigned rank, tot;
    Scan(tmp).ExclusiveSum(eq, rank, tot);
    if (eq && base + rank + 1 == need) s_cut = i;
    __syncthreads();
    base += tot;
    if (s_cut >= 0) break;
  }
  if (threadIdx.x == 0) st->cut = s_cut;
}

template <int SHADOW, bool THRESH>
__device__ __forceinline__ void lot_apply_one(long long i, float& wi, float gi, unsigned T, long long cut, float top,
                                              float theta, float alpha, float factor, bool decay, uint8_t& mk,
                                              unsigned long long& cnt) {
  const float x = fabsf(__fmul_rn(wi, gi));
  bool kept;
  if constexpr (THRESH) {
    const float xn = top > 0.f ? __fdiv_rn(x, top) : x;  // xi_scores(normalize) then xi > theta
    kept = xn > theta;
    cnt += kept;
  } else {
    const unsigned key = __float_as_uint(x);
    kept = key > T || (key == T && i <= cut);
  }
  if (kept) wi = __fsub_rn(wi, __fmul_rn(alpha, gi));  // transferable_step (apply_update, no momentum)
  else if (decay) wi = __fmul_rn(wi, factor);          // variant_decay
  mk = kept ? 1 : 0;
}

template <int SHADOW>
__device__ __forceinline__ void store_shadow4(void* sh, long long i, float4 v) {
  if constexpr (SHADOW == 1) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(sh) + i) = u;
  }
  if constexpr (SHADOW == 2) {
    float r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t t;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(r[k]));
      r[k] = __uint_as_float(t);
    }
    *reinterpret_cast<float4*>(static_cast<float*>(sh) + i) = make_float4(r[0], r[1], r[2], r[3]);
  }
}

template <int SHADOW, bool THRESH>
__global__ void __launch_bounds__(256) lot_apply_kernel(float* __restrict__ w, const float* __restrict__ g, long long n,
                                                        LotState* st, float theta, float alpha, float factor,
                                                        bool decay, void* __restrict__ shadow,
                                                        uint8_t* __restrict__ mask) {
  using Red = cub::BlockReduce<unsigned long long, 256>;
  __shared__ typename Red::TempStorage tmp;
  const unsigned T = st->prefix;
  const long long cut = st->cut;
  const float top = __uint_as_float(st->max_bits);
  unsigned long long cnt = 0;
  const long long n4 = n / 4;
  for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n4; q += (long long)gridDim.x * 256) {
    const long long i = 4 * q;
    float4 wv = *reinterpret_cast<const float4*>(w + i);
    const float4 gv = ld4(g + i);
    uchar4 mk;
    lot_apply_one<SHADOW, THRESH>(i, wv.x, gv.x, T, cut, top, theta, alpha, factor, decay, mk.x, cnt);
    lot_apply_one<SHADOW, THRESH>(i + 1, wv.y, gv.y, T, cut, top, theta, alpha, factor, decay, mk.y, cnt);
    lot_apply_one<SHADOW, THRESH>(i + 2, wv.z, gv.z, T, cut, top, theta, alpha, factor, decay, mk.z, cnt);
    lot_apply_one<SHADOW, THRESH>(i + 3, wv.w, gv.w, T, cut, top, theta, alpha, factor, decay, mk.w, cnt);
    *reinterpret_cast<float4*>(w + i) = wv;
    *reinterpret_cast<uchar4*>(mask + i) = mk;
    store_shadow4<SHADOW>(shadow, i, wv);
  }
  if (blockIdx.x == 0) {  // scalar tail
    for (long long i = 4 * n4 + threadIdx.x; i < n; i += 256) {
      float wi = w[i];
      uint8_t mk;
      lot_apply_one<SHADOW, THRESH>(i, wi, g[i], T, cut, top, theta, alpha, factor, decay, mk, cnt);
      w[i] = wi;
      mask[i] = mk;
      if constexpr (SHADOW == 1) static_cast<__nv_bfloat16*>(shadow)[i] = __float2bfloat16_rn(wi);
      if constexpr (SHADOW == 2) {
        uint32_t t;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(wi));
        static_cast<float*>(shadow)[i] = __uint_as_float(t);
      }
    }
  }
  if constexpr (THRESH) {
    cnt = Red(tmp).Sum(cnt);
    if (threadIdx.x == 0 && cnt) atomicAdd(&st->count, cnt);
  }
}

__global__ void __launch_bounds__(kPassBlock) lot_max_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                                             long long n, LotState* st) {
  unsigned m = 0;
  const long long n4 = n / 4;
  for (long long q = blockIdx.x * (long long)kPassBlock + threadIdx.x; q < n4; q += (long long)gridDim.x * kPassBlock) {
    const float4 a = ld4(w + 4 * q), b = ld4(g + 4 * q);
    m = max(max(max(m, key_of(a.x, b.x)), key_of(a.y, b.y)), max(key_of(a.z, b.z), key_of(a.w, b.w)));
  }
  if (blockIdx.x == 0)
    for (long long i = 4 * n4 + threadIdx.x; i < n; i += kPassBlock) m = max(m, xi_key(w, g, i));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(&st->max_bits, m);
}

__global__ void lot_init_kernel(LotState* st, unsigned long long keep) {
  st->need = keep;
  st->gt = 0;
  st->eq = 0;
  st->prefix = 0;
  st->max_bits = 0;
  st->cut = 0x7fffffffffffffffll;
  st->count = 0;
}

int g_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

size_t lottery_ws_bytes() {
  return 256 /*state*/ + size_t(kBins1) * 4 + size_t(kBins2) * 4 + size_t(4096) * 8 + 1024;
}

// Fused Moses step. mode 1 threshold (normalised, strict), 2 ratio (top `keep`, index tie-break).
void lottery_step_fused(float* w, const float* g, long long n, int mode, float theta, long long keep, float alpha,
                        float factor, bool decay, Shadow sh, uint8_t* mask, void* ws, unsigned long long* popcount_dev,
                        cudaStream_t st) {
  uint8_t* p = static_cast<uint8_t*>(ws);
  LotState* S = reinterpret_cast<LotState*>(p);
  unsigned* hist1 = reinterpret_cast<unsigned*>(p + 256);
  unsigned* hist2 = hist1 + kBins1;
  unsigned long long* block_eq = reinterpret_cast<unsigned long long*>(hist2 + kBins2);
  const int sms = g_sms();
  static bool configured = false;
  if (!configured) {
    MOSES_CUDA(cudaFuncSetAttribute(lot_hist1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins1 * 4));
    MOSES_CUDA(cudaFuncSetAttribute(lot_hist2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins2 * 2));
    configured = true;
  }
  lot_init_kernel<<<1, 1, 0, st>>>(S, (unsigned long long)keep);
  const int agrid = std::max<long long>(1, std::min<long long>((n / 4 + 255) / 256, (long long)sms * 16));
  if (mode == 1) {
    lot_max_kernel<<<sms * 2, kPassBlock, 0, st>>>(w, g, n, S);  // 2 x 1024 threads per SM
#define LOT_T(K) lot_apply_kernel<K, true><<<agrid, 256, 0, st>>>(w, g, n, S, theta, alpha, factor, decay, sh.ptr, mask)
    if (sh.kind == 1) LOT_T(1); else if (sh.kind == 2) LOT_T(2); else LOT_T(0);
#undef LOT_T
  } else {
    lot_hist1_kernel<<<sms, kPassBlock, kBins1 * 4, st>>>(w, g, n, hist1);
    lot_pick_kernel<kBins1><<<1, 1024, 0, st>>>(S, hist1, 16, false);
    lot_hist2_kernel<<<sms, kPassBlock, kBins2 * 2, st>>>(w, g, n, S, hist2);
    lot_pick_kernel<kBins2><<<1, 1024, 0, st>>>(S, hist2, 0, true);
    const int nb = std::min(4096, sms * 4);
    const long long chunk = (n + nb - 1) / nb;
    lot_eq_count_kernel<<<nb, kPassBlock, 0, st>>>(w, g, n, chunk, S, block_eq);
    lot_cut_kernel<<<1, kPassBlock, 0, st>>>(w, g, n, chunk, nb, S, block_eq);
#define LOT_R(K) lot_apply_kernel<K, false><<<agrid, 256, 0, st>>>(w, g, n, S, theta, alpha, factor, decay, sh.ptr, mask)
    if (sh.kind == 1) LOT_R(1); else if (sh.kind == 2) LOT_R(2); else LOT_R(0);
#undef LOT_R
  }
  if (popcount_dev) {
    // threshold: the counted kept scalars; ratio: exactly `keep`
    MOSES_CUDA(cudaMemcpyAsync(popcount_dev, &S->count, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
  }
  MOSES_CUDA(cudaGetLastError());
}

}  // namespace moses
