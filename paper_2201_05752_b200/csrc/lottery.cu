// lottery.cu — the Moses adaptation step (tuner.cpp:258-262) as few HBM passes as the exact
// selection allows: xi = |w*g| is never materialised, every pass recomputes it from (w, g).
//
//   threshold (lottery.cpp:152-157, normalised): ONE pass (lot_thresh_pass_kernel) + a candidate fix-up,
//     15 B/param. A stratified sample gives max_s <= max(xi), so T_s = thresh_key(max_s) <= T = thresh_key(max)
//     (fl(x / max) <= fl(x / max_s): division rounding is monotone). Keys < T_s are final in the pass
//     (variant: decayed, mask 0); keys >= T_s keep their w, get mask byte 2 and join a candidate list;
//     once the pass has produced the exact max, lot_thresh_fix_kernel resolves only those (or, if the list
//     overflowed, every mask byte still 2). Exact for any input: no estimate can misclassify a scalar.
//   ratio     (lottery.cpp:158-175, top ceil(rho*N), ties by index):
//     pass 1  15-bit histogram of xi bits [30:16] (xi >= 0, so the bit pattern orders like the value)
//     pass 2  16-bit histogram of bits [15:0] within the chosen bucket  -> exact threshold key T
//     pass 3  only if some keys equal to T must be dropped: per-block counts of key == T, then the
//             index of the last kept equal key (ascending-index tie-break, lottery.cpp:169-172)
//     pass 4  fused apply: kept = key > T || (key == T && i <= cut);  w -= alpha*g (kept) /
//             w *= 1 - alpha*lambda (others); operand shadow + mask byte written      31-39 B/param
// vs the algorithmic 15 B/param (read w, g; write w, bf16 shadow, mask byte).
// Large vectors (n >= 16M scalars, w + g beyond L2) take the sampled-bracket variant of pass 2:
//     pass 0  stratified sample (one float4 per 4 KB) -> 15-bit histogram -> bucket bracket
//             [blo, bhi] that holds the keep-th key with a 6-sigma margin
//     pass 1  full 15-bit histogram + compaction of every (key, index) whose bucket is in the
//             bracket (block-aggregated appends)
//     pass 2  16-bit histogram over the compacted candidates only (a few % of n), when the exact
//             bucket b1 from pass 1 lies in the bracket; otherwise the (w, g) pass 2 runs as before
//   so the ratio step reads (w, g) twice instead of three times: ~23 B/param.
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
  unsigned blo, bhi;         // sampled bucket bracket (compaction path); blo > bhi: no compaction
  unsigned long long cand_n; // compacted candidates appended by pass 1
  unsigned long long cand_cap;
  int cand_over;             // pass 1 ran out of candidate space
  int use_cand;              // selection runs over the candidates (set by lot_decide_kernel)
  unsigned long long need0;  // keep
  unsigned long long above;  // keys whose bucket lies above the bracket
  unsigned long long eqc_n;  // candidates with key == T collected for the index cut
  int cut_done;              // the cut was found over the candidates
  unsigned smax_bits;        // threshold: max xi key of the stratified sample (a lower bound of max_bits)
};
static_assert(sizeof(LotState) <= 256, "LotState must fit its workspace slot");

constexpr long long kCandMinN = 1ll << 24;  // compaction path from 16M scalars (w + g = 128 MB > L2)
constexpr int kSampleStride = 256;           // float4 groups per sample stratum (one sample per 4 KB)

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

struct LotState;
__device__ __forceinline__ bool use_cand_of(const LotState* st);
template <bool CHECK>
__global__ void __launch_bounds__(kPassBlock) lot_hist1_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                                               long long n, unsigned* __restrict__ hist,
                                                               const LotState* st) {
  extern __shared__ unsigned sh[];
  if (CHECK && use_cand_of(st)) return;  // the compacted candidates carry the selection
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
__device__ __forceinline__ bool cand_path(const LotState* st);
template <bool CHECK>
__global__ void __launch_bounds__(kPassBlock) lot_hist2_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                                               long long n, const LotState* st,
                                                               unsigned* __restrict__ hist) {
  extern __shared__ unsigned short sh16[];
  __shared__ int s_any;
  if (CHECK && cand_path(st)) return;  // pass 2 already done over the compacted candidates
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

__device__ __forceinline__ unsigned mix32(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// Pass 0: one float4 of (w, g) at a hashed position inside every stratum of kSampleStride groups.
__global__ void __launch_bounds__(kPassBlock) lot_sample_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                                                long long n, unsigned* __restrict__ hist) {
  extern __shared__ unsigned sh[];
  for (int d = threadIdx.x; d < kBins1; d += kPassBlock) sh[d] = 0;
  __syncthreads();
  const long long strata = n / 4 / kSampleStride;
  for (long long j0 = blockIdx.x * (long long)kPassBlock; j0 < strata; j0 += (long long)gridDim.x * kPassBlock) {
    const long long j = j0 + threadIdx.x;
    const bool ok = j < strata;
    float4 a = make_float4(0, 0, 0, 0), b = a;
    if (ok) {
      const long long q = j * kSampleStride + (mix32(unsigned(j)) % kSampleStride);
      a = ld4(w + 4 * q);
      b = ld4(g + 4 * q);
    }
    hist_add(sh, key_of(a.x, b.x) >> 16, ok);
    hist_add(sh, key_of(a.y, b.y) >> 16, ok);
    hist_add(sh, key_of(a.z, b.z) >> 16, ok);
    hist_add(sh, key_of(a.w, b.w) >> 16, ok);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kBins1; d += kPassBlock)
    if (sh[d]) atomicAdd(&hist[d], sh[d]);
}

// One block: bucket bracket [blo, bhi] around the sample rank of the keep-th key (+- 6 sigma + 32).
// Sample ranks are converted to integers once; the two owning threads locate their digits like
// lot_pick_kernel (sum, scan, then one re-read of the owning chunk).
__global__ void __launch_bounds__(1024) lot_bracket_kernel(LotState* st, unsigned* hist, long long n) {
  using Scan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned s_lo, s_hi;
  __shared__ unsigned long long s_above_hi, s_upto_lo;
  constexpr int PER = kBins1 / 1024;
  const uint4* h4 = reinterpret_cast<const uint4*>(hist + kBins1 - PER * (threadIdx.x + 1));
  unsigned long long local = 0;
#pragma unroll 4
  for (int q = 0; q < PER / 4; ++q) {
    const uint4 v = h4[q];
    local += (unsigned long long)v.x + v.y + v.z + v.w;
  }
  unsigned long long before, total;
  Scan(tmp).ExclusiveSum(local, before, total);
  const double frac = double(total) / double(n);
  const double need_s = double(st->need0) * frac;
  const double delta = 6.0 * sqrt(fmax(need_s, 1.0)) + 32.0;
  const long long r_hi = (long long)floor(need_s - delta);  // < 0: bracket open at the top
  const unsigned long long r_lo = (unsigned long long)ceil(need_s + delta);
  if (threadIdx.x == 0) {
    s_lo = 0;
    s_hi = kBins1 - 1;
    s_above_hi = 0;
    s_upto_lo = ~0ull;
  }
  __syncthreads();
  const unsigned* hc = hist + kBins1 - PER * (threadIdx.x + 1);
  // digit holding sample rank r_hi (0-based): before <= r_hi < before + local
  if (r_hi >= 0 && before <= (unsigned long long)r_hi && (unsigned long long)r_hi < before + local) {
    unsigned long long run = before;
    for (int q = PER - 1; q >= 0; --q) {
      const unsigned long long v = hc[q];
      if ((unsigned long long)r_hi < run + v) {
        s_hi = unsigned(kBins1 - PER * (threadIdx.x + 1) + q);
        s_above_hi = run;
        break;
      }
      run += v;
    }
  }
  // digit where the cumulative count reaches r_lo: before < r_lo <= before + local
  if (before < r_lo && r_lo <= before + local) {
    unsigned long long run = before;
    for (int q = PER - 1; q >= 0; --q) {
      const unsigned long long v = hc[q];
      if (r_lo <= run + v) {
        s_lo = unsigned(kBins1 - PER * (threadIdx.x + 1) + q);
        s_upto_lo = run + v;
        break;
      }
      run += v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned lo = s_lo, hi = s_hi;
    const bool found = s_upto_lo != ~0ull;  // r_lo <= total
    const double in = found ? double(s_upto_lo - s_above_hi) : 0.0;  // sampled keys in [lo, hi]
    const double est = in / fmax(frac, 1e-300) * 1.25 + 4096.0;
    const bool ok = total > 0 && found && lo > 0 && lo <= hi && est < double(st->cand_cap);
    st->blo = ok ? lo : 1u;
    st->bhi = ok ? hi : 0u;
  }
  __syncthreads();
  uint4* z4 = reinterpret_cast<uint4*>(hist);
  for (int d = threadIdx.x; d < kBins1 / 4; d += 1024) z4[d] = make_uint4(0, 0, 0, 0);
}

// Pass 1 with compaction: count the keys whose bucket lies above the bracket (register counters)
// and append every (key, index) whose bucket lies in [blo, bhi] to `cand`. Each warp stages its
// appends in its own shared-memory slice and flushes them with one global atomic per 128+ entries,
// so the pass has no block barriers; the next float4 pair is loaded before the current one is
// processed (two loads in flight per thread).
constexpr int kWarpStage = 256;  // entries per warp slice (flush at >= 128: one iteration adds <= 128)
__global__ void __launch_bounds__(kPassBlock) lot_pass1c_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                                                long long n, LotState* st, uint2* __restrict__ cand) {
  extern __shared__ uint2 sc_all[];
  using Red = cub::BlockReduce<unsigned long long, kPassBlock>;
  __shared__ typename Red::TempStorage rtmp;
  const unsigned blo = st->blo, bhi = st->bhi;
  if (blo > bhi) return;  // bracket disabled: the (w, g) histogram passes run instead
  const unsigned lane = threadIdx.x & 31;
  uint2* sc = sc_all + (threadIdx.x >> 5) * kWarpStage;
  const unsigned long long cap = st->cand_cap;
  unsigned cnt = 0;  // warp-uniform
  unsigned long long above = 0;
  auto flush = [&]() {  // warp-collective
    __syncwarp();  // the lanes' staging writes before the copy-out reads them
    unsigned long long b = 0;
    if (lane == 0) {
      b = atomicAdd(&st->cand_n, (unsigned long long)cnt);
      if (b + cnt > cap) st->cand_over = 1;
    }
    b = __shfl_sync(0xffffffffu, b, 0);
    if (b + cnt <= cap)
      for (unsigned i = lane; i < cnt; i += 32) cand[b + i] = sc[i];
    __syncwarp();
    cnt = 0;
  };
  auto take = [&](unsigned key, long long i, bool ok) {  // warp-collective
    const unsigned bk = key >> 16;
    above += (ok && bk > bhi) ? 1u : 0u;
    const bool in = ok && bk >= blo && bk <= bhi;
    const unsigned ball = __ballot_sync(0xffffffffu, in);
    if (in) sc[cnt + __popc(ball & ((1u << lane) - 1u))] = make_uint2(key, unsigned(i));
    cnt += __popc(ball);
  };
  const long long n4 = n / 4;
  const long long stride = (long long)gridDim.x * kPassBlock;
  long long q = blockIdx.x * (long long)kPassBlock + threadIdx.x;
  const long long qend = (n4 + kPassBlock - 1) / kPassBlock * kPassBlock;  // warp-uniform trip count
  float4 a = make_float4(0, 0, 0, 0), b = a;
  if (q < n4) {
    a = ld4(w + 4 * q);
    b = ld4(g + 4 * q);
  }
  for (; q < qend; q += stride) {
    const bool ok = q < n4;
    const long long qn = q + stride;
    float4 an = make_float4(0, 0, 0, 0), bn = an;
    if (qn < n4) {
      an = ld4(w + 4 * qn);
      bn = ld4(g + 4 * qn);
    }
    take(key_of(a.x, b.x), 4 * q, ok);
    take(key_of(a.y, b.y), 4 * q + 1, ok);
    take(key_of(a.z, b.z), 4 * q + 2, ok);
    take(key_of(a.w, b.w), 4 * q + 3, ok);
    if (cnt >= kWarpStage - 128) flush();
    a = an;
    b = bn;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // scalar tail (< 4 scalars), warp 0
    const long long i = 4 * n4 + lane;
    const bool ok = i < n;
    take(ok ? xi_key(w, g, i) : 0u, i, ok);
  }
  if (cnt) flush();
  above = Red(rtmp).Sum(above);
  if (threadIdx.x == 0 && above) atomicAdd(&st->above, above);
}

// Compaction path usable: no overflow and the keep-th key lies among the candidates.
__device__ __forceinline__ bool cand_ok(const LotState* st) {
  return st->blo <= st->bhi && st->cand_over == 0 && st->above < st->need0 && st->need0 - st->above <= st->cand_n;
}

// one thread: set the selection state for whichever path runs
__global__ void lot_decide_kernel(LotState* st) {
  if (cand_ok(st)) {
    st->gt = st->above;
    st->need = st->need0 - st->above;
    st->use_cand = 1;
  } else {
    st->use_cand = 0;
  }
}

// 15-bit bucket histogram over the compacted candidates (compaction path only).
__global__ void __launch_bounds__(kPassBlock) lot_hist1_cand_kernel(const uint2* __restrict__ cand, const LotState* st,
                                                                    unsigned* __restrict__ hist) {
  extern __shared__ unsigned sh[];
  if (!st->use_cand) return;
  for (int d = threadIdx.x; d < kBins1; d += kPassBlock) sh[d] = 0;
  __syncthreads();
  const unsigned long long nc = st->cand_n;
  for (unsigned long long i0 = blockIdx.x * (unsigned long long)kPassBlock; i0 < nc;
       i0 += gridDim.x * (unsigned long long)kPassBlock) {
    const unsigned long long i = i0 + threadIdx.x;
    const bool ok = i < nc;
    hist_add(sh, ok ? (cand[i].x >> 16) : 0u, ok);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kBins1; d += kPassBlock)
    if (sh[d]) atomicAdd(&hist[d], sh[d]);
}

__device__ __forceinline__ bool cand_path(const LotState* st) { return st->use_cand != 0; }
__device__ __forceinline__ bool use_cand_of(const LotState* st) { return st->use_cand != 0; }

// Pass 2 over the compacted candidates (only when the exact bucket b1 lies in the bracket).
__global__ void __launch_bounds__(256) lot_hist2c_kernel(const uint2* __restrict__ cand, const LotState* st,
                                                         unsigned* __restrict__ hist) {
  if (!cand_path(st)) return;
  const unsigned b1 = st->prefix;
  const unsigned long long nc = st->cand_n;
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i - threadIdx.x < nc; i += gridDim.x * 256ull) {
    const bool ok = i < nc;
    const unsigned key = ok ? cand[i].x : 0u;
    const bool in = ok && (key >> kB2) == b1;
    const unsigned d = key & (kBins2 - 1);
    const unsigned d0 = __shfl_sync(0xffffffffu, d, 0);
    if (__all_sync(0xffffffffu, in && d == d0)) {
      if ((threadIdx.x & 31) == 0) atomicAdd(&hist[d0], 32u);
    } else if (in) {
      atomicAdd(&hist[d], 1u);
    }
  }
}

// Single block: choose the digit where the descending cumulative count reaches `need`.
// Thread t owns the PER consecutive digits BINS-1-t*PER ... BINS-PER-t*PER (descending); the bins
// are read twice (sum, then locate) instead of being held in registers.
template <int BINS>
__global__ void __launch_bounds__(1024) lot_pick_kernel(LotState* st, unsigned* hist, int shift, bool last) {
  using Scan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr int PER = BINS / 1024;
  const unsigned long long need = st->need;  // read before any thread updates the state
  const uint4* h4 = reinterpret_cast<const uint4*>(hist + BINS - PER * (threadIdx.x + 1));  // ascending chunk
  unsigned long long local = 0;
#pragma unroll 4
  for (int q = 0; q < PER / 4; ++q) {
    const uint4 v = h4[q];
    local += (unsigned long long)v.x + v.y + v.z + v.w;
  }
  unsigned long long before;
  Scan(tmp).ExclusiveSum(local, before);
  if (before < need && before + local >= need) {  // the crossing digit is in this thread's chunk
    const unsigned* hc = hist + BINS - PER * (threadIdx.x + 1);
    unsigned long long run = before;
    for (int q = PER - 1; q >= 0; --q) {  // descending digits
      const unsigned long long v = hc[q];
      if (run + v >= need) {
        const int d = BINS - PER * (threadIdx.x + 1) + q;
        st->need = need - run;
        st->gt += run;
        st->prefix = shift ? unsigned(d) : ((st->prefix << kB2) | unsigned(d));
        if (last) {
          st->eq = v;
          st->cut = 0x7fffffffffffffffll;
        }
        break;
      }
      run += v;
    }
  }
  __syncthreads();
  uint4* z4 = reinterpret_cast<uint4*>(hist);
  for (int d = threadIdx.x; d < BINS / 4; d += 1024) z4[d] = make_uint4(0, 0, 0, 0);  // ready for the next pass
}

// Ties at T straddling the cut, compaction path: every key == T is a candidate, so collect their
// indices (up to kEqCap) and let one block sort them; the need-th smallest index is the cut.
constexpr int kEqCap = 4096;
__global__ void __launch_bounds__(256) lot_eq_cand_kernel(const uint2* __restrict__ cand, LotState* st,
                                                          unsigned* __restrict__ eq_idx) {
  if (!st->use_cand || st->need >= st->eq || st->eq > kEqCap) return;
  const unsigned T = st->prefix;
  const unsigned long long nc = st->cand_n;
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < nc; i += gridDim.x * 256ull) {
    const uint2 c = cand[i];
    if (c.x == T) {
      const unsigned long long slot = atomicAdd(&st->eqc_n, 1ull);
      if (slot < kEqCap) eq_idx[slot] = c.y;
    }
  }
}

__global__ void __launch_bounds__(1024) lot_cut_cand_kernel(LotState* st, const unsigned* __restrict__ eq_idx) {
  __shared__ unsigned sk[kEqCap];
  if (!st->use_cand || st->need >= st->eq || st->eq > kEqCap || st->eqc_n != st->eq) return;
  const int m = int(st->eq);
  for (int i = threadIdx.x; i < kEqCap; i += 1024) sk[i] = i < m ? eq_idx[i] : 0xffffffffu;
  __syncthreads();
  for (int k = 2; k <= kEqCap; k <<= 1) {  // bitonic sort, ascending
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < kEqCap; i += 1024) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & k) == 0;
          const unsigned x = sk[i], y = sk[p];
          if ((x > y) == up) {
            sk[i] = y;
            sk[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    st->cut = (long long)sk[st->need - 1];
    st->cut_done = 1;
  }
}

// pass 3 (only when ties at T straddle the cut): per-block counts of key == T over fixed chunks
__global__ void __launch_bounds__(kPassBlock) lot_eq_count_kernel(const float* __restrict__ w,
                                                                  const float* __restrict__ g, long long n,
                                                                  long long chunk, const LotState* st,
                                                                  unsigned long long* __restrict__ block_eq) {
  using Red = cub::BlockReduce<unsigned long long, kPassBlock>;
  __shared__ typename Red::TempStorage tmp;
  if (st->need >= st->eq || st->cut_done) return;  // every key equal to T is kept, or cut already found
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
  if (st->need >= st->eq || st->cut_done) return;
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

// Normalised threshold test without a per-scalar division: for top > 0, fl(x / top) is monotone
// non-decreasing in x >= 0, so fl(x / top) > theta  <=>  bits(x) >= K, with K the smallest
// non-negative float bit pattern that passes (31-step binary search, exact __fdiv_rn). top == 0
// means every xi is 0 and xi_scores does not normalise (lottery.cpp:51-55): test x > theta.
__device__ __forceinline__ unsigned thresh_key(float top, float theta) {
  auto pass = [&](unsigned k) {
    const float x = __uint_as_float(k);
    return (top > 0.f ? __fdiv_rn(x, top) : x) > theta;
  };
  unsigned lo = 0, hi = 0x7f800000u;  // +inf
  if (!pass(hi)) return 0x7f800001u;  // nothing passes
  while (lo < hi) {
    const unsigned mid = lo + (hi - lo) / 2;
    if (pass(mid)) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Optimizer of the transferable scalars: plain step w -= alpha*g (transferable_step,
// lottery.cpp:92-97), or masked Adam (the north star's Adam variant; same arithmetic as adam_kernel
// and the oracle's adam_update, no FMA contraction).
struct StepOpt {
  float* m1 = nullptr;  // null: plain step
  float* m2 = nullptr;
  float b1 = 0.f, b2 = 0.f, eps = 0.f, c1 = 1.f, c2 = 1.f;
};
__device__ __forceinline__ float adam_scalar(float wi, float gi, float& m1, float& m2, float lr, const StepOpt& o) {
  const float a = __fadd_rn(__fmul_rn(o.b1, m1), __fmul_rn(__fsub_rn(1.f, o.b1), gi));
  const float b = __fadd_rn(__fmul_rn(o.b2, m2), __fmul_rn(__fsub_rn(1.f, o.b2), __fmul_rn(gi, gi)));
  m1 = a;
  m2 = b;
  const float mh = __fdiv_rn(a, o.c1);
  const float vh = __fdiv_rn(b, o.c2);
  return __fsub_rn(wi, __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), o.eps)));
}

template <int SHADOW, bool THRESH>
__device__ __forceinline__ void lot_apply_one(long long i, float& wi, float gi, unsigned T, long long cut, float top,
                                              float theta, float alpha, float factor, bool decay, uint8_t& mk,
                                              unsigned long long& cnt, const StepOpt& opt, float& m1, float& m2) {
  const float x = fabsf(__fmul_rn(wi, gi));
  bool kept;
  if constexpr (THRESH) {
    kept = __float_as_uint(x) >= T;  // == (xi / max > theta): T = thresh_key(max, theta)
    cnt += kept;
  } else {
    const unsigned key = __float_as_uint(x);
    kept = key > T || (key == T && i <= cut);
  }
  if (kept) wi = opt.m1 ? adam_scalar(wi, gi, m1, m2, alpha, opt)  // masked Adam
                        : __fsub_rn(wi, __fmul_rn(alpha, gi));     // transferable_step (apply_update, no momentum)
  else if (decay) wi = __fmul_rn(wi, factor);                      // variant_decay
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
                                                        uint8_t* __restrict__ mask, const StepOpt opt) {
  using Red = cub::BlockReduce<unsigned long long, 256>;
  __shared__ typename Red::TempStorage tmp;
  __shared__ unsigned s_tk;
  const long long cut = st->cut;
  const float top = __uint_as_float(st->max_bits);
  if constexpr (THRESH) {
    if (threadIdx.x == 0) s_tk = thresh_key(top, theta);
    __syncthreads();
  }
  const unsigned T = THRESH ? s_tk : st->prefix;
  unsigned long long cnt = 0;
  const long long n4 = n / 4;
  for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n4; q += (long long)gridDim.x * 256) {
    const long long i = 4 * q;
    float4 wv = *reinterpret_cast<const float4*>(w + i);
    const float4 gv = ld4(g + i);
    float4 a1 = make_float4(0, 0, 0, 0), a2 = a1;
    if (opt.m1) {
      a1 = *reinterpret_cast<const float4*>(opt.m1 + i);
      a2 = *reinterpret_cast<const float4*>(opt.m2 + i);
    }
    uchar4 mk;
    lot_apply_one<SHADOW, THRESH>(i, wv.x, gv.x, T, cut, top, theta, alpha, factor, decay, mk.x, cnt, opt, a1.x, a2.x);
    lot_apply_one<SHADOW, THRESH>(i + 1, wv.y, gv.y, T, cut, top, theta, alpha, factor, decay, mk.y, cnt, opt, a1.y, a2.y);
    lot_apply_one<SHADOW, THRESH>(i + 2, wv.z, gv.z, T, cut, top, theta, alpha, factor, decay, mk.z, cnt, opt, a1.z, a2.z);
    lot_apply_one<SHADOW, THRESH>(i + 3, wv.w, gv.w, T, cut, top, theta, alpha, factor, decay, mk.w, cnt, opt, a1.w, a2.w);
    if (opt.m1) {
      *reinterpret_cast<float4*>(opt.m1 + i) = a1;
      *reinterpret_cast<float4*>(opt.m2 + i) = a2;
    }
    *reinterpret_cast<float4*>(w + i) = wv;
    *reinterpret_cast<uchar4*>(mask + i) = mk;
    store_shadow4<SHADOW>(shadow, i, wv);
  }
  if (blockIdx.x == 0) {  // scalar tail
    for (long long i = 4 * n4 + threadIdx.x; i < n; i += 256) {
      float wi = w[i];
      uint8_t mk;
      float a1 = opt.m1 ? opt.m1[i] : 0.f, a2 = opt.m1 ? opt.m2[i] : 0.f;
      lot_apply_one<SHADOW, THRESH>(i, wi, g[i], T, cut, top, theta, alpha, factor, decay, mk, cnt, opt, a1, a2);
      if (opt.m1) {
        opt.m1[i] = a1;
        opt.m2[i] = a2;
      }
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
  const long long stride = (long long)gridDim.x * kPassBlock;
  long long q = blockIdx.x * (long long)kPassBlock + threadIdx.x;
  float4 a = make_float4(0, 0, 0, 0), b = a;
  if (q < n4) {
    a = ld4(w + 4 * q);
    b = ld4(g + 4 * q);
  }
  for (; q < n4; q += stride) {  // next pair loaded before the current one is reduced
    const long long qn = q + stride;
    float4 an = make_float4(0, 0, 0, 0), bn = an;
    if (qn < n4) {
      an = ld4(w + 4 * qn);
      bn = ld4(g + 4 * qn);
    }
    m = max(max(max(m, key_of(a.x, b.x)), key_of(a.y, b.y)), max(key_of(a.z, b.z), key_of(a.w, b.w)));
    a = an;
    b = bn;
  }
  if (blockIdx.x == 0)
    for (long long i = 4 * n4 + threadIdx.x; i < n; i += kPassBlock) m = max(m, xi_key(w, g, i));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(&st->max_bits, m);
}

// ---------------------------------------------------------------- threshold step: one (w, g) pass
// Sample max over one float4 of (w, g) per stratum (lot_sample_kernel's positions): a lower bound of max.
__global__ void __launch_bounds__(kPassBlock) lot_tsample_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                                                 long long n, LotState* st) {
  unsigned m = 0;
  const long long strata = n / 4 / kSampleStride;
  for (long long j = blockIdx.x * (long long)kPassBlock + threadIdx.x; j < strata; j += (long long)gridDim.x * kPassBlock) {
    const long long q = j * kSampleStride + (mix32(unsigned(j)) % kSampleStride);
    const float4 a = ld4(w + 4 * q), b = ld4(g + 4 * q);
    m = max(max(max(m, key_of(a.x, b.x)), key_of(a.y, b.y)), max(key_of(a.z, b.z), key_of(a.w, b.w)));
  }
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(&st->smax_bits, m);
}

// The pass: every scalar read once; keys below T_s finished (decay / mask 0 / shadow), the rest left as
// candidates (w and its shadow rewritten unchanged so every line is written whole, mask byte 2, index
// appended warp-aggregated to `cand`); the exact max accumulated with atomicMax.
template <int SHADOW>
__global__ void __launch_bounds__(256) lot_thresh_pass_kernel(float* __restrict__ w, const float* __restrict__ g,
                                                              long long n, LotState* st, float theta, float factor,
                                                              bool decay, void* __restrict__ shadow,
                                                              uint8_t* __restrict__ mask, unsigned* __restrict__ cand) {
  __shared__ unsigned s_ts;
  if (threadIdx.x == 0) {
    const unsigned sm = st->smax_bits;
    s_ts = sm == 0 ? 0u : thresh_key(__uint_as_float(sm), theta);  // max_s == 0: no bound, all candidates
  }
  __syncthreads();
  const unsigned Ts = s_ts;
  const unsigned long long cap = st->cand_cap;
  const unsigned lane = threadIdx.x & 31;
  unsigned m = 0;
  auto one = [&](float& wi, float gi, uint8_t& mk, long long i) {  // warp-collective (append)
    const unsigned key = __float_as_uint(fabsf(__fmul_rn(wi, gi)));
    m = max(m, key);
    const bool c = key >= Ts && i < n;
    if (!c && decay) wi = __fmul_rn(wi, factor);
    mk = c ? 2 : 0;
    const unsigned ball = __ballot_sync(0xffffffffu, c);
    if (ball) {
      unsigned long long b = 0;
      if (lane == 0) {
        b = atomicAdd(&st->cand_n, (unsigned long long)__popc(ball));
        if (b + __popc(ball) > cap) st->cand_over = 1;
      }
      b = __shfl_sync(0xffffffffu, b, 0);
      const unsigned long long slot = b + __popc(ball & ((1u << lane) - 1u));
      if (c && slot < cap) cand[slot] = unsigned(i);
    }
  };
  const long long n4 = n / 4;
  const long long qend = (n4 + 255) / 256 * 256;  // warp-uniform trip count (the ballots)
  for (long long q = blockIdx.x * 256ll + threadIdx.x; q < qend; q += (long long)gridDim.x * 256) {
    const bool ok = q < n4;
    const long long i = 4 * q;
    float4 wv = make_float4(0, 0, 0, 0), gv = wv;
    if (ok) {
      wv = *reinterpret_cast<const float4*>(w + i);
      gv = ld4(g + i);
    }
    uchar4 mk;
    one(wv.x, gv.x, mk.x, ok ? i : n);
    one(wv.y, gv.y, mk.y, ok ? i + 1 : n);
    one(wv.z, gv.z, mk.z, ok ? i + 2 : n);
    one(wv.w, gv.w, mk.w, ok ? i + 3 : n);
    if (ok) {
      *reinterpret_cast<float4*>(w + i) = wv;
      *reinterpret_cast<uchar4*>(mask + i) = mk;
      store_shadow4<SHADOW>(shadow, i, wv);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // scalar tail (< 4 scalars), warp 0
    const long long i = 4 * n4 + lane;
    float wi = i < n ? w[i] : 0.f;
    const float gi = i < n ? g[i] : 0.f;
    uint8_t mk;
    one(wi, gi, mk, i < n ? i : n);
    if (i < n) {
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
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0 && m) atomicMax(&st->max_bits, m);
}

// Candidates against the exact T = thresh_key(max, theta): the same per-scalar step as lot_apply_one.
// List mode (no overflow): grid-stride over cand[0, cand_n). Overflow: grid-stride over the mask bytes.
template <int SHADOW>
__global__ void __launch_bounds__(256) lot_thresh_fix_kernel(float* __restrict__ w, const float* __restrict__ g,
                                                             long long n, LotState* st, float theta, float alpha,
                                                             float factor, bool decay, void* __restrict__ shadow,
                                                             uint8_t* __restrict__ mask, const unsigned* __restrict__ cand,
                                                             const StepOpt opt) {
  using Red = cub::BlockReduce<unsigned long long, 256>;
  __shared__ typename Red::TempStorage tmp;
  __shared__ unsigned s_t;
  if (threadIdx.x == 0) s_t = thresh_key(__uint_as_float(st->max_bits), theta);
  __syncthreads();
  const unsigned T = s_t;
  unsigned long long cnt = 0;
  auto fix = [&](long long i) {
    float wi = w[i];
    float a1 = opt.m1 ? opt.m1[i] : 0.f, a2 = opt.m1 ? opt.m2[i] : 0.f;
    uint8_t mk;
    lot_apply_one<SHADOW, true>(i, wi, g[i], T, 0, 0.f, theta, alpha, factor, decay, mk, cnt, opt, a1, a2);
    if (opt.m1) {
      opt.m1[i] = a1;
      opt.m2[i] = a2;
    }
    w[i] = wi;
    mask[i] = mk;
    if constexpr (SHADOW == 1) static_cast<__nv_bfloat16*>(shadow)[i] = __float2bfloat16_rn(wi);
    if constexpr (SHADOW == 2) {
      uint32_t t;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(wi));
      static_cast<float*>(shadow)[i] = __uint_as_float(t);
    }
  };
  const long long stride = (long long)gridDim.x * 256;
  if (!st->cand_over) {
    const long long nc = (long long)st->cand_n;
    for (long long k = blockIdx.x * 256ll + threadIdx.x; k < nc; k += stride) fix(cand[k]);
  } else {
    const long long n16 = n / 16;
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n16; q += stride) {
      const uint4 v = *reinterpret_cast<const uint4*>(mask + 16 * q);
      const unsigned words[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (words[b] & 0x02020202u)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if ((words[b] >> (8 * e)) & 2u) fix(16 * q + 4 * b + e);
    }
    for (long long i = 16 * n16 + blockIdx.x * 256ll + threadIdx.x; i < n; i += stride)
      if (mask[i] == 2) fix(i);
  }
  cnt = Red(tmp).Sum(cnt);
  if (threadIdx.x == 0 && cnt) atomicAdd(&st->count, cnt);
}

// ---------------------------------------------------------------- single-launch resident step
// For the cost model's own parameter counts (P <= 148 x 512 x 16 ~ 1.2M; the 4x512 model has
// 872,961) the whole step is ONE cooperative launch: every thread keeps its <= 16 (w, g) pairs in
// registers, so HBM/L2 see exactly one read of (w, g) and one write of (w, mask, shadow) — the
// algorithmic 15 B/param — and the selection runs between grid barriers instead of kernel launches:
//   ratio:      3 radix digits (11/11/10 bits of the xi key; block histograms -> global, every block
//               re-derives the chosen digit from the global histogram), then the ties at T are
//               ranked in index order through per-block equal counts, then the fused apply;
//   threshold:  block max -> global max, then the fused apply (popcount accumulated).
// Block b owns indices [b*chunk, (b+1)*chunk); thread t holds b*chunk + j*512 + t, j < E.
constexpr int kResThreads = 512, kResE = 16;

struct ResState {
  unsigned bar_count, bar_gen;
  unsigned max_bits;
  unsigned long long count;
  unsigned hist1[2048], hist2[2048], hist3[1024];
  unsigned long long block_eq[1024];
};

__device__ unsigned long long g_res_trace[8];  // CTA 0's phase stamps (globaltimer), debug read-out
__device__ __forceinline__ void res_stamp(int k) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    g_res_trace[k] = v;
  }
}

// acquire/release grid barrier (no full fences, no back-off sleep: the whole grid is resident)
__device__ __forceinline__ void res_grid_sync(ResState* st) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g0, arrived;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(&st->bar_gen) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(&st->bar_count) : "memory");
    if (arrived == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(&st->bar_count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&st->bar_gen) : "memory");
    } else {
      unsigned gg;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gg) : "l"(&st->bar_gen) : "memory");
      } while (gg == g0);
    }
  }
  __syncthreads();
}

// every block: descending cumulative over `bins` global counts -> the digit where it reaches `need`
template <int BINS>
__device__ __forceinline__ void res_pick(const unsigned* hist, unsigned long long need, unsigned* s_digit,
                                         unsigned long long* s_before) {
  using Scan = cub::BlockScan<unsigned long long, kResThreads>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr int PER = BINS / kResThreads;  // 2 or 1, descending digits per thread
  unsigned long long v[PER], local = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    v[q] = __ldcg(hist + (BINS - 1 - (threadIdx.x * PER + q)));
    local += v[q];
  }
  unsigned long long before;
  Scan(tmp).ExclusiveSum(local, before);
  unsigned long long run = before;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (run < need && run + v[q] >= need) {
      *s_digit = unsigned(BINS - 1 - (threadIdx.x * PER + q));
      *s_before = run;
    }
    run += v[q];
  }
  __syncthreads();
}

template <int SHADOW, bool THRESH>
__global__ void __launch_bounds__(kResThreads, 1)
    lot_resident_kernel(float* __restrict__ w, const float* __restrict__ g, long long n, long long chunk, int E,
                        unsigned long long keep, float theta, float alpha, float factor, bool decay,
                        void* __restrict__ shadow, long long lo_off, uint8_t* __restrict__ mask, ResState* st,
                        unsigned long long* popcount_out, const StepOpt opt) {
  __shared__ unsigned sh[2048];
  __shared__ unsigned s_digit;
  __shared__ unsigned long long s_before;
  using Red = cub::BlockReduce<unsigned long long, kResThreads>;
  __shared__ typename Red::TempStorage rtmp;
  res_stamp(0);
  const long long base = blockIdx.x * chunk;
  float wv[kResE], gv[kResE];
#pragma unroll
  for (int j = 0; j < kResE; ++j) {
    const long long i = base + (long long)j * kResThreads + threadIdx.x;
    const bool ok = j < E && i < n && i < base + chunk;
    wv[j] = ok ? w[i] : 0.f;
    gv[j] = ok ? __ldg(g + i) : 0.f;
  }
  auto valid = [&](int j) {
    const long long i = base + (long long)j * kResThreads + threadIdx.x;
    return j < E && i < n && i < base + chunk;
  };
  unsigned T = 0;
  unsigned long long need_eq = 0, eq_total = 0;  // ratio: keys == T still to keep / present
  float top = 0.f;
  if (blockIdx.x == 0) {  // buffers first written after the first barrier
    for (int d = threadIdx.x; d < 2048; d += kResThreads) st->hist2[d] = 0;
    for (int d = threadIdx.x; d < 1024; d += kResThreads) st->hist3[d] = 0;
    if (threadIdx.x == 0) st->count = 0;
  }
  if constexpr (THRESH) {
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < kResE; ++j)
      if (valid(j)) m = max(m, key_of(wv[j], gv[j]));
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(&st->max_bits, m);
    res_grid_sync(st);
    top = __uint_as_float(__ldcg(&st->max_bits));
  } else {
    // digit 1: bits [31:21]
    for (int d = threadIdx.x; d < 2048; d += kResThreads) sh[d] = 0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kResE; ++j)
      if (valid(j)) atomicAdd(&sh[key_of(wv[j], gv[j]) >> 21], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < 2048; d += kResThreads)
      if (sh[d]) atomicAdd(&st->hist1[d], sh[d]);
    res_grid_sync(st);
    res_stamp(1);
    res_pick<2048>(st->hist1, keep, &s_digit, &s_before);
    const unsigned d1 = s_digit;
    unsigned long long need = keep - s_before;
    // digit 2: bits [20:10] among keys with digit 1 == d1
    for (int d = threadIdx.x; d < 2048; d += kResThreads) sh[d] = 0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kResE; ++j) {
      const unsigned k = key_of(wv[j], gv[j]);
      if (valid(j) && (k >> 21) == d1) atomicAdd(&sh[(k >> 10) & 2047u], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 2048; d += kResThreads)
      if (sh[d]) atomicAdd(&st->hist2[d], sh[d]);
    res_grid_sync(st);
    res_stamp(2);
    if (blockIdx.x == 0)  // every block has read hist1 (before the barrier): clear it for the next call
      for (int d = threadIdx.x; d < 2048; d += kResThreads) st->hist1[d] = 0;
    res_pick<2048>(st->hist2, need, &s_digit, &s_before);
    const unsigned p2 = (d1 << 11) | s_digit;
    need -= s_before;
    // digit 3: bits [9:0] among keys with bits [31:10] == p2
    for (int d = threadIdx.x; d < 1024; d += kResThreads) sh[d] = 0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kResE; ++j) {
      const unsigned k = key_of(wv[j], gv[j]);
      if (valid(j) && (k >> 10) == p2) atomicAdd(&sh[k & 1023u], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 1024; d += kResThreads)
      if (sh[d]) atomicAdd(&st->hist3[d], sh[d]);
    res_grid_sync(st);
    res_stamp(3);
    res_pick<1024>(st->hist3, need, &s_digit, &s_before);
    T = (p2 << 10) | s_digit;
    need_eq = need - s_before;
    eq_total = __ldcg(&st->hist3[s_digit]);
    if (need_eq < eq_total) {  // ties at T straddle the cut: rank them in index order
      unsigned long long c = 0;
#pragma unroll
      for (int j = 0; j < kResE; ++j) c += (valid(j) && key_of(wv[j], gv[j]) == T) ? 1u : 0u;
      c = Red(rtmp).Sum(c);
      if (threadIdx.x == 0) st->block_eq[blockIdx.x] = c;
      res_grid_sync(st);
    }
  }
  res_stamp(4);
  // ---- fused apply (the same per-scalar arithmetic as lot_apply_kernel)
  unsigned long long eq_before = 0;  // keys == T in lower-indexed blocks
  if (!THRESH && need_eq < eq_total) {
    unsigned long long c = 0;
    for (int b = threadIdx.x; b < int(blockIdx.x); b += kResThreads) c += __ldcg(&st->block_eq[b]);
    eq_before = Red(rtmp).Sum(c);
    if (threadIdx.x == 0) s_before = eq_before;
    __syncthreads();
    eq_before = s_before;
  }
  using ScanU = cub::BlockScan<unsigned, kResThreads>;
  __shared__ typename ScanU::TempStorage stmp;
  unsigned long long cnt = 0;
#pragma unroll
  for (int j = 0; j < kResE; ++j) {
    const long long i = base + (long long)j * kResThreads + threadIdx.x;
    const bool ok = valid(j);
    bool kept = false;
    const float x = fabsf(__fmul_rn(wv[j], gv[j]));
    if constexpr (THRESH) {
      const float xn = top > 0.f ? __fdiv_rn(x, top) : x;
      kept = ok && xn > theta;
      cnt += kept;
    } else {
      const unsigned key = __float_as_uint(x);
      const bool eq = ok && key == T;
      if (need_eq < eq_total) {  // block-ordered rank of this equal key (index order: j, then t)
        unsigned r, tot;
        ScanU(stmp).ExclusiveSum(eq ? 1u : 0u, r, tot);
        kept = ok && (key > T || (eq && eq_before + r < need_eq));
        eq_before += tot;
        __syncthreads();
      } else {
        kept = ok && key >= T;
      }
    }
    if (ok) {
      float wi = wv[j];
      if (kept) {
        if (opt.m1) {  // masked Adam
          float a1 = opt.m1[i], a2 = opt.m2[i];
          wi = adam_scalar(wi, gv[j], a1, a2, alpha, opt);
          opt.m1[i] = a1;
          opt.m2[i] = a2;
        } else {
          wi = __fsub_rn(wi, __fmul_rn(alpha, gv[j]));
        }
      } else if (decay) {
        wi = __fmul_rn(wi, factor);
      }
      w[i] = wi;
      mask[i] = kept ? 1 : 0;
      if constexpr (SHADOW == 1) static_cast<__nv_bfloat16*>(shadow)[i] = __float2bfloat16_rn(wi);
      if constexpr (SHADOW == 2) {
        uint32_t tt;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(tt) : "f"(wi));
        static_cast<float*>(shadow)[i] = __uint_as_float(tt);
      }
      if constexpr (SHADOW == 3) {  // 3xTF32 pair (kernels.cu store_operand<float>)
        uint32_t hh, ll;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hh) : "f"(wi));
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(ll) : "f"(wi - __uint_as_float(hh)));
        static_cast<float*>(shadow)[i] = __uint_as_float(hh);
        static_cast<float*>(shadow)[i + lo_off] = __uint_as_float(ll);
      }
      if constexpr (SHADOW == 4) {  // split bf16 pair (kernels.cu store_shadow<4>)
        const __nv_bfloat16 hb = __float2bfloat16_rn(wi);
        static_cast<__nv_bfloat16*>(shadow)[i] = hb;
        static_cast<__nv_bfloat16*>(shadow)[i + lo_off] = __float2bfloat16_rn(wi - __bfloat162float(hb));
      }
    }
  }
  res_stamp(5);
  if constexpr (THRESH) {
    cnt = Red(rtmp).Sum(cnt);
    if (threadIdx.x == 0 && cnt) atomicAdd(&st->count, cnt);
    res_grid_sync(st);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (popcount_out) *popcount_out = st->count;
      st->max_bits = 0;  // ready for the next call
    }
  }
}

static size_t res_state_bytes() { return (sizeof(ResState) + 255) / 256 * 256; }

__global__ void lot_init_kernel(LotState* st, unsigned long long keep, unsigned long long cap) {
  st->need = keep;
  st->blo = 1;
  st->bhi = 0;
  st->cand_n = 0;
  st->cand_cap = cap;
  st->cand_over = 0;
  st->use_cand = 0;
  st->need0 = keep;
  st->above = 0;
  st->eqc_n = 0;
  st->cut_done = 0;
  st->gt = 0;
  st->eq = 0;
  st->prefix = 0;
  st->max_bits = 0;
  st->smax_bits = 0;
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

static long long cand_capacity(long long n) { return n >= kCandMinN ? n / 16 + 65536 : 0; }

size_t lottery_ws_bytes(long long n) {
  return res_state_bytes() + 256 /*state*/ + size_t(kBins1) * 4 * 2 /*hist1, sample hist*/ + size_t(kBins2) * 4 +
         size_t(4096) * 8 + size_t(kEqCap) * 4 +
         size_t(cand_capacity(n)) * 8 + 1024;
}

// Fused Moses step. mode 1 threshold (normalised, strict), 2 ratio (top `keep`, index tie-break).
int lottery_step_fused(float* w, const float* g, long long n, int mode, float theta, long long keep, float alpha,
                       float factor, bool decay, Shadow sh, uint8_t* mask, void* ws, unsigned long long* popcount_dev,
                       cudaStream_t st, const AdamOpt* adam) {
  StepOpt opt;
  if (adam) {
    opt.m1 = adam->m1;
    opt.m2 = adam->m2;
    opt.b1 = adam->b1;
    opt.b2 = adam->b2;
    opt.eps = adam->eps;
    opt.c1 = adam->c1;
    opt.c2 = adam->c2;
  }
  ResState* R = static_cast<ResState*>(ws);  // zeroed at allocation; every call leaves it reusable
  uint8_t* p = static_cast<uint8_t*>(ws) + res_state_bytes();
  LotState* S = reinterpret_cast<LotState*>(p);
  unsigned* hist1 = reinterpret_cast<unsigned*>(p + 256);
  unsigned* hist2 = hist1 + kBins1;
  unsigned long long* block_eq = reinterpret_cast<unsigned long long*>(hist2 + kBins2);
  unsigned* hist_s = reinterpret_cast<unsigned*>(block_eq + 4096);
  unsigned* eq_idx = hist_s + kBins1;
  uint2* cand = reinterpret_cast<uint2*>(eq_idx + kEqCap);
  const long long cap = cand_capacity(n);
  const bool compact = mode != 1 && cap > 0 && n < (1ll << 32);
  const int sms = g_sms();
  static bool configured = false;
  if (!configured) {
    MOSES_CUDA(cudaFuncSetAttribute(lot_hist2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins2 * 2));
    MOSES_CUDA(cudaFuncSetAttribute(lot_hist2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins2 * 2));
    MOSES_CUDA(cudaFuncSetAttribute(lot_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins1 * 4));
    MOSES_CUDA(cudaFuncSetAttribute(lot_hist1_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins1 * 4));
    MOSES_CUDA(cudaFuncSetAttribute(lot_hist1_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins1 * 4));
    MOSES_CUDA(cudaFuncSetAttribute(lot_hist1_cand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins1 * 4));
    MOSES_CUDA(cudaFuncSetAttribute(lot_pass1c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (kPassBlock / 32) * kWarpStage * 8));
    configured = true;
  }
  // the cost model's own sizes: one cooperative launch with register-resident (w, g)
  if (n <= (long long)sms * kResThreads * kResE && n >= 1) {
    const long long chunk = (n + sms - 1) / sms;
    const int E = int((chunk + kResThreads - 1) / kResThreads);
    unsigned long long* pop = popcount_dev;
    const unsigned long long ukeep = (unsigned long long)keep;
    void* shp = sh.ptr;
    long long lo_off = sh.kind == 3 ? shadow_lo_offset(n) : sh.lo_off;
    int grid = sms;
    StepOpt o = opt;
    void* args[] = {&w,   (void*)&g, &n,    (void*)&chunk, (void*)&E, (void*)&ukeep, &theta, &alpha, &factor,
                    &decay, &shp,    &lo_off, &mask,        &R,        &pop,          &o};
    const void* fns[2][5] = {{(const void*)lot_resident_kernel<0, false>, (const void*)lot_resident_kernel<1, false>,
                              (const void*)lot_resident_kernel<2, false>, (const void*)lot_resident_kernel<3, false>,
                              (const void*)lot_resident_kernel<4, false>},
                             {(const void*)lot_resident_kernel<0, true>, (const void*)lot_resident_kernel<1, true>,
                              (const void*)lot_resident_kernel<2, true>, (const void*)lot_resident_kernel<3, true>,
                              (const void*)lot_resident_kernel<4, true>}};
    const void* fn = fns[mode == 1 ? 1 : 0][sh.kind >= 0 && sh.kind <= 4 ? sh.kind : 0];
    MOSES_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kResThreads), args, 0, st));
    MOSES_CUDA(cudaGetLastError());
    return 1;
  }
  // threshold mode: the candidate list holds 32-bit indices in the (key, index) pair buffer (2x the entries)
  const long long tcap = n < (1ll << 32) ? 2 * cap : 0;
  lot_init_kernel<<<1, 1, 0, st>>>(S, (unsigned long long)keep, (unsigned long long)(mode == 1 ? tcap : cap));
  const int agrid = std::max<long long>(1, std::min<long long>((n / 4 + 255) / 256, (long long)sms * 16));
  if (mode == 1) {  // one (w, g) pass + candidate fix-up (module comment)
    unsigned* tcand = reinterpret_cast<unsigned*>(cand);
    lot_tsample_kernel<<<sms, kPassBlock, 0, st>>>(w, g, n, S);
    const int pgrid = std::max<long long>(1, std::min<long long>((n / 4 + 255) / 256, (long long)sms * 8));
#define LOT_T(K)                                                                                                \
  lot_thresh_pass_kernel<K><<<pgrid, 256, 0, st>>>(w, g, n, S, theta, factor, decay, sh.ptr, mask, tcand);      \
  lot_thresh_fix_kernel<K><<<sms * 4, 256, 0, st>>>(w, g, n, S, theta, alpha, factor, decay, sh.ptr, mask, tcand, opt)
    if (sh.kind == 1) { LOT_T(1); } else if (sh.kind == 2) { LOT_T(2); } else { LOT_T(0); }
#undef LOT_T
  } else {
    if (compact) {
      lot_sample_kernel<<<sms, kPassBlock, kBins1 * 4, st>>>(w, g, n, hist_s);
      lot_bracket_kernel<<<1, 1024, 0, st>>>(S, hist_s, n);
      lot_pass1c_kernel<<<sms * 2, kPassBlock, (kPassBlock / 32) * kWarpStage * 8, st>>>(w, g, n, S, cand);
      lot_decide_kernel<<<1, 1, 0, st>>>(S);
      lot_hist1_kernel<true><<<sms, kPassBlock, kBins1 * 4, st>>>(w, g, n, hist1, S);      // fallback only
      lot_hist1_cand_kernel<<<sms, kPassBlock, kBins1 * 4, st>>>(cand, S, hist1);          // fast path only
      lot_pick_kernel<kBins1><<<1, 1024, 0, st>>>(S, hist1, 16, false);
      lot_hist2c_kernel<<<sms * 8, 256, 0, st>>>(cand, S, hist2);                          // fast path only
      lot_hist2_kernel<true><<<sms, kPassBlock, kBins2 * 2, st>>>(w, g, n, S, hist2);      // fallback only
    } else {
      lot_hist1_kernel<false><<<sms, kPassBlock, kBins1 * 4, st>>>(w, g, n, hist1, S);
      lot_pick_kernel<kBins1><<<1, 1024, 0, st>>>(S, hist1, 16, false);
      lot_hist2_kernel<false><<<sms, kPassBlock, kBins2 * 2, st>>>(w, g, n, S, hist2);
    }
    lot_pick_kernel<kBins2><<<1, 1024, 0, st>>>(S, hist2, 0, true);
    if (compact) {
      lot_eq_cand_kernel<<<sms * 4, 256, 0, st>>>(cand, S, eq_idx);
      lot_cut_cand_kernel<<<1, 1024, 0, st>>>(S, eq_idx);
    }
    const int nb = 4096;  // chunks for the general tie cut (block_eq capacity)
    const long long chunk = (n + nb - 1) / nb;
    lot_eq_count_kernel<<<nb, kPassBlock, 0, st>>>(w, g, n, chunk, S, block_eq);
    lot_cut_kernel<<<1, kPassBlock, 0, st>>>(w, g, n, chunk, nb, S, block_eq);
#define LOT_R(K) lot_apply_kernel<K, false><<<agrid, 256, 0, st>>>(w, g, n, S, theta, alpha, factor, decay, sh.ptr, mask, opt)
    if (sh.kind == 1) LOT_R(1); else if (sh.kind == 2) LOT_R(2); else LOT_R(0);
#undef LOT_R
  }
  if (popcount_dev) {
    // threshold: the counted kept scalars; ratio: exactly `keep`
    MOSES_CUDA(cudaMemcpyAsync(popcount_dev, &S->count, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
  }
  MOSES_CUDA(cudaGetLastError());
  if (sh.kind >= 3) refresh_shadow(w, n, sh, st);  // split operand pairs: not written by the pass kernels
  return (mode == 1 ? 4 : (compact ? 16 : 8)) + (sh.kind >= 3 ? 1 : 0);  // kernels launched
}

void lottery_res_trace_read(unsigned long long* out8) {
  MOSES_CUDA(cudaMemcpyFromSymbol(out8, g_res_trace, sizeof(unsigned long long) * 8));
}

}  // namespace moses
