// topk.cu — one-launch candidate top-k for large scored pools (search.cpp:32-37 order: score
// descending, then index ascending; select_batch takes the first k, search.cpp:82-95).
//
// ONE cooperative kernel, phases separated by grid barriers:
//   sample  one full 128-byte line (32 scores) at a hashed position in every 2048-score stratum
//           (1/64 of the pool, 1/64 of its bytes) -> order-preserving keys, kept, and a histogram of
//           their top 13 bits
//   tau     the key of sample rank r = k/64 + 4 sqrt(k/64) + 16 from the top, to as many further
//           digit levels (11, 8 bits) over the sampled keys of the chosen prefix as needed; every key
//           >= tau is a candidate (expected ~64 r of them, >= k with overwhelming probability)
//   pass    ONE read of the pool (4 float4 loads in flight per thread): keys >= tau appended as
//           (key, index) through per-warp staging
//   final   exact rank of every candidate by counting the candidates that precede it in
//           (key desc, index asc) order — (candidate block, comparison chunk) items over every warp,
//           partial counts summed with integer atomics — and the first k written at their ranks
// If the candidates overflow or fall short of k (adversarial score layouts), the kernel raises a flag
// and the caller runs the exact three-pass radix select instead (kernels.cu). Either way the result is
// the exact top-k: the candidate set holds every key >= tau and at least k keys, so it holds the top k.
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include <cub/block/block_scan.cuh>

#include "kernels.cuh"
#include "ptx.cuh"

namespace moses {
namespace {

constexpr int kTkLine = 32;
constexpr int kTkStratum = 2048;
constexpr int kTkCap = 16384;
constexpr int kTkThreads = 1024;
constexpr int kTkWarps = kTkThreads / 32;
constexpr int kTkWarpStage = 128;
constexpr int kTkBits0 = 13, kTkBits1 = 11, kTkBits2 = 8;  // digit levels over the 32-bit key
constexpr int kTkBins0 = 1 << kTkBits0, kTkBins1 = 1 << kTkBits1, kTkBins2 = 1 << kTkBits2;
constexpr int kTkHist = kTkBins0 + kTkBins1 + kTkBins2;
constexpr int kTkDynSmem = kTkCap * 8;  // >= the pass staging (kTkWarps * kTkWarpStage * 8)
static_assert(kTkDynSmem >= kTkWarps * kTkWarpStage * 8, "staging");
// a digit level is enough once at most this many sampled keys lie at or above its bucket's lower bound
// (~64x as many candidates expected: ~10K of the 16K candidate capacity). The 13-bit level 0
// (1/16-octave buckets) usually settles a normal pool's top-1024 threshold alone (5.4K candidates
// instead of 3.7K after a second level): with the grid-wide exact-rank phase on composite keys that
// is 95 vs 96 us per call over 100M scores.
constexpr unsigned kTkLoose = 160;

// Persistent per device, zero between launches: allocated zeroed once, and every launch restores it (the
// grid barrier's arrival count returns to 0 at each barrier, the histograms are cleared once their last
// reader has passed the barrier after the pass, and launches alternate between two candidate counters,
// each cleared during the other's launch), so a call is one launch with no memset in front of it.
struct TkState {
  unsigned bar[2];  // grid barrier: arrivals, generation
  unsigned parity;  // which candidate counter this launch uses (the other is cleared for the next)
  unsigned pad;
  unsigned long long cand_n[2];
  unsigned hist[kTkHist];  // level 0 | level 1 | level 2
};

__device__ __forceinline__ unsigned tk_key(float f) {  // larger float -> larger key (kernels.cu float_key_desc)
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ unsigned tk_mix(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__device__ unsigned long long g_tk_trace[16];  // CTA 0's phase stamps (globaltimer), debug read-out
__device__ __forceinline__ void tk_stamp(int k) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    g_tk_trace[k] = v;
  }
}

__device__ __forceinline__ void tk_grid_sync(unsigned* bar) {  // bar[0] arrivals, bar[1] generation
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

// shared histogram increment of digit d for the lanes with `in` (plain shared atomics: warp aggregation
// with match.any measured slower — its issue rate, not the address conflicts, bounds the sample phase)
__device__ __forceinline__ void tk_hist_add(unsigned* h, bool in, unsigned d) {
  if (in) atomicAdd(h + d, 1u);
}

// the digit holding descending rank `need` (1-based) of a global histogram of NB bins:
// out[0] = digit, out[1] = its rank within the digit, out[2] = keys at or above the digit's lower bound
template <int NB>
__device__ __forceinline__ void tk_pick(const unsigned* gh, unsigned need, unsigned* out, void* scan_tmp) {
  using Scan = cub::BlockScan<unsigned, kTkThreads>;
  constexpr int PER = NB >= kTkThreads ? NB / kTkThreads : 1;
  unsigned c[PER], tot = 0;
#pragma unroll
  for (int u = 0; u < PER; ++u) {  // bins in descending digit order
    const int b = int(threadIdx.x) * PER + u;
    c[u] = b < NB ? __ldcg(gh + (NB - 1 - b)) : 0u;
    tot += c[u];
  }
  unsigned excl;
  Scan(*reinterpret_cast<typename Scan::TempStorage*>(scan_tmp)).ExclusiveSum(tot, excl);
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    if (excl < need && need <= excl + c[u]) {
      out[0] = unsigned(NB - 1 - (int(threadIdx.x) * PER + u));
      out[1] = need - excl;
      out[2] = excl + c[u];
    }
    excl += c[u];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kTkThreads, 1)
    tk_fused_kernel(const float* __restrict__ s, long long n, long long k, unsigned r, TkState* st,
                    unsigned* __restrict__ keys, uint2* __restrict__ cand, unsigned* __restrict__ ranks,
                    unsigned* __restrict__ out_key,
                    long long* __restrict__ out_idx, unsigned* __restrict__ fail_out) {
  __shared__ unsigned h[kTkBins0];
  extern __shared__ __align__(16) uint2 dyn[];  // pass: per-warp staging; final: the candidates
  uint2* stage_all = dyn;
  __shared__ __align__(16) unsigned char scan_tmp[sizeof(typename cub::BlockScan<unsigned, kTkThreads>::TempStorage)];
  __shared__ unsigned sel[3];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const long long strata = n / kTkStratum;
  const long long ns = strata * kTkLine;

  tk_stamp(0);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_tk_trace[9] = ~0ull;
    g_tk_trace[10] = 0;
  }
  for (int i = int(blockIdx.x) * kTkThreads + t; i < kTkCap; i += int(gridDim.x) * kTkThreads) ranks[i] = 0;
  const unsigned par = __ldcg(&st->parity);
  unsigned long long* cand_n = &st->cand_n[par];
  // ---- sample + histogram of the top kTkBits0 key bits
  for (int i = t; i < kTkBins0; i += kTkThreads) h[i] = 0;
  __syncthreads();
  {  // SU strata per warp in flight (each line is one dependent HBM round trip otherwise)
    constexpr int SU = 8;
    const long long gw = (long long)gridDim.x * kTkWarps;
    const long long jend = (strata + gw * SU - 1) / (gw * SU) * (gw * SU);  // whole warps iterate together
    for (long long j0 = blockIdx.x * (long long)kTkWarps + warp; j0 < jend; j0 += gw * SU) {
      float v[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const long long j = j0 + u * gw;
        const int line = int(tk_mix(unsigned(j)) % unsigned(kTkStratum / kTkLine));
        v[u] = j < strata ? __ldg(s + j * kTkStratum + line * kTkLine + lane) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const long long j = j0 + u * gw;
        const bool ok = j < strata;
        const unsigned key = tk_key(v[u]);
        if (ok) keys[j * kTkLine + lane] = key;
        tk_hist_add(h, ok, key >> (32 - kTkBits0));
      }
    }
  }
  tk_stamp(7);
  __syncthreads();
  for (int i = t; i < kTkBins0; i += kTkThreads)
    if (h[i]) atomicAdd(&st->hist[i], h[i]);
  tk_grid_sync(st->bar);
  tk_stamp(1);

  // ---- tau: the sample key of rank r to as many digit levels (13, 11, 8 bits) as the candidate count
  // needs — the lower bound of the bucket holding it once few enough sampled keys lie at or above that
  // bound (a lower tau only adds candidates), the exact key after all three levels
  tk_pick<kTkBins0>(st->hist, r, sel, scan_tmp);
  unsigned prefix = sel[0], need = sel[1], ge = sel[2];
  int bits = kTkBits0;
  const long long gt = (long long)gridDim.x * kTkThreads;
  const long long q4 = ns / 4;
  constexpr int LU = 4;  // sampled-key loads in flight per thread
  const long long qend = (q4 + gt * LU - 1) / (gt * LU) * (gt * LU);
  int lev = 1;
  for (; lev <= 2 && ge > kTkLoose; ++lev) {
    const int shift = 32 - bits;  // prefix bits are key >> shift
    const int dbits = lev == 1 ? kTkBits1 : kTkBits2;
    const unsigned dmask = (1u << dbits) - 1u;
    const int dshift = shift - dbits;
    unsigned* gh = st->hist + (lev == 1 ? kTkBins0 : kTkBins0 + kTkBins1);
    for (int i = t; i <= int(dmask); i += kTkThreads) h[i] = 0;
    __syncthreads();
    for (long long q0 = blockIdx.x * (long long)kTkThreads + t; q0 < qend; q0 += gt * LU) {
      uint4 v[LU];
#pragma unroll
      for (int u = 0; u < LU; ++u) {
        const long long q = q0 + u * gt;
        v[u] = q < q4 ? __ldcg(reinterpret_cast<const uint4*>(keys) + q) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < LU; ++u) {
        const bool ok = q0 + u * gt < q4;
        tk_hist_add(h, ok && (v[u].x >> shift) == prefix, (v[u].x >> dshift) & dmask);
        tk_hist_add(h, ok && (v[u].y >> shift) == prefix, (v[u].y >> dshift) & dmask);
        tk_hist_add(h, ok && (v[u].z >> shift) == prefix, (v[u].z >> dshift) & dmask);
        tk_hist_add(h, ok && (v[u].w >> shift) == prefix, (v[u].w >> dshift) & dmask);
      }
    }
    __syncthreads();
    for (int i = t; i <= int(dmask); i += kTkThreads)
      if (h[i]) atomicAdd(gh + i, h[i]);
    tk_grid_sync(st->bar);
    tk_stamp(1 + lev);
    if (lev == 1) tk_pick<kTkBins1>(gh, need, sel, scan_tmp);
    else tk_pick<kTkBins2>(gh, need, sel, scan_tmp);
    prefix = (prefix << dbits) | sel[0];
    ge = (r - need) + sel[2];  // keys above the previous bucket + those at or above this one's bound in it
    need = sel[1];
    bits += dbits;
  }
  for (; lev <= 2; ++lev) tk_stamp(1 + lev);
  const unsigned tau = bits == 32 ? prefix : prefix << (32 - bits);

  // ---- the one full pass: every key >= tau appended as (key, index)
  {
    uint2* sc = stage_all + warp * kTkWarpStage;
    unsigned cnt = 0;  // warp-uniform
    auto flush = [&]() {
      __syncwarp();  // the lanes' staging writes before the copy-out reads them
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(cand_n, (unsigned long long)cnt);
      b = __shfl_sync(0xffffffffu, b, 0);
      if (b + cnt <= kTkCap)
        for (unsigned i = lane; i < cnt; i += 32) cand[b + i] = sc[i];
      __syncwarp();
      cnt = 0;
    };
    auto take4 = [&](float4 a, long long i0, bool ok) {  // the 4 scores of one float4
      const unsigned k0 = tk_key(a.x), k1 = tk_key(a.y), k2 = tk_key(a.z), k3 = tk_key(a.w);
      const bool any = ok && (max(max(k0, k1), max(k2, k3)) >= tau);
      if (!__any_sync(0xffffffffu, any)) return;
      const unsigned kk[4] = {k0, k1, k2, k3};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool in = ok && kk[u] >= tau;
        const unsigned ball = __ballot_sync(0xffffffffu, in);
        if (in) sc[cnt + __popc(ball & ((1u << lane) - 1u))] = make_uint2(kk[u], unsigned(i0 + u));
        cnt += __popc(ball);
      }
      if (cnt > kTkWarpStage - 128) flush();
    };
    // chunks of U * kTkThreads float4 (64 KB), grid-strided (handing the last quarter out dynamically
    // balanced the CTAs' end times but its per-chunk barriers cost more than the imbalance)
    const long long n4 = n / 4;
    constexpr int U = 4;
    const long long nch = (n4 + U * kTkThreads - 1) / (U * kTkThreads);
    for (long long ch = blockIdx.x; ch < nch; ch += gridDim.x) {
      float4 a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long q = (ch * U + u) * kTkThreads + t;
        a[u] = q < n4 ? __ldcs(reinterpret_cast<const float4*>(s) + q) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long q = (ch * U + u) * kTkThreads + t;
        take4(a[u], 4 * q, q < n4);
      }
    }
    if (blockIdx.x == 0 && warp == 0) {  // scalar tail (< 4 scores)
      const long long i = 4 * n4 + lane;
      const bool ok = i < n;
      const unsigned key = ok ? tk_key(s[i]) : 0u;
      const bool in = ok && key >= tau;
      const unsigned ball = __ballot_sync(0xffffffffu, in);
      if (in) sc[cnt + __popc(ball & ((1u << lane) - 1u))] = make_uint2(key, unsigned(i));
      cnt += __popc(ball);
    }
    if (cnt) flush();
  }
  tk_stamp(4);
  if (threadIdx.x == 0) {  // earliest / latest pass end over the CTAs
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    atomicMin(&g_tk_trace[9], v);
    atomicMax(&g_tk_trace[10], v);
  }
  tk_grid_sync(st->bar);
  tk_stamp(5);
  // every CTA is past its last histogram read: clear them for the next launch
  for (int i = blockIdx.x * kTkThreads + t; i < kTkHist; i += gridDim.x * kTkThreads) st->hist[i] = 0;
  if (blockIdx.x == 0 && t == 0) {  // every CTA read `parity` at its start: the next launch uses the other
    st->cand_n[par ^ 1u] = 0;       // counter (unused by this one), so this one's needs no clearing barrier
    st->parity = par ^ 1u;
  }

  // ---- exact ranks of the candidates; the first k out
  if (t == 0) sel[0] = unsigned(min(__ldcg(cand_n), (unsigned long long)kTkCap + 1));
  __syncthreads();
  const unsigned c = sel[0];
  if (blockIdx.x == 0 && t == 0) g_tk_trace[8] = c;
  if (c > unsigned(kTkCap) || c < unsigned(k)) {
    if (blockIdx.x == 0 && t == 0) *fail_out = 1;
    return;
  }
  if (blockIdx.x == 0 && t == 0) *fail_out = 0;
  const int cn = int(c);
  // (block of 32 candidates, chunk of the comparisons) items over every warp of the grid: lanes own
  // candidates, each item counts the candidates of its chunk that precede them, the partial counts meet
  // in ranks[] (atomics: integer sums, any order) — then one barrier and the first k written at their ranks
  const int cb_n = (cn + 31) / 32;
  const int gw = int(gridDim.x) * kTkWarps;
  const int jc_n = max(1, gw / cb_n);
  const int items = cb_n * jc_n;
  if (int(blockIdx.x) * kTkWarps < items) {  // CTA-uniform
    // order-composite keys: (key << 32) | ~index is larger exactly when the candidate comes first
    unsigned long long* comp = reinterpret_cast<unsigned long long*>(dyn);
    for (int i = t; i < cn; i += kTkThreads) {
      const uint2 v = __ldcg(cand + i);
      comp[i] = (static_cast<unsigned long long>(v.x) << 32) | static_cast<unsigned long long>(~v.y);
    }
    __syncthreads();
    for (int it = int(blockIdx.x) * kTkWarps + warp; it < items; it += gw) {
      const int cb = it / jc_n, jc = it - cb * jc_n;
      const int i = cb * 32 + lane;
      const unsigned long long me = i < cn ? comp[i] : ~0ull;
      const int j0 = int((long long)cn * jc / jc_n), j1 = int((long long)cn * (jc + 1) / jc_n);
      unsigned before = 0;
#pragma unroll 8
      for (int j = j0; j < j1; ++j) before += comp[j] > me ? 1u : 0u;  // one address per warp: a broadcast
      if (i < cn && before) atomicAdd(ranks + i, before);
    }
  }
  tk_grid_sync(st->bar);
  for (int i = int(blockIdx.x) * kTkThreads + t; i < cn; i += int(gridDim.x) * kTkThreads) {
    const unsigned rank = __ldcg(ranks + i);
    if (rank < unsigned(k)) {
      const uint2 me = __ldcg(cand + i);
      out_key[rank] = me.x;
      out_idx[rank] = (long long)me.y;
    }
  }
  tk_stamp(6);
}

int tk_grid() {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 148, per = 0;
    MOSES_CUDA(cudaGetDevice(&dev));
    MOSES_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MOSES_CUDA(cudaFuncSetAttribute(tk_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTkDynSmem));
    MOSES_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tk_fused_kernel, kTkThreads, kTkDynSmem));
    grid = sms * std::max(per, 1);
  }
  return grid;
}

}  // namespace

void topk_trace_read(unsigned long long* out16) {
  MOSES_CUDA(cudaMemcpyFromSymbol(out16, g_tk_trace, sizeof(unsigned long long) * 16));
}

static long long tk_samples(long long n) { return n / kTkStratum * kTkLine; }

size_t topk_fast_ws_bytes(long long n) {  // [flag word | candidates | ranks | sampled keys]
  return 256 + size_t(kTkCap) * 12 + size_t(std::max(tk_samples(n), 1ll)) * 4 + 256;
}

static TkState* tk_state() {
  constexpr int kMaxDev = 64;
  static TkState* st[kMaxDev] = {};
  int dev = 0;
  MOSES_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) throw std::runtime_error("device ordinal out of range");
  if (!st[dev]) {
    TkState* p = nullptr;
    MOSES_CUDA(cudaMalloc(&p, sizeof(TkState)));
    MOSES_CUDA(cudaMemset(p, 0, sizeof(TkState)));
    MOSES_CUDA(cudaDeviceSynchronize());
    st[dev] = p;
  }
  return st[dev];
}

bool topk_fast_launch(const float* scores, long long n, long long k, void* ws, unsigned* out_key, long long* out_idx,
                      unsigned* fail_out, cudaStream_t st) {
  if (n < (1ll << 20) || n >= (1ll << 32) || k > kTopkMax || k <= 0) return false;
  const long long ns = tk_samples(n);
  const double ks = double(k) * double(ns) / double(n);
  const long long r = (long long)std::ceil(ks + 4.0 * std::sqrt(ks) + 16.0);
  if (r > ns) return false;
  TkState* S = tk_state();
  uint8_t* p = static_cast<uint8_t*>(ws) + 256;
  uint2* cand = reinterpret_cast<uint2*>(p);
  unsigned* ranks = reinterpret_cast<unsigned*>(p + size_t(kTkCap) * 8);
  unsigned* keys = ranks + kTkCap;
  unsigned ru = unsigned(r);
  void* args[] = {(void*)&scores, (void*)&n,   (void*)&k,       (void*)&ru,      (void*)&S,       (void*)&keys,
                  (void*)&cand,   (void*)&ranks, (void*)&out_key, (void*)&out_idx, (void*)&fail_out};
  const int grid = tk_grid();
  MOSES_CUDA(cudaLaunchCooperativeKernel((const void*)tk_fused_kernel, dim3(grid), dim3(kTkThreads), args, kTkDynSmem, st));
  return true;
}

bool topk_fast(const float* scores, long long n, long long k, void* ws, unsigned* out_key, long long* out_idx,
               cudaStream_t st) {
  unsigned* fail_dev = static_cast<unsigned*>(ws);
  if (!topk_fast_launch(scores, n, k, ws, out_key, out_idx, fail_dev, st)) return false;
  unsigned fail = 1;
  MOSES_CUDA(cudaMemcpyAsync(&fail, fail_dev, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  MOSES_CUDA(cudaStreamSynchronize(st));
  return fail == 0;
}

}  // namespace moses
