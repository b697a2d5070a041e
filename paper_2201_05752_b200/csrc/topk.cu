// topk.cu — one-pass candidate top-k for large scored pools (search.cpp:32-37 order: score
// descending, then index ascending; select_batch takes the first k, search.cpp:82-95).
//
//   sample  one full 128-byte line (32 scores) at a hashed position in every 2048-score stratum
//           (1/64 of the pool, 1/64 of its bytes) -> order-preserving keys, written compactly
//   tau     the exact key of sample rank r = k/64 + 4 sqrt(k/64) + 16 from the top (the radix
//           select of kernels.cu over the sample): every key >= tau is a candidate (expected ~64 r
//           of them, >= k with overwhelming probability)
//   pass    ONE read of the pool: keys >= tau appended (key, index) with per-warp staging
//   final   one block sorts the <= 16384 candidates by (key desc, index asc) and emits the first k
// If the candidates overflow or fall short of k (adversarial score layouts), the caller runs the
// exact three-pass radix select instead (kernels.cu). Either way the result is the exact top-k:
// the candidate set contains every key >= tau and holds at least k keys, so it contains the top k.
#include <algorithm>
#include <cmath>

#include <cub/block/block_scan.cuh>

#include "kernels.cuh"
#include "ptx.cuh"

namespace moses {
namespace {

constexpr int kTkLine = 32;
constexpr int kTkStratum = 2048;
constexpr int kTkCap = 16384;
constexpr int kTkBlock = 1024;
constexpr int kTkWarpStage = 128;

struct TkState {
  unsigned fail;
  unsigned long long cand_n;
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

__global__ void tk_init_kernel(TkState* st) {
  st->fail = 0;
  st->cand_n = 0;
}

// one warp per stratum: lane l reads score l of the stratum's sampled line (one coalesced 128 B)
__global__ void __launch_bounds__(256) tk_sample_kernel(const float* __restrict__ s, long long n,
                                                        unsigned* __restrict__ keys) {
  const long long strata = n / kTkStratum;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * 8;
  for (long long j = blockIdx.x * 8ll + (threadIdx.x >> 5); j < strata; j += warps) {
    const int line = int(tk_mix(unsigned(j)) % unsigned(kTkStratum / kTkLine));
    keys[j * kTkLine + lane] = tk_key(__ldg(s + j * kTkStratum + line * kTkLine + lane));
  }
}

// the one full pass: every key >= tau appended as (key, index)
__global__ void __launch_bounds__(kTkBlock) tk_pass_kernel(const float* __restrict__ s, long long n, TkState* st,
                                                           const unsigned* __restrict__ tau_key,
                                                           uint2* __restrict__ cand) {
  __shared__ uint2 stage_all[(kTkBlock / 32) * kTkWarpStage];
  const unsigned tau = *tau_key;
  const unsigned lane = threadIdx.x & 31;
  uint2* sc = stage_all + (threadIdx.x >> 5) * kTkWarpStage;
  unsigned cnt = 0;  // warp-uniform
  auto flush = [&]() {
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(&st->cand_n, (unsigned long long)cnt);
    b = __shfl_sync(0xffffffffu, b, 0);
    if (b + cnt <= kTkCap)
      for (unsigned i = lane; i < cnt; i += 32) cand[b + i] = sc[i];
    __syncwarp();
    cnt = 0;
  };
  auto take = [&](float v, long long i, bool ok) {
    const unsigned key = tk_key(v);
    const bool in = ok && key >= tau;
    const unsigned ball = __ballot_sync(0xffffffffu, in);
    if (in) sc[cnt + __popc(ball & ((1u << lane) - 1u))] = make_uint2(key, unsigned(i));
    cnt += __popc(ball);
  };
  const long long n4 = n / 4;
  const long long stride = (long long)gridDim.x * kTkBlock;
  const long long qend = (n4 + kTkBlock - 1) / kTkBlock * kTkBlock;
  long long q = blockIdx.x * (long long)kTkBlock + threadIdx.x;
  float4 a = make_float4(0, 0, 0, 0);
  if (q < n4) a = __ldg(reinterpret_cast<const float4*>(s) + q);
  for (; q < qend; q += stride) {
    const bool ok = q < n4;
    const long long qn = q + stride;
    float4 an = make_float4(0, 0, 0, 0);
    if (qn < n4) an = __ldg(reinterpret_cast<const float4*>(s) + qn);
    take(a.x, 4 * q, ok);
    take(a.y, 4 * q + 1, ok);
    take(a.z, 4 * q + 2, ok);
    take(a.w, 4 * q + 3, ok);
    if (cnt > kTkWarpStage - 128) flush();
    a = an;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // scalar tail (< 4 scores)
    const long long i = 4 * n4 + lane;
    take(i < n ? s[i] : 0.f, i, i < n);
  }
  if (cnt) flush();
}

// one block: exact (key desc, index asc) order of the candidates, first k out
__global__ void __launch_bounds__(kTkBlock) tk_final_kernel(TkState* st, const uint2* __restrict__ cand, long long k,
                                                            unsigned* __restrict__ out_key, long long* __restrict__ out_idx) {
  extern __shared__ uint2 sk[];
  const unsigned long long c = st->cand_n;
  if (st->fail || c > kTkCap || c < (unsigned long long)k) {
    if (threadIdx.x == 0) st->fail = 1;
    return;
  }
  int np = 1;
  while (np < int(c)) np <<= 1;
  for (int t = threadIdx.x; t < np; t += kTkBlock) sk[t] = t < int(c) ? cand[t] : make_uint2(0u, 0xffffffffu);
  __syncthreads();
  for (int size = 2; size <= np; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < np; t += kTkBlock) {
        const int o = t ^ stride;
        if (o > t) {
          const bool first = (t & size) == 0;
          const uint2 x = sk[t], y = sk[o];
          const bool x_before_y = x.x > y.x || (x.x == y.x && x.y < y.y);
          if (x_before_y != first) {
            sk[t] = y;
            sk[o] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < k; t += kTkBlock) {
    out_key[t] = sk[t].x;
    out_idx[t] = (long long)sk[t].y;
  }
}

}  // namespace

static long long tk_samples(long long n) { return n / kTkStratum * kTkLine; }

size_t topk_fast_ws_bytes(long long n) {
  return 256 + size_t(kTkCap) * 8 + select_ws_bytes(std::max(tk_samples(n), 1ll), nullptr) + 1024;
}

bool topk_fast(const float* scores, long long n, long long k, void* ws, unsigned* out_key, long long* out_idx,
               cudaStream_t st) {
  if (n < (1ll << 20) || n >= (1ll << 32) || k > kTopkMax || k <= 0) return false;
  const long long ns = tk_samples(n);
  const double ks = double(k) * double(ns) / double(n);
  const long long r = (long long)std::ceil(ks + 4.0 * std::sqrt(ks) + 16.0);
  if (r > ns) return false;
  uint8_t* p = static_cast<uint8_t*>(ws);
  TkState* S = reinterpret_cast<TkState*>(p);
  uint2* cand = reinterpret_cast<uint2*>(p + 256);
  SelectWs sel;
  select_ws_carve(p + 256 + size_t(kTkCap) * 8, ns, &sel);
  static bool init = false;
  if (!init) {
    MOSES_CUDA(cudaFuncSetAttribute(tk_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTkCap * 8));
    init = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tk_init_kernel<<<1, 1, 0, st>>>(S);
  tk_sample_kernel<<<sms * 8, 256, 0, st>>>(scores, n, sel.keys);
  select_kth_key(ns, (unsigned long long)r, sel, st);
  tk_pass_kernel<<<sms * 2, kTkBlock, 0, st>>>(scores, n, S, sel_result_key(sel), cand);
  tk_final_kernel<<<1, kTkBlock, kTkCap * 8, st>>>(S, cand, k, out_key, out_idx);
  MOSES_CUDA(cudaGetLastError());
  unsigned fail = 1;
  MOSES_CUDA(cudaMemcpyAsync(&fail, &S->fail, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  MOSES_CUDA(cudaStreamSynchronize(st));
  return fail == 0;
}

}  // namespace moses
