// gemm_wgrad_sk.cuh — split-bf16 weight gradients of every level in one launch, split over the batch
// rows (K) inside thread-block clusters.
//
//   G_l [(dims_l + 1) x dims_{l+1}] = [act_l | 1]^T dZ_{l+1}     (K = rows of the batch)
//   with every operand a bf16 (hi, lo) pair: G = A_hi B_hi + A_hi B_lo + A_lo B_hi  (model.cpp:113-119)
//
// Why (profiles/r2 timelines): wgrad_group_split_kernel runs one CTA per 128 x 64 tile over ALL batch
// rows — 136 CTAs at cfg2, 56 at cfg5 — and each k-block moves 96 KB of 16 KB boxes for 768 MMA
// cycles, so the per-SM TMA ingest (profiles/r2/tma_ingest_bench.json) sets the pace: 32 us at cfg2,
// 44 us at cfg5. Here a CTA owns a 128 x 256 tile (MMA N = 256: 1536 MMA cycles per 96 KB stage, under
// the ~100 B/clk the TMA reaches with two issuing warps and >= 64 KB stages), and the S CTAs of a
// cluster split the tile's rows. Each keeps its fp32 partial in shared memory; after a cluster
// barrier CTA s sums rows [s*128/S, (s+1)*128/S) of all S partials over DSMEM in split order (fixed
// order: deterministic) and runs the update epilogue (gemm_group.cuh arithmetic) on them.
//
// Bias rows. A level whose input width is a multiple of 128 would need a fifth 128-row M tile for its
// single bias row (the ones column of act_l). Instead, the drain warps of that level's CTAs sum the
// dZ hi/lo columns of every stage on the CUDA cores while the tensor core works — m-tile j of an
// n-tile takes columns [j*bias_w, (j+1)*bias_w) of it (fp32, fixed row order within a split, split
// order across the cluster).
//
// Precision: TMEM chunks of kChunkKb k-blocks (128 rows) are promoted into fp32 registers by the drain
// warps while the next chunk accumulates (double-buffered, 2 x 256 TMEM columns), as in
// wgrad_group_split_kernel.
//
// 352 threads: warps 0-7 drain / epilogue (warp w: TMEM lanes 32(w%4).., columns 128(w/4)..),
// warp 8 TMA producer of the hi planes, warp 9 of the lo planes, warp 10 MMA issuer.
#pragma once
#include "gemm_group.cuh"

namespace moses {

struct WgskCfg {
  // BK = 32 rows per stage, 4 stages: the ring is TMA-latency bound (an operand block lands ~2K cycles
  // after issue), so more, smaller stages in flight beat 2 x 96 KB (1.9-2.0K cycles per 64 rows measured)
  static constexpr int BM = 128, BN = 256, BK = 32;
  static constexpr int kBox = 64 * BK * 2;              // one 64-element MN chunk x BK rows: 4 KB
  static constexpr int kABytes = BM * BK * 2;           // 8 KB per plane
  static constexpr int kBBytes = BN * BK * 2;           // 16 KB per plane
  static constexpr int kHalfStage = kABytes + kBBytes;  // A and B of one plane: 48 KB
  static constexpr int kStageBytes = 2 * kHalfStage;    // [A_hi | B_hi | A_lo | B_lo]: 48 KB
  static constexpr int kStages = 4;
  static constexpr int kChunkKb = 4;                    // 128 rows per TMEM chunk
  static constexpr int kPad = BN + 4;                   // fp32 partial row stride (float4 stores conflict-free)
  static constexpr int kPartBytes = BM * kPad * 4;      // 133,120 B, reuses the stage memory
  static constexpr int kThreads = 352;
  static constexpr int kDrainThreads = 256;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
  static_assert(kPartBytes + (2 * kDrainThreads + BN) * 4 <= kStages * kStageBytes, "partial tile must fit the stage memory");
};

struct WgskArgs {
  GroupArgs ga;                   // levels, K, tile table (tiles_n counts BN = 256 tiles), outputs
  int S;                          // CTAs per cluster = splits of K per tile
  int Mg[kGroupMax];              // G rows the MMA tiles produce (dims + 1, or dims when bias_sep)
  int bias_sep[kGroupMax];        // bias row summed on the CUDA cores (dims % 128 == 0)
  int bias_row[kGroupMax];        // G row index of the bias (= dims_l)
  int bias_w[kGroupMax];          // bias columns per m-tile (even, divides BN; BN: m-tile 0 only)
  int kc;                         // k-blocks per TMEM chunk (promotion interval)
  float* ws;                      // S > 1: L2 workspace, one slot of kSlotFloats per CTA
  unsigned long long* trace;      // optional: clock64 stamps of block 0 (tools/wgsk_trace.py)
};

constexpr int kSlotFloats = WgskCfg::BM * WgskCfg::BN + WgskCfg::BN;  // partial tile + bias sums
constexpr int kWgskMaxCtas = 148;

namespace wgsk {
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_cluster_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// shared -> global bulk copy (bulk_group completion); global -> shared bulk copy (mbarrier complete_tx)
__device__ __forceinline__ void bulk_store(float* gdst, const float* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(ptx::smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(float* sdst, const float* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// g[e] = gv; UPDATE: v = mu*v + g; w -= lr*v (no FMA contraction; sgd_kernel arithmetic) and the
// (hi, lo) bf16 operand shadow of w.
template <bool UPDATE>
__device__ __forceinline__ void store1(const GroupArgs& a, int lev, long long e, float gv) {
  a.g[lev][e] = gv;
  if constexpr (UPDATE) {
    const float vi = __fadd_rn(__fmul_rn(a.mu, a.mom[lev][e]), gv);
    const float wi = __fsub_rn(a.w[lev][e], __fmul_rn(a.lr, vi));
    a.mom[lev][e] = vi;
    a.w[lev][e] = wi;
    const __nv_bfloat16 h = __float2bfloat16_rn(wi);
    a.shadow[lev][e] = h;
    a.shadow_lo[lev][e] = __float2bfloat16_rn(wi - __bfloat162float(h));
  }
}
template <bool UPDATE>
__device__ __forceinline__ void store4(const GroupArgs& a, int lev, long long e, float4 gv, float4 w0, float4 v0) {
  float* __restrict__ g = a.g[lev];
  *reinterpret_cast<float4*>(g + e) = gv;
  if constexpr (UPDATE) {
    float* __restrict__ w = a.w[lev];
    float* __restrict__ v = a.mom[lev];
    float4 vo, wo;
    auto upd = [&](float gi, float vi0, float wi0, float& vi, float& wi) {
      vi = __fadd_rn(__fmul_rn(a.mu, vi0), gi);
      wi = __fsub_rn(wi0, __fmul_rn(a.lr, vi));
    };
    upd(gv.x, v0.x, w0.x, vo.x, wo.x);
    upd(gv.y, v0.y, w0.y, vo.y, wo.y);
    upd(gv.z, v0.z, w0.z, vo.z, wo.z);
    upd(gv.w, v0.w, w0.w, vo.w, wo.w);
    *reinterpret_cast<float4*>(v + e) = vo;
    *reinterpret_cast<float4*>(w + e) = wo;
    const __nv_bfloat162 p0 = __floats2bfloat162_rn(wo.x, wo.y), p1 = __floats2bfloat162_rn(wo.z, wo.w);
    const __nv_bfloat162 l0 = __floats2bfloat162_rn(wo.x - __low2float(p0), wo.y - __high2float(p0));
    const __nv_bfloat162 l1 = __floats2bfloat162_rn(wo.z - __low2float(p1), wo.w - __high2float(p1));
    uint2 ph, pl;
    ph.x = *reinterpret_cast<const uint32_t*>(&p0);
    ph.y = *reinterpret_cast<const uint32_t*>(&p1);
    pl.x = *reinterpret_cast<const uint32_t*>(&l0);
    pl.y = *reinterpret_cast<const uint32_t*>(&l1);
    *reinterpret_cast<uint2*>(a.shadow[lev] + e) = ph;
    *reinterpret_cast<uint2*>(a.shadow_lo[lev] + e) = pl;
  }
}
}  // namespace wgsk

template <bool UPDATE>
__global__ void __launch_bounds__(WgskCfg::kThreads, 1)
    wgrad_sk_kernel(const __grid_constant__ GroupMapsSplit maps, const __grid_constant__ WgskArgs args) {
  using C = WgskCfg;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK;
  const int KC = args.kc;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*BF16*/, true, true, BM, BN);
  const GroupArgs& ga = args.ga;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* bfull = empty_bar + C::kStages;  // [2] TMEM buffer holds a finished chunk
  uint64_t* bempty = bfull + 2;              // [2] drain warps consumed the buffer
  uint64_t* gbar = bempty + 2;               // S > 1: the S slot slices of this CTA's rows have landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbar + 1);

  const int S = args.S;
  const int tile = int(blockIdx.x) / S, split = int(blockIdx.x) % S;  // split == %cluster_ctarank
  int lev = 0;
  while (lev + 1 < ga.n && tile >= ga.tile_begin[lev + 1]) ++lev;
  const int local = tile - ga.tile_begin[lev];
  const int m0 = (local / ga.tiles_n[lev]) * BM, n0 = (local % ga.tiles_n[lev]) * BN;
  const int N = ga.N[lev];
  const int bias_w = args.bias_w[lev];
  const int bias_c0 = (m0 / BM) * bias_w;  // this CTA's bias columns [bias_c0, bias_c0 + bias_w) of the tile
  const bool bias_here = args.bias_sep[lev] != 0 && bias_c0 < BN;

  // this split's k-blocks: whole 128-row chunks
  const int kb_total = (ga.K + BK - 1) / BK;
  const int ch_total = (kb_total + KC - 1) / KC;
  const int kb_begin = (split * ch_total / S) * KC;
  const int kb_end = min(((split + 1) * ch_total / S) * KC, kb_total);
  const int nkb = max(0, kb_end - kb_begin);
  const int nchunks = (nkb + KC - 1) / KC;

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full_bar[s], 2);                      // one expect_tx arrival per plane producer
      ptx::mbar_init(&empty_bar[s], bias_here ? 1 + 8 : 1);  // MMA commit (+ the 8 bias-summing warps)
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&bfull[b], 1);
      ptx::mbar_init(&bempty[b], 8);
    }
    ptx::mbar_init(gbar, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(tmem_slot);
  if (args.trace && blockIdx.x == 0 && threadIdx.x == 0) args.trace[130] = clock64();
  if (args.trace && threadIdx.x == 0 && blockIdx.x < 148) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    args.trace[131 + 2 * blockIdx.x] = t;
  }
  ptx::pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 320) {  // step bookkeeping folded into the step's last kernel
    if (ga.counter != nullptr) *ga.counter += 1;
    if (ga.loss_acc != nullptr) *ga.loss_acc += *ga.loss_src;
    if (ga.loss_copy != nullptr) *ga.loss_copy = *ga.loss_src;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  float* part = reinterpret_cast<float*>(smem);                                  // [BM][kPad]
  float* bpart = reinterpret_cast<float*>(smem + C::kPartBytes);  // [k-groups][bias_w]: 2 * kDrainThreads floats
  float* btot = bpart + 2 * C::kDrainThreads;                                       // [BN]

  if (warp == 8 || warp == 9) {
    if (lane == 0) {
      const int plane = int(warp) - 8;
      const CUtensorMap* tA = plane ? &maps.a_lo[lev] : &maps.a[lev];
      const CUtensorMap* tB = plane ? &maps.b_lo[lev] : &maps.b[lev];
      ptx::tma_prefetch_desc(tA);
      ptx::tma_prefetch_desc(tB);
      for (int i = 0; i < nkb; ++i) {
        const int stage = i % C::kStages;
        const uint32_t phase = uint32_t(i / C::kStages) & 1u;
        ptx::mbar_wait(&empty_bar[stage], phase ^ 1u);
        uint8_t* base = smem + stage * C::kStageBytes + plane * C::kHalfStage;
        if (args.trace && blockIdx.x == 0 && i < 32) args.trace[plane * 32 + i] = clock64();
        ptx::mbar_arrive_expect_tx(&full_bar[stage], C::kHalfStage);
        const int k0 = (kb_begin + i) * BK;
        ptx::tma_load_2d(base, tA, &full_bar[stage], m0, k0);
        ptx::tma_load_2d(base + C::kBox, tA, &full_bar[stage], m0 + 64, k0);
#pragma unroll
        for (int j = 0; j < BN / 64; ++j)
          ptx::tma_load_2d(base + C::kABytes + j * C::kBox, tB, &full_bar[stage], n0 + 64 * j, k0);
      }
    }
    __syncwarp();
  } else if (warp == 10) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int stage = i % C::kStages;
        const uint32_t phase = uint32_t(i / C::kStages) & 1u;
        const int c = i / KC, buf = c & 1;
        const bool first = (i % KC) == 0;
        if (first && c >= 2) {
          ptx::mbar_wait(&bempty[buf], uint32_t((c - 2) >> 1) & 1u);  // chunk c-2 drained
          ptx::tc_fence_after();
        }
        ptx::mbar_wait(&full_bar[stage], phase);
        ptx::tc_fence_after();
        if (args.trace && blockIdx.x == 0 && i < 32) args.trace[64 + i] = clock64();
        const uint32_t sa = ptx::smem_u32(smem + stage * C::kStageBytes);
        const uint32_t sb = sa + C::kABytes, sal = sa + C::kHalfStage, sbl = sal + C::kABytes;
        const uint32_t tacc = tmem_base + uint32_t(buf * BN);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t ah = ptx::sw128_desc(sa + kk * 2048, C::kBox, 1024, 2);
          const uint64_t bh = ptx::sw128_desc(sb + kk * 2048, C::kBox, 1024, 2);
          const uint64_t al = ptx::sw128_desc(sal + kk * 2048, C::kBox, 1024, 2);
          const uint64_t bl = ptx::sw128_desc(sbl + kk * 2048, C::kBox, 1024, 2);
          // small terms first: they never dominate the running sum's exponent
          ptx::umma_f16(tacc, ah, bl, kIdesc, (!first || kk > 0) ? 1u : 0u);
          ptx::umma_f16(tacc, al, bh, kIdesc, 1u);
          ptx::umma_f16(tacc, ah, bh, kIdesc, 1u);
        }
        ptx::umma_commit(&empty_bar[stage]);
        if ((i % KC) == KC - 1 || i == nkb - 1) ptx::umma_commit(&bfull[buf]);
      }
    }
    __syncwarp();
  } else {
    // drain warps
    const uint32_t q = warp & 3u, h = warp >> 2;
    const int row = int(q * 32 + lane);
    const uint32_t t_row = tmem_base + ((q * 32u) << 16) + h * 128u;
    float acc[128];
#pragma unroll
    for (int j = 0; j < 128; ++j) acc[j] = 0.f;
    // bias: thread t sums columns bias_c0 + 2cp, +1 over its k-group of every stage
    const int t = int(threadIdx.x);
    const int pairs = bias_w >> 1, kgroups = C::kDrainThreads / max(pairs, 1), krows = BK / max(kgroups, 1);
    const int cp = t % max(pairs, 1), kh = t / max(pairs, 1);
    const int bcol = bias_c0 + 2 * cp, bchunk = bcol >> 6, nc = bcol & 63;
    float bs0 = 0.f, bs1 = 0.f;
    int i = 0;
    for (int c = 0; c < nchunks; ++c) {
      if (bias_here) {
        const int iend = min(nkb, (c + 1) * KC);
        for (; i < iend; ++i) {
          const int stage = i % C::kStages;
          ptx::mbar_wait(&full_bar[stage], uint32_t(i / C::kStages) & 1u);
          const uint32_t bh = ptx::smem_u32(smem + stage * C::kStageBytes + C::kABytes) + uint32_t(bchunk * C::kBox);
          const uint32_t bl = bh + C::kHalfStage;
          if (kh < kgroups) {
            for (int kr = 0; kr < krows; ++kr) {
              const int k = kh * krows + kr;
              const uint32_t off = uint32_t(k * 128 + ((((nc >> 3) ^ (k & 7)) << 4) | ((nc & 7) * 2)));
              uint32_t vh, vl;
              asm volatile("ld.shared.b32 %0, [%1];" : "=r"(vh) : "r"(bh + off));
              asm volatile("ld.shared.b32 %0, [%1];" : "=r"(vl) : "r"(bl + off));
              const __nv_bfloat162 h2 = *reinterpret_cast<const __nv_bfloat162*>(&vh);
              const __nv_bfloat162 l2 = *reinterpret_cast<const __nv_bfloat162*>(&vl);
              bs0 += __low2float(h2) + __low2float(l2);  // hi + lo is exact in fp32
              bs1 += __high2float(h2) + __high2float(l2);
            }
          }
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&empty_bar[stage]);
        }
      }
      const int buf = c & 1;
      ptx::mbar_wait(&bfull[buf], uint32_t(c >> 1) & 1u);
      ptx::tc_fence_after();
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(t_row + uint32_t(buf * BN + qq * 32), r);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[qq * 32 + j] += __uint_as_float(r[j]);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bempty[buf]);
      if (args.trace && blockIdx.x == 0 && threadIdx.x == 0 && c < 32) args.trace[96 + c] = clock64();
    }
    if (args.trace && blockIdx.x == 0 && threadIdx.x == 0) args.trace[128] = clock64();
    ptx::pdl_launch_dependents();
    wgsk::named_sync(1, C::kDrainThreads);  // every stage read (MMAs and bias sums) before reuse
    float* prow = part + row * C::kPad + h * 128;
#pragma unroll
    for (int j = 0; j < 128; j += 4)
      *reinterpret_cast<float4*>(prow + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    if (bias_here) {  // k-groups combined in order: btot[j] = sum of column bias_c0 + j
      if (kh < kgroups) {
        bpart[kh * bias_w + 2 * cp] = bs0;
        bpart[kh * bias_w + 2 * cp + 1] = bs1;
      }
      wgsk::named_sync(1, C::kDrainThreads);
      if (t < bias_w) {
        float sum = 0.f;
        for (int g = 0; g < kgroups; ++g) sum += bpart[g * bias_w + t];
        btot[t] = sum;
      }
    }
    wgsk::named_sync(1, C::kDrainThreads);
  }

  // ---- split reduction. S > 1: every CTA publishes its partial (and bias sums) to its slot of the
  // L2 workspace with bulk copies (TMA engine, one 1 KB row each; LSU stores and DSMEM both move only
  // ~20-25 B/clk per SM); after the cluster barrier CTA `split` bulk-loads rows [r0, r1) of the S slots
  // into shared memory, sums them in split order and runs the epilogue.
  const int r0 = split * BM / S, r1 = (split + 1) * BM / S;
  float* gbuf = reinterpret_cast<float*>(smem);  // S > 1: [S][r1 - r0][BN], over the published partial
  const float* slots = args.ws + size_t(tile) * size_t(S) * kSlotFloats;
  if (S > 1) {
    float* slot = args.ws + size_t(blockIdx.x) * kSlotFloats;
    if (threadIdx.x < C::kDrainThreads) {
      if (bias_here && int(threadIdx.x) < bias_w) slot[BM * BN + threadIdx.x] = btot[threadIdx.x];
      wgsk::fence_proxy_async_smem();  // the partial's generic smem writes -> the bulk copies' reads
      wgsk::named_sync(1, C::kDrainThreads);
      if (lane == 0) {  // warp w: rows [16w, 16w + 16)
        for (int r = int(warp) * 16; r < int(warp) * 16 + 16; ++r)
          wgsk::bulk_store(slot + r * BN, part + r * C::kPad, BN * 4);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
      __syncwarp();
    }
  }
  if (args.trace && blockIdx.x == 0 && threadIdx.x == 0) args.trace[127] = clock64();
  ptx::cluster_sync();  // release / acquire at cluster scope: every slot is complete
  if (args.trace && blockIdx.x == 0 && threadIdx.x == 0) args.trace[126] = clock64();
  if (S > 1) {
    if (threadIdx.x == 0) {
      wgsk::fence_proxy_async_global();
      const uint32_t bytes = uint32_t((r1 - r0) * BN * 4);
      ptx::mbar_arrive_expect_tx(gbar, bytes * uint32_t(S));
      for (int p = 0; p < S; ++p)
        wgsk::bulk_load(gbuf + size_t(p) * (r1 - r0) * BN, slots + size_t(p) * kSlotFloats + size_t(r0) * BN, bytes, gbar);
    }
    ptx::mbar_wait(gbar, 0);
  }
  {
    const int Mg = args.Mg[lev];
    auto src = [&](int p, int r, int c) -> float4 {
      if (S == 1) return *reinterpret_cast<const float4*>(part + r * C::kPad + c);
      return *reinterpret_cast<const float4*>(gbuf + (size_t(p) * (r1 - r0) + (r - r0)) * BN + c);
    };
    const int items = (r1 - r0) * (BN / 4);
    const bool vec = (N % 4) == 0 && ((reinterpret_cast<uintptr_t>(ga.g[lev]) | reinterpret_cast<uintptr_t>(ga.w[lev]) |
                                       reinterpret_cast<uintptr_t>(ga.mom[lev])) & 15) == 0 &&
                     ((reinterpret_cast<uintptr_t>(ga.shadow[lev]) | reinterpret_cast<uintptr_t>(ga.shadow_lo[lev])) & 7) == 0;
    constexpr int U = 3;  // items in flight per thread: their S partial loads (and w, v) issued together
    for (int base = int(threadIdx.x); base < items; base += C::kThreads * U) {
      float4 pv[U][8], w0[U], v0[U];
      int rr[U], cc[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * C::kThreads;
        rr[u] = r0 + idx / (BN / 4);
        cc[u] = (idx % (BN / 4)) * 4;
        ok[u] = idx < items && m0 + rr[u] < Mg && n0 + cc[u] < N;
#pragma unroll
        for (int p = 0; p < 8; ++p)
          if (ok[u] && p < S) pv[u][p] = src(p, rr[u], cc[u]);
        if (UPDATE && vec && ok[u] && n0 + cc[u] + 4 <= N) {
          const long long e = (long long)(m0 + rr[u]) * N + n0 + cc[u];
          w0[u] = *reinterpret_cast<const float4*>(ga.w[lev] + e);
          v0[u] = *reinterpret_cast<const float4*>(ga.mom[lev] + e);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
        float4 sum = pv[u][0];
#pragma unroll
        for (int p = 1; p < 8; ++p)
          if (p < S) {
            sum.x += pv[u][p].x;
            sum.y += pv[u][p].y;
            sum.z += pv[u][p].z;
            sum.w += pv[u][p].w;
          }
        const int n = n0 + cc[u];
        const long long e = (long long)(m0 + rr[u]) * N + n;
        if (vec && n + 4 <= N) {
          wgsk::store4<UPDATE>(ga, lev, e, sum, w0[u], v0[u]);
        } else {
          const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
          for (int j = 0; j < 4 && n + j < N; ++j) wgsk::store1<UPDATE>(ga, lev, e + j, sv[j]);
        }
      }
    }
    if (bias_here) {
      const int c0 = split * bias_w / S, c1 = (split + 1) * bias_w / S;
      for (int c = c0 + int(threadIdx.x); c < c1; c += C::kThreads) {
        const int n = n0 + bias_c0 + c;
        if (n >= N) continue;
        float sum = 0.f;
        for (int p = 0; p < S; ++p) sum += S == 1 ? btot[c] : __ldcg(slots + size_t(p) * kSlotFloats + BM * BN + c);
        wgsk::store1<UPDATE>(ga, lev, (long long)args.bias_row[lev] * N + n, sum);
      }
    }
  }
  if (args.trace && blockIdx.x == 0 && threadIdx.x == 0) args.trace[129] = clock64();
  if (args.trace && threadIdx.x == 0 && blockIdx.x < 148) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    args.trace[132 + 2 * blockIdx.x] = t;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace moses
