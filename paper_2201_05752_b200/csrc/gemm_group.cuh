// gemm_group.cuh — every level's weight-gradient GEMM of a training step in ONE launch (bf16).
//
//   G_l [(dims_l + 1) x dims_{l+1}] = [act_l | 1]^T dZ_{l+1}     (K = rows of the batch)
//
// One CTA per 128 x 64 output tile of one level (tile table in GroupArgs); both operands are
// MN-major views of the row-major activation / dZ buffers, exactly as the per-level launches
// (umma_gemm_kernel<bf16, 64, MN, MN, StoreF32>) — same tiles, same K order, same values.
// At batch 512 programs the per-level launches ran back to back on the side stream (~14 us each,
// mostly fixed cost); one launch of all ~136 tiles fills the GPU once.
//
// UPDATE: the epilogue also applies the momentum-SGD step to the parameters it just produced
// (tuner.cpp:146-147 / sgd_kernel arithmetic, element for element: v = mu*v + g; w -= lr*v, no
// FMA contraction) and refreshes the bf16 operand shadow — the separate update pass over P
// parameters disappears from the step.
#pragma once
#include "gemm.cuh"

namespace moses {

constexpr int kGroupMax = 8;

struct GroupMaps {
  CUtensorMap a[kGroupMax];  // act_l  [K rows][ld] (MN-major view, M = dims_l + 1 incl. the ones column)
  CUtensorMap b[kGroupMax];  // dZ_l+1 [K rows][ld] (MN-major view)
};
// SPLIT (MOSES_PREC_BF16X3): the lo planes of both operands; G = A_hi B_hi + A_hi B_lo + A_lo B_hi
struct GroupMapsSplit : GroupMaps {
  CUtensorMap a_lo[kGroupMax];
  CUtensorMap b_lo[kGroupMax];
};

struct GroupArgs {
  int n;                       // levels
  int K;                       // batch rows
  int tile_begin[kGroupMax + 1];
  int tiles_n[kGroupMax];
  int M[kGroupMax], N[kGroupMax];
  float* g[kGroupMax];         // gradient block of the level (row-major [M][N])
  float* w[kGroupMax];         // UPDATE: parameters / momentum / bf16 shadow of the same block
  float* mom[kGroupMax];
  __nv_bfloat16* shadow[kGroupMax];
  __nv_bfloat16* shadow_lo[kGroupMax];  // SPLIT: lo half of the operand shadow (hi + lo = w to 2^-18)
  float lr, mu;
  long long* counter;      // optional: step counter advanced once (training graphs' batch index)
  const double* loss_src;  // optional: *loss_acc += *loss_src once (epoch loss sum)
  double* loss_acc;
  double* loss_copy;       // optional: *loss_copy = *loss_src once (per-step loss mailbox)
};

// BK = 128 K rows per stage: MN-major boxes of {64, 128} = 16 KB. The per-SM TMA ingest rate grows
// with the box size (tools/tma_bench.cu, profiles/r2/tma_ingest_bench.json: 8 KB boxes ~22-29 B/clk,
// 16 KB ~33-52, 32 KB ~66-88), while the ring depth does not matter.
struct GroupCfg {
  static constexpr int BM = 128, BN = 64, BK = 128;
  static constexpr int kABytes = BM * BK * 2, kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = 4;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
};
// split bf16 (MOSES_PREC_BF16X3): [A_hi | B_hi | A_lo | B_lo] per stage; TMEM accumulators promoted
// into fp32 registers every kPromoteKb k-blocks
struct GroupSplitCfg {
  static constexpr int BM = 128, BN = 64, BK = 128;
  static constexpr int kABytes = BM * BK * 2, kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = 2 * (kABytes + kBBytes);
  static constexpr int kStages = 2;
  static constexpr int kPromoteKb = 1;            // 128 K elements (384 products) per TMEM chunk
  static constexpr uint32_t kTmemCols = 2 * BN;   // double-buffered accumulator
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
};

// Tile (BM x BN fp32 in shared memory, row stride BN + 1) -> g [-> momentum step of w / v and the
// bf16 operand shadow (SPLIT: its hi/lo pair)], coalesced row-major passes by every thread of the CTA.
template <bool UPDATE, bool SPLIT, int BM, int BN>
__device__ __forceinline__ void group_update_epilogue(const float* tile, const GroupArgs& args, int lev, int m0, int n0,
                                                      int M, int N) {
  constexpr int kPad = BN + 1;
  const int rows = min(BM, M - m0), cols = min(BN, N - n0);
  float* __restrict__ g = args.g[lev];
  float* __restrict__ w = args.w[lev];
  float* __restrict__ v = args.mom[lev];
  __nv_bfloat16* __restrict__ sh = args.shadow[lev];
  __nv_bfloat16* __restrict__ shl = args.shadow_lo[lev];
  auto upd = [&](float gv, float vi0, float wi0, float& vi, float& wi) {
    vi = __fadd_rn(__fmul_rn(args.mu, vi0), gv);
    wi = __fsub_rn(wi0, __fmul_rn(args.lr, vi));
  };
  const bool vec = cols == BN && (N % 4) == 0 && ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(w) |
                                                   reinterpret_cast<uintptr_t>(v)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(sh) & 7) == 0;
  if (vec) {
    // float4 per thread, 4 independent float4 in flight (the update is HBM-latency bound when the
    // parameters are not L2-resident)
    constexpr int kV = BM * BN / 4, kU = 4;
    for (int base = threadIdx.x; base < kV; base += blockDim.x * kU) {
      float4 gv[kU], vv[kU], wv[kU];
      long long e[kU];
      bool ok[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int idx = base + u * blockDim.x;
        const int r = (idx * 4) / BN, c = (idx * 4) - r * BN;
        ok[u] = idx < kV && r < rows;
        e[u] = (long long)(m0 + r) * N + n0 + c;
        const float* t = tile + r * kPad + c;
        gv[u] = make_float4(t[0], t[1], t[2], t[3]);
        if (UPDATE && ok[u]) {
          vv[u] = *reinterpret_cast<const float4*>(v + e[u]);
          wv[u] = *reinterpret_cast<const float4*>(w + e[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (!ok[u]) continue;
        *reinterpret_cast<float4*>(g + e[u]) = gv[u];
        if constexpr (UPDATE) {
          float4 vo, wo;
          upd(gv[u].x, vv[u].x, wv[u].x, vo.x, wo.x);
          upd(gv[u].y, vv[u].y, wv[u].y, vo.y, wo.y);
          upd(gv[u].z, vv[u].z, wv[u].z, vo.z, wo.z);
          upd(gv[u].w, vv[u].w, wv[u].w, vo.w, wo.w);
          *reinterpret_cast<float4*>(v + e[u]) = vo;
          *reinterpret_cast<float4*>(w + e[u]) = wo;
          __nv_bfloat162 p0 = __floats2bfloat162_rn(wo.x, wo.y), p1 = __floats2bfloat162_rn(wo.z, wo.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&p0);
          pk.y = *reinterpret_cast<uint32_t*>(&p1);
          *reinterpret_cast<uint2*>(sh + e[u]) = pk;
          if constexpr (SPLIT) {
            __nv_bfloat162 l0 = __floats2bfloat162_rn(wo.x - __low2float(p0), wo.y - __high2float(p0));
            __nv_bfloat162 l1 = __floats2bfloat162_rn(wo.z - __low2float(p1), wo.w - __high2float(p1));
            uint2 pl;
            pl.x = *reinterpret_cast<uint32_t*>(&l0);
            pl.y = *reinterpret_cast<uint32_t*>(&l1);
            *reinterpret_cast<uint2*>(shl + e[u]) = pl;
          }
        }
      }
    }
  } else {
    for (int idx = threadIdx.x; idx < BM * BN; idx += blockDim.x) {
      const int r = idx / BN, c = idx - r * BN;
      if (r >= rows || c >= cols) continue;
      const long long e = (long long)(m0 + r) * N + n0 + c;
      const float gv = tile[r * kPad + c];
      g[e] = gv;
      if constexpr (UPDATE) {
        float vi, wi;
        upd(gv, v[e], w[e], vi, wi);
        v[e] = vi;
        w[e] = wi;
        sh[e] = __float2bfloat16_rn(wi);
        if constexpr (SPLIT) shl[e] = __float2bfloat16_rn(wi - __bfloat162float(sh[e]));
      }
    }
  }

}

template <bool UPDATE>
__global__ void __launch_bounds__(128, 1)
    wgrad_group_kernel(const __grid_constant__ GroupMaps maps, const __grid_constant__ GroupArgs args) {
  using C = GroupCfg;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, STAGES = C::kStages;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*BF16*/, true, true, BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* accum_bar = empty_bar + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_bar + 1);

  // tile -> (level, m tile, n tile)
  const int t = blockIdx.x;
  int lev = 0;
  while (lev + 1 < args.n && t >= args.tile_begin[lev + 1]) ++lev;
  const int local = t - args.tile_begin[lev];
  const int m0 = (local / args.tiles_n[lev]) * BM, n0 = (local % args.tiles_n[lev]) * BN;
  const int M = args.M[lev], N = args.N[lev];
  const CUtensorMap* tmA = &maps.a[lev];
  const CUtensorMap* tmB = &maps.b[lev];

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int num_kb = (args.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(tmA);
    ptx::tma_prefetch_desc(tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    ptx::mbar_init(accum_bar, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<BN>(tmem_slot);
  ptx::pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 32) {  // step bookkeeping folded into the step's last kernel
    if (args.counter != nullptr) *args.counter += 1;
    if (args.loss_acc != nullptr) *args.loss_acc += *args.loss_src;
    if (args.loss_copy != nullptr) *args.loss_copy = *args.loss_src;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * C::kStageBytes;
        uint8_t* sb = sa + C::kABytes;
        ptx::mbar_arrive_expect_tx(&full_bar[stage], C::kStageBytes);
        const int k0 = kb * BK;
        ptx::tma_load_2d(sa, tmA, &full_bar[stage], m0, k0);
        ptx::tma_load_2d(sa + BK * 128, tmA, &full_bar[stage], m0 + 64, k0);
        ptx::tma_load_2d(sb, tmB, &full_bar[stage], n0, k0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        ptx::mbar_wait(&full_bar[stage], phase);
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(smem + stage * C::kStageBytes);
        const uint32_t sb = sa + C::kABytes;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t ad = ptx::sw128_desc(sa + kk * 2048, BK * 128, 1024, 2);
          const uint64_t bd = ptx::sw128_desc(sb + kk * 2048, BK * 128, 1024, 2);
          ptx::umma_f16(tmem_base, ad, bd, kIdesc, (kb > 0 || kk > 0) ? 1u : 0u);
        }
        ptx::umma_commit(&empty_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      ptx::umma_commit(accum_bar);
    }
    __syncwarp();
  }

  // Epilogue: TMEM -> padded smem tile (the pipeline stages are free once the accumulator is
  // complete) -> coalesced row-major passes over g (and w / momentum / shadow when UPDATE).
  constexpr int kPad = BN + 1;
  float* tile = reinterpret_cast<float*>(smem);
  const int row = int(warp) * 32 + int(lane);
  const uint32_t t_row = tmem_base + ((warp * 32u) << 16);
  ptx::mbar_wait(accum_bar, 0);
  ptx::tc_fence_after();
  ptx::pdl_launch_dependents();
#pragma unroll
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) tile[row * kPad + c * 32 + j] = __uint_as_float(r[j]);
  }
  __syncthreads();
  group_update_epilogue<UPDATE, false, C::BM, C::BN>(tile, args, lev, m0, n0, M, N);

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<BN>(tmem_base);
  }
}

// Split-bf16 grouped wgrad: G = A_hi B_hi + A_hi B_lo + A_lo B_hi over K = the batch rows. The sums
// run over ~2.3K-18K rows of mixed-sign dZ, where the tensor-core accumulator (not a round-to-nearest
// fp32 adder) drifts by ~1e-3 of the result; so, as in gemm_split.cuh, the MMAs of every kPromoteKb
// k-blocks go to one of two TMEM buffers and the drain warps add the finished chunk into fp32
// registers while the next chunk accumulates. 192 threads: warps 0-3 drain + epilogue, warp 4 TMA
// producer, warp 5 MMA issuer.
template <bool UPDATE>
__global__ void __launch_bounds__(192, 1)
    wgrad_group_split_kernel(const __grid_constant__ GroupMapsSplit maps, const __grid_constant__ GroupArgs args) {
  using C = GroupSplitCfg;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, STAGES = C::kStages, KC = C::kPromoteKb;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*BF16*/, true, true, BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* bfull = empty_bar + STAGES;  // [2] accumulator buffer holds a finished chunk
  uint64_t* bempty = bfull + 2;          // [2] drain warps have consumed the buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + 2);

  const int t = blockIdx.x;
  int lev = 0;
  while (lev + 1 < args.n && t >= args.tile_begin[lev + 1]) ++lev;
  const int local = t - args.tile_begin[lev];
  const int m0 = (local / args.tiles_n[lev]) * BM, n0 = (local % args.tiles_n[lev]) * BN;
  const int M = args.M[lev], N = args.N[lev];

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int num_kb = (args.K + BK - 1) / BK;
  const int nchunks = (num_kb + KC - 1) / KC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&bfull[b], 1);
      ptx::mbar_init(&bempty[b], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
  ptx::pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 160) {  // step bookkeeping folded into the step's last kernel
    if (args.counter != nullptr) *args.counter += 1;
    if (args.loss_acc != nullptr) *args.loss_acc += *args.loss_src;
    if (args.loss_copy != nullptr) *args.loss_copy = *args.loss_src;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {
      const CUtensorMap* tmA = &maps.a[lev];
      const CUtensorMap* tmB = &maps.b[lev];
      const CUtensorMap* tmAl = &maps.a_lo[lev];
      const CUtensorMap* tmBl = &maps.b_lo[lev];
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * C::kStageBytes;
        uint8_t* sb = sa + C::kABytes;
        uint8_t* sal = sb + C::kBBytes;
        uint8_t* sbl = sal + C::kABytes;
        ptx::mbar_arrive_expect_tx(&full_bar[stage], C::kStageBytes);
        const int k0 = kb * BK;
        ptx::tma_load_2d(sa, tmA, &full_bar[stage], m0, k0);
        ptx::tma_load_2d(sa + BK * 128, tmA, &full_bar[stage], m0 + 64, k0);
        ptx::tma_load_2d(sb, tmB, &full_bar[stage], n0, k0);
        ptx::tma_load_2d(sal, tmAl, &full_bar[stage], m0, k0);
        ptx::tma_load_2d(sal + BK * 128, tmAl, &full_bar[stage], m0 + 64, k0);
        ptx::tma_load_2d(sbl, tmBl, &full_bar[stage], n0, k0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        const int c = kb / KC, buf = c & 1;
        const bool first = (kb % KC) == 0;
        if (first && c >= 2) {
          ptx::mbar_wait(&bempty[buf], uint32_t((c - 2) >> 1) & 1u);  // chunk c-2 drained
          ptx::tc_fence_after();
        }
        ptx::mbar_wait(&full_bar[stage], phase);
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(smem + stage * C::kStageBytes);
        const uint32_t sb = sa + C::kABytes, sal = sb + C::kBBytes, sbl = sal + C::kABytes;
        const uint32_t tacc = tmem_base + uint32_t(buf * BN);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t ah = ptx::sw128_desc(sa + kk * 2048, BK * 128, 1024, 2);
          const uint64_t bh = ptx::sw128_desc(sb + kk * 2048, BK * 128, 1024, 2);
          const uint64_t al = ptx::sw128_desc(sal + kk * 2048, BK * 128, 1024, 2);
          const uint64_t bl = ptx::sw128_desc(sbl + kk * 2048, BK * 128, 1024, 2);
          // small terms first: they never dominate the running sum's exponent
          ptx::umma_f16(tacc, ah, bl, kIdesc, (!first || kk > 0) ? 1u : 0u);
          ptx::umma_f16(tacc, al, bh, kIdesc, 1u);
          ptx::umma_f16(tacc, ah, bh, kIdesc, 1u);
        }
        ptx::umma_commit(&empty_bar[stage]);
        if ((kb % KC) == KC - 1 || kb == num_kb - 1) ptx::umma_commit(&bfull[buf]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    // drain: warp w owns TMEM lanes / tile rows 32w..32w+31; fp32 register accumulation per chunk
    const int row = int(warp) * 32 + int(lane);
    const uint32_t t_row = tmem_base + ((warp * 32u) << 16);
    float acc[BN];
#pragma unroll
    for (int j = 0; j < BN; ++j) acc[j] = 0.f;
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      ptx::mbar_wait(&bfull[buf], uint32_t(c >> 1) & 1u);
      ptx::tc_fence_after();
#pragma unroll
      for (int q = 0; q < BN / 32; ++q) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(t_row + uint32_t(buf * BN + q * 32), r);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[q * 32 + j] += __uint_as_float(r[j]);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bempty[buf]);
    }
    ptx::pdl_launch_dependents();
    // every stage is free once the last chunk is drained: the tile reuses the pipeline memory
    float* tile = reinterpret_cast<float*>(smem);
#pragma unroll
    for (int j = 0; j < BN; ++j) tile[row * (BN + 1) + j] = acc[j];
  }
  __syncthreads();
  group_update_epilogue<UPDATE, true, BM, BN>(reinterpret_cast<const float*>(smem), args, lev, m0, n0, M, N);

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

}  // namespace moses
