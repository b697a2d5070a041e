// gemm_persistent.cuh — persistent, warp-specialised tcgen05 GEMM for large row counts
// (candidate-pool scoring: 64K-row chunks; TenSet-shaped training: ~2.3K statement rows).
//
// One CTA per SM loops over 128 x BN output tiles (static round-robin, M fastest so CTAs running
// together share the B tile in L2). Roles:
//   warp 0      TMA producer  — streams A/B K-blocks through a STAGES-deep smem ring, across tiles
//   warp 1      MMA issuer    — one thread issues tcgen05.mma into one of TWO TMEM accumulators
//   warps 2..5  epilogue      — drain the other accumulator (tcgen05.ld) while the next tile's MMAs run
// Two accumulators of BN fp32 columns (2*BN <= 512 TMEM columns) double-buffer the MMA/epilogue
// hand-off (tmem_full / tmem_empty mbarriers), so the epilogue and the next tile's prologue are
// hidden behind tensor-core work. Epilogues are the ones of gemm.cuh (Fwd / Dgrad / StoreF32).
#pragma once
#include "gemm.cuh"

namespace moses {

template <typename T, int BN>
struct PCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 128 / int(sizeof(T));
  static constexpr int kABytes = BM * 128;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (200 * 1024 / kStageBytes) > 8 ? 8 : (200 * 1024 / kStageBytes);
  static constexpr int kMNChunk = 128 / int(sizeof(T));
  static constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int kThreads = 192;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 512;
};

template <typename T, int BN, bool A_MN, bool B_MN, int EPI>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& args, uint32_t t_acc, int m0, int n0, int n_tile,
                                              int row) {
  const int m = m0 + row;
  const bool row_ok = m < args.M;
  float hp = 0.f, hp2 = 0.f;
  constexpr int kMaskVec = 32 * int(sizeof(T)) / 16;
  uint4 mk[kMaskVec];
  auto load_mask = [&](int c) {
    if constexpr (EPI == int(Epi::Dgrad)) {
      const int nb = n0 + c * 32;
      if (row_ok && nb + 32 <= args.N) {
        const uint4* src =
            reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(args.mask) + (long long)m * args.ldm + nb);
#pragma unroll
        for (int q = 0; q < kMaskVec; ++q) mk[q] = __ldg(src + q);
      } else {
#pragma unroll
        for (int q = 0; q < kMaskVec; ++q) mk[q] = make_uint4(0, 0, 0, 0);
        if (row_ok && nb < args.N) {
          const T* mrow = reinterpret_cast<const T*>(args.mask) + (long long)m * args.ldm + nb;
          T* dst = reinterpret_cast<T*>(mk);
          const int cnt = args.N - nb;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < cnt) dst[j] = mrow[j];
        }
      }
    }
  };
  load_mask(0);
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(t_acc + c * 32, r);
    ptx::tmem_ld_wait();
    const int nb = n0 + c * 32;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
    if constexpr (EPI == int(Epi::Dgrad)) {
      const T* mv = reinterpret_cast<const T*>(mk);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = static_cast<float>(mv[j]) > 0.f ? v[j] : 0.f;
      if (c + 1 < BN / 32) load_mask(c + 1);
    }
    if (!row_ok || nb >= args.N) continue;
    const int nvalid = min(32, args.N - nb);
    if constexpr (EPI == int(Epi::Fwd)) {
      if (nvalid == 32) {
        const float4* b4 = reinterpret_cast<const float4*>(args.bias + nb);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 bb = __ldg(b4 + q);
          v[4 * q] += bb.x; v[4 * q + 1] += bb.y; v[4 * q + 2] += bb.z; v[4 * q + 3] += bb.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += (j < nvalid) ? __ldg(args.bias + nb + j) : 0.f;
      }
      if (args.relu) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
      }
      if (args.head_w != nullptr) {
#pragma unroll
        for (int j = 0; j < 32; ++j) hp = fmaf(v[j], (j < nvalid) ? __ldg(args.head_w + nb + j) : 0.f, hp);
      }
      if (args.head_u != nullptr) {
#pragma unroll
        for (int j = 0; j < 32; ++j) hp2 = fmaf(v[j], (j < nvalid) ? __ldg(args.head_u + nb + j) : 0.f, hp2);
      }
    }
    if constexpr (EPI == int(Epi::StoreF32)) {
      float* orow = reinterpret_cast<float*>(args.out) + (long long)m * args.ldo + nb;
      if (nvalid == 32 && (args.ldo % 4) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(orow + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nvalid) orow[j] = v[j];
      }
    } else {
      if (args.out == nullptr) continue;
      T* orow = reinterpret_cast<T*>(args.out) + (long long)m * args.ldo + nb;
      if constexpr (sizeof(T) == 2) {
        if (nvalid == 32) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 pk;
            __nv_bfloat162 p0 = __floats2bfloat162_rn(v[j], v[j + 1]);
            __nv_bfloat162 p1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
            __nv_bfloat162 p2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]);
            __nv_bfloat162 p3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
            pk.x = *reinterpret_cast<uint32_t*>(&p0);
            pk.y = *reinterpret_cast<uint32_t*>(&p1);
            pk.z = *reinterpret_cast<uint32_t*>(&p2);
            pk.w = *reinterpret_cast<uint32_t*>(&p3);
            *reinterpret_cast<uint4*>(orow + j) = pk;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nvalid) orow[j] = __float2bfloat16_rn(v[j]);
        }
      } else {
        if (args.round_out) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = tf32_round(v[j]);
        }
        if (nvalid == 32) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(orow + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nvalid) orow[j] = v[j];
        }
      }
    }
  }
  if constexpr (EPI == int(Epi::Fwd)) {
    if (row_ok && args.head_part != nullptr) args.head_part[(long long)n_tile * args.head_ld + m] = hp;
    if (row_ok && args.head_part2 != nullptr) args.head_part2[(long long)n_tile * args.head_ld + m] = hp2;
  }
}

template <typename T, int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(192, 1)
    umma_gemm_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const GemmArgs args, int tiles_m, int tiles_n) {
  using Cfg = PCfg<T, BN>;
  constexpr int BM = Cfg::BM, BK = Cfg::BK, STAGES = Cfg::kStages;
  constexpr int UK = UmmaType<T>::kUmmaK;
  constexpr uint32_t kIdesc = ptx::umma_idesc(UmmaType<T>::kFormat, A_MN, B_MN, BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull = empty_bar + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int num_kb = (args.K + BK - 1) / BK;
  const int tiles = tiles_m * tiles_n;
  ptx::pdl_launch_dependents();

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);  // every epilogue thread releases the accumulator
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::pdl_wait();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m0 = (t % tiles_m) * BM, n0 = (t / tiles_m) * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStageBytes;
          uint8_t* sb = sa + Cfg::kABytes;
          ptx::mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          const int k0 = kb * BK;
          if constexpr (A_MN) {
#pragma unroll
            for (int c = 0; c < BM / Cfg::kMNChunk; ++c)
              ptx::tma_load_2d(sa + c * (BK * 128), &tmA, &full_bar[stage], m0 + c * Cfg::kMNChunk, k0);
          } else {
            ptx::tma_load_2d(sa, &tmA, &full_bar[stage], k0, m0);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int c = 0; c < BN / Cfg::kMNChunk; ++c)
              ptx::tma_load_2d(sb + c * (BK * 128), &tmB, &full_bar[stage], n0 + c * Cfg::kMNChunk, k0);
          } else {
            ptx::tma_load_2d(sb, &tmB, &full_bar[stage], k0, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        const uint32_t use = uint32_t(i >> 1);
        ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);  // epilogue has drained this accumulator
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = A_MN ? ptx::sw128_desc(sa + kk * args.mn_kstep, BK * 128, args.mn_sbo, args.mn_layout)
                                     : ptx::sw128_desc(sa + kk * UK * int(sizeof(T)), 16, 1024);
            const uint64_t bd = B_MN ? ptx::sw128_desc(sb + kk * args.mn_kstep, BK * 128, args.mn_sbo, args.mn_layout)
                                     : ptx::sw128_desc(sb + kk * UK * int(sizeof(T)), 16, 1024);
            const uint32_t accum = (kb > 0 || kk > 0) ? 1u : 0u;
            if constexpr (sizeof(T) == 2) ptx::umma_f16(d, ad, bd, kIdesc, accum);
            else ptx::umma_tf32(d, ad, bd, kIdesc, accum);
          }
          ptx::umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // epilogue warps 2..5: TMEM lane quarter = warp % 4
    const int quarter = int(warp & 3);
    const int row = quarter * 32 + int(lane);
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int acc = i & 1;
      const uint32_t use = uint32_t(i >> 1);
      ptx::mbar_wait(&tfull[acc], use & 1);
      ptx::tc_fence_after();
      const int n_tile = t / tiles_m;
      const uint32_t t_acc = tmem_base + uint32_t(acc * BN) + (uint32_t(quarter * 32) << 16);
      epilogue_tile<T, BN, A_MN, B_MN, EPI>(args, t_acc, (t % tiles_m) * BM, n_tile * BN, n_tile, row);
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

}  // namespace moses
