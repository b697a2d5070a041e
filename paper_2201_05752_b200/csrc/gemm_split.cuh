// gemm_split.cuh — 3xTF32 GEMM for the fp32 parity mode (MOSES_PREC_FP32).
//
// Every operand arrives as a (hi, lo) pair of tf32-representable fp32 buffers with
// hi = rna_tf32(v), lo = rna_tf32(v - hi); the product is a_hi*b_hi + a_hi*b_lo + a_lo*b_hi
// (the lo*lo term is below fp32 resolution). The tensor-core accumulator is not a round-to-
// nearest fp32 adder, so long K chains drift: the partial sums are PROMOTED into fp32 registers
// every kPromoteKb k-blocks (128 K elements), the DeepSeek-V3 recipe for low-precision
// accumulators. Two TMEM accumulator buffers let the MMA warp run chunk c+1 while the drain
// warps add chunk c into their registers.
//
// 192 threads: warps 0-3 drain + epilogue (warp w owns TMEM lanes / tile rows 32w..32w+31),
// warp 4 = TMA producer, warp 5 = MMA issuer. One CTA per 128 x BN output tile.
#pragma once
#include "gemm.cuh"

namespace moses {

template <int BN>
struct SCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 32;                    // tf32: one 128-byte swizzle row of K
  static constexpr int kABytes = BM * 128;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStageBytes = 2 * (kABytes + kBBytes);  // [A_hi | B_hi | A_lo | B_lo]
  static constexpr int kStages = (200 * 1024 / kStageBytes) > 6 ? 6 : (200 * 1024 / kStageBytes);
  static constexpr int kMNChunk = 32;              // fp32 elements per 128-byte MN row
  static constexpr int kPromoteKb = 4;             // promote every 4 k-blocks = 128 K elements
  static constexpr uint32_t kTmemCols = 2 * BN;    // double-buffered accumulator
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
};

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(192, 1)
    umma_gemm_split(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmAlo, const __grid_constant__ CUtensorMap tmBlo,
                    const GemmArgs args) {
  using Cfg = SCfg<BN>;
  constexpr int BM = Cfg::BM, BK = Cfg::BK, STAGES = Cfg::kStages, KC = Cfg::kPromoteKb;
  constexpr int UK = 8;
  constexpr uint32_t kIdesc = ptx::umma_idesc(2 /*TF32*/, A_MN, B_MN, BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* bfull = empty_bar + STAGES;  // [2] accumulator buffer holds a finished chunk
  uint64_t* bempty = bfull + 2;          // [2] drain warps have consumed the buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + 2);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
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
  if (warp == 0) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::pdl_wait();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 4) {
    // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      auto load = [&](uint8_t* dst, const CUtensorMap* tm, bool mn, int rows, int base, int k0) {
        if (mn) {
          for (int c = 0; c < rows / Cfg::kMNChunk; ++c)
            ptx::tma_load_2d(dst + c * (BK * 128), tm, &full_bar[stage], base + c * Cfg::kMNChunk, k0);
        } else {
          ptx::tma_load_2d(dst, tm, &full_bar[stage], k0, base);
        }
      };
      for (int kb = 0; kb < num_kb; ++kb) {
        ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * Cfg::kStageBytes;
        uint8_t* sb = sa + Cfg::kABytes;
        uint8_t* sal = sb + Cfg::kBBytes;
        uint8_t* sbl = sal + Cfg::kABytes;
        ptx::mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
        const int k0 = kb * BK;
        load(sa, &tmA, A_MN, BM, m0, k0);
        load(sb, &tmB, B_MN, BN, n0, k0);
        load(sal, &tmAlo, A_MN, BM, m0, k0);
        load(sbl, &tmBlo, B_MN, BN, n0, k0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ---------------- MMA issuer (single thread)
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
        const uint32_t sa = ptx::smem_u32(smem + stage * Cfg::kStageBytes);
        const uint32_t sb = sa + Cfg::kABytes, sal = sb + Cfg::kBBytes, sbl = sal + Cfg::kABytes;
        const uint32_t tacc = tmem_base + uint32_t(buf * BN);
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk) {
          auto desc = [&](uint32_t base, bool mn) {
            return mn ? ptx::sw128_desc(base + kk * args.mn_kstep, BK * 128, args.mn_sbo, args.mn_layout)
                      : ptx::sw128_desc(base + kk * UK * 4, 16, 1024);
          };
          const uint64_t ah = desc(sa, A_MN), bh = desc(sb, B_MN), al = desc(sal, A_MN), bl = desc(sbl, B_MN);
          // small terms first: they never dominate the running sum's exponent
          ptx::umma_tf32(tacc, ah, bl, kIdesc, (!first || kk > 0) ? 1u : 0u);
          ptx::umma_tf32(tacc, al, bh, kIdesc, 1u);
          ptx::umma_tf32(tacc, ah, bh, kIdesc, 1u);
        }
        ptx::umma_commit(&empty_bar[stage]);
        if ((kb % KC) == KC - 1 || kb == num_kb - 1) ptx::umma_commit(&bfull[buf]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    // ---------------- drain (fp32 promotion) + epilogue: warps 0-3, one tile row per thread
    const int row = int(warp) * 32 + int(lane);
    const int m = m0 + row;
    const bool row_ok = m < args.M;
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

    float hp = 0.f, hp2 = 0.f;
#pragma unroll
    for (int q = 0; q < BN / 32; ++q) {
      const int nb = n0 + q * 32;
      if (!row_ok || nb >= args.N) continue;
      const int nvalid = min(32, args.N - nb);
      float* v = acc + q * 32;
      if constexpr (EPI == int(Epi::Dgrad)) {
        const float* mrow = reinterpret_cast<const float*>(args.mask) + (long long)m * args.ldm + nb;
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (j < nvalid && __ldg(mrow + j) > 0.f) ? v[j] : 0.f;
      }
      if constexpr (EPI == int(Epi::Fwd)) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float b = (j < nvalid && args.bias) ? __ldg(args.bias + nb + j) : 0.f;
          v[j] += b;
          if (args.relu) v[j] = fmaxf(v[j], 0.f);
          if (args.head_w) hp = fmaf(v[j], j < nvalid ? __ldg(args.head_w + nb + j) : 0.f, hp);
          if (args.head_u) hp2 = fmaf(v[j], j < nvalid ? __ldg(args.head_u + nb + j) : 0.f, hp2);
        }
      }
      if (args.out == nullptr) continue;
      float* orow = reinterpret_cast<float*>(args.out) + (long long)m * args.ldo + nb;
      if (EPI != int(Epi::StoreF32) && args.out_lo != nullptr) {
        float* lrow = reinterpret_cast<float*>(args.out_lo) + (long long)m * args.ldo + nb;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float hi = tf32_round(v[j]);
          if (j < nvalid) {
            orow[j] = hi;
            lrow[j] = tf32_round(v[j] - hi);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nvalid) orow[j] = v[j];
      }
    }
    if constexpr (EPI == int(Epi::Fwd)) {
      // per-N-tile partial head dots, same layout as the other GEMM kernels (fixed-order sums)
      if (row_ok && args.head_part != nullptr) args.head_part[(long long)blockIdx.y * args.head_ld + m] = hp;
      if (row_ok && args.head_part2 != nullptr) args.head_part2[(long long)blockIdx.y * args.head_ld + m] = hp2;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

}  // namespace moses
