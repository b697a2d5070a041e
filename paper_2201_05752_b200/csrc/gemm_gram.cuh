// gemm_gram.cuh — Gaussian-kernel Gram reduction on the tensor cores (north-star (4): the MMD
// domain-discrepancy loss as a tiled kernel-matrix reduction).
//
//   S(X, Y) = sum_{i,j} exp(-|x_i - y_j|^2 / (2 sigma^2)),   |x - y|^2 = |x|^2 + |y|^2 - 2 x.y
//
// The x.y tile is a tcgen05 kind::tf32 GEMM (128 x 128 tiles, TMA-staged K-major operands, two TMEM
// accumulators so the exp epilogue of one tile overlaps the MMAs of the next); the epilogue turns
// each accumulator row into sum_j exp2(-c * max(nx_i + ny_j - 2 dot, 0)) and every warp writes one
// fixed-order partial, so the reduction is deterministic (no float atomics). Operands are rounded
// to tf32 (RNA) once and the squared norms are computed from the rounded values, so the distance
// of a point to itself cancels to fp32 rounding. Symmetric Grams (X = Y) visit only the upper
// triangle of tiles and count off-diagonal tiles twice.
#pragma once
#include "gemm.cuh"

namespace moses {

struct GramArgs {
  int M, N, K;
  const float* nx;  // [M] squared norms of the (tf32-rounded) rows of X
  const float* ny;  // [N]
  float c;          // log2(e) / (2 sigma^2)
  int sym;          // X == Y: upper-triangle tiles only
  double* part;     // [tiles * 4] per-warp partial sums
};

struct GCfg {
  static constexpr int BM = 128, BN = 128, BK = 32;  // tf32: 32 fp32 per 128-byte swizzle row
  static constexpr int kABytes = BM * 128, kBBytes = BN * 128, kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = 6;
  static constexpr int kThreads = 192;
  static constexpr uint32_t kTmemCols = 2 * BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
};

// tile u -> (mi, ni): full grid M-fastest, or the upper triangle (mi <= ni) column by column
__device__ __forceinline__ void gram_tile(long long u, int tiles_m, bool sym, int& mi, int& ni) {
  if (!sym) {
    mi = int(u % tiles_m);
    ni = int(u / tiles_m);
    return;
  }
  long long c = (long long)((sqrt(8.0 * double(u) + 1.0) - 1.0) * 0.5);
  while (c * (c + 1) / 2 > u) --c;
  while ((c + 1) * (c + 2) / 2 <= u) ++c;
  ni = int(c);
  mi = int(u - c * (c + 1) / 2);
}

__global__ void __launch_bounds__(GCfg::kThreads, 1)
    umma_gram_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GramArgs args, int tiles_m, long long tiles) {
  using Cfg = GCfg;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::kStages, UK = 8;
  constexpr uint32_t kIdesc = ptx::umma_idesc(2 /*tf32*/, false, false, BM, BN);
  const bool sym = args.sym != 0;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull = empty_bar + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int num_kb = (args.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (long long u = blockIdx.x; u < tiles; u += gridDim.x) {
        int mi, ni;
        gram_tile(u, tiles_m, sym, mi, ni);
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStageBytes;
          ptx::mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          ptx::tma_load_2d(sa, &tmA, &full_bar[stage], kb * BK, mi * BM);
          ptx::tma_load_2d(sa + Cfg::kABytes, &tmB, &full_bar[stage], kb * BK, ni * BN);
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
      for (long long u = blockIdx.x; u < tiles; u += gridDim.x, ++i) {
        const int acc = i & 1;
        const uint32_t use = uint32_t(i >> 1);
        ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk)
            ptx::umma_tf32(d, ptx::sw128_desc(sa + kk * UK * 4, 16, 1024), ptx::sw128_desc(sb + kk * UK * 4, 16, 1024),
                           kIdesc, (kb > 0 || kk > 0) ? 1u : 0u);
          ptx::umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    const int quarter = int(warp & 3);
    const int row = quarter * 32 + int(lane);
    int i = 0;
    for (long long u = blockIdx.x; u < tiles; u += gridDim.x, ++i) {
      const int acc = i & 1;
      const uint32_t use = uint32_t(i >> 1);
      int mi, ni;
      gram_tile(u, tiles_m, sym, mi, ni);
      const int m = mi * BM + row;
      const bool row_ok = m < args.M;
      const float nxm = row_ok ? __ldg(args.nx + m) : 0.f;
      ptx::mbar_wait(&tfull[acc], use & 1);
      ptx::tc_fence_after();
      const uint32_t t_acc = tmem_base + uint32_t(acc * BN) + (uint32_t(quarter * 32) << 16);
      float s = 0.f;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(t_acc + c * 32, r);
        ptx::tmem_ld_wait();
        if (c + 1 == BN / 32) {  // accumulator drained: hand it back to the MMA warp
          ptx::tc_fence_before();
          ptx::mbar_arrive(&tempty[acc]);
        }
        const int nb = ni * BN + c * 32;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = nb + j;
          const float nyn = n < args.N ? __ldg(args.ny + n) : 0.f;
          const float d2 = fmaxf(fmaf(-2.f, __uint_as_float(r[j]), nxm + nyn), 0.f);
          const float k = exp2f(-d2 * args.c);
          s += (row_ok && n < args.N) ? k : 0.f;
        }
      }
      double ds = double(s);
#pragma unroll
      for (int o = 16; o; o >>= 1) ds += __shfl_xor_sync(0xffffffffu, ds, o);
      if (lane == 0) args.part[u * 4 + quarter] = (sym && ni != mi) ? 2.0 * ds : ds;
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
