// gemm_fwd.cuh — persistent forward-layer GEMM for candidate-pool scoring (bf16, Epi::Fwd).
//
// Same warp-specialised mainloop as gemm_persistent.cuh (TMA producer warp, single-thread
// tcgen05.mma issuer, two TMEM accumulators so the epilogue of tile i overlaps the MMAs of tile
// i+1), with the epilogue rebuilt for the scoring shape (K = 512: the 128 x 256 accumulator drain
// is half of the mainloop time, so a slow drain paces the tensor core):
//   * 8 epilogue warps (two per TMEM lane quarter, each owning half of the tile's columns);
//   * bias + ReLU + head dot products in registers, the bf16 activation tile written to a per-warp
//     128-byte-swizzled staging box (conflict-free 16-B st.shared) and stored with one TMA tensor
//     store per 32 x 64 box (coalesced full-line writes instead of one row per thread);
//   * head partials per 128-column half-tile: head_part[(2 * n_tile + half) * head_ld + m]
//     (fixed-order sums downstream; the caller sees head tiles of BN / 2 columns).
#pragma once
#include "gemm_persistent.cuh"

namespace moses {

namespace fwd_detail {
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
}  // namespace fwd_detail

// One epilogue warp's share of a tile: rows quarter*32 + lane of [m0, m0+128), kHalf accumulator
// columns starting at output column nb0 (TMEM address t_acc). bias + ReLU + head dots in registers,
// the bf16 activations through a 32 x 64 SW128 staging box and one TMA store per box; head partials
// go to head_part[head_tile * head_ld + m]. `release` runs once the accumulator is in registers.
// SPLIT (split bf16, gemm_fwd2.cuh umma_fwd_pair_split): the activations leave as a hi / lo pair
// (hi = rn(v), lo = rn(v - hi)) through the one staging box: hi stored, box drained, lo stored (tmC_lo).
// (Measured: per-thread direct row stores instead made the layer 1.4x slower than its mainloop.)
template <int kHalf, bool SPLIT = false, typename Release>
__device__ __forceinline__ void fwd_epi_tile(const GemmArgs& args, const CUtensorMap* tmC, uint8_t* stg, uint32_t t_acc,
                                             int m0, int quarter, int nb0, int head_tile, Release&& release,
                                             const CUtensorMap* tmC_lo = nullptr) {
  using namespace fwd_detail;
  const int lane = int(threadIdx.x & 31);
  const int m = m0 + quarter * 32 + lane;
  const bool store = args.out != nullptr;
  float hp = 0.f, hp2 = 0.f;
#pragma unroll 1
  for (int g = 0; g < kHalf / 64; ++g) {
    uint32_t r0[32], r1[32];
    ptx::tmem_ld_32x32b_x32(t_acc + g * 64, r0);
    ptx::tmem_ld_32x32b_x32(t_acc + g * 64 + 32, r1);
    ptx::tmem_ld_wait();
    if (g + 1 == kHalf / 64) release();  // accumulator fully drained into registers
    const int nb = nb0 + g * 64;
    if (nb >= args.N) continue;
    const bool full = nb + 64 <= args.N;
    float v[64];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      v[j] = __uint_as_float(r0[j]);
      v[32 + j] = __uint_as_float(r1[j]);
    }
    if (full) {
      const float4* b4 = reinterpret_cast<const float4*>(args.bias + nb);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float4 bb = __ldg(b4 + q);
        v[4 * q] += bb.x; v[4 * q + 1] += bb.y; v[4 * q + 2] += bb.z; v[4 * q + 3] += bb.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = (nb + j < args.N) ? v[j] + __ldg(args.bias + nb + j) : 0.f;
    }
    if (args.relu) {
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = fmaxf(v[j], 0.f);
    }
    if (args.head_w != nullptr) {
#pragma unroll
      for (int j = 0; j < 64; ++j) hp = fmaf(v[j], (full || nb + j < args.N) ? __ldg(args.head_w + nb + j) : 0.f, hp);
    }
    if (args.head_u != nullptr) {
#pragma unroll
      for (int j = 0; j < 64; ++j) hp2 = fmaf(v[j], (full || nb + j < args.N) ? __ldg(args.head_u + nb + j) : 0.f, hp2);
    }
    if (store && SPLIT) {
#pragma unroll
      for (int plane = 0; plane < 2; ++plane) {  // hi box, then (box drained) lo box
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
        uint8_t* srow = stg + lane * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 pk;
          __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x0 = v[8 * c + 2 * e], x1 = v[8 * c + 2 * e + 1];
            const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
            p2[e] = plane == 0 ? h : __floats2bfloat162_rn(x0 - __low2float(h), x1 - __high2float(h));
          }
          *reinterpret_cast<uint4*>(srow + ((c ^ (lane & 7)) << 4)) = pk;  // SW128: chunk ^ (row % 8)
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(plane == 0 ? tmC : tmC_lo, stg, nb, m0 + quarter * 32);  // rows >= M / cols >= N clipped
          bulk_commit();
        }
      }
    } else if (store) {
      if (lane == 0) bulk_wait_read0();  // previous box has left the staging buffer
      __syncwarp();
      uint8_t* srow = stg + lane * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 pk;
        __nv_bfloat162 p0 = __floats2bfloat162_rn(v[8 * c], v[8 * c + 1]);
        __nv_bfloat162 p1 = __floats2bfloat162_rn(v[8 * c + 2], v[8 * c + 3]);
        __nv_bfloat162 p2 = __floats2bfloat162_rn(v[8 * c + 4], v[8 * c + 5]);
        __nv_bfloat162 p3 = __floats2bfloat162_rn(v[8 * c + 6], v[8 * c + 7]);
        pk.x = *reinterpret_cast<uint32_t*>(&p0);
        pk.y = *reinterpret_cast<uint32_t*>(&p1);
        pk.z = *reinterpret_cast<uint32_t*>(&p2);
        pk.w = *reinterpret_cast<uint32_t*>(&p3);
        *reinterpret_cast<uint4*>(srow + ((c ^ (lane & 7)) << 4)) = pk;  // SW128: chunk ^ (row % 8)
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmC, stg, nb, m0 + quarter * 32);  // rows >= M / cols >= N are clipped
        bulk_commit();
      }
    }
  }
  if (m < args.M) {
    const long long slot = (long long)head_tile * args.head_ld + m;
    if (args.head_part != nullptr) args.head_part[slot] = hp;
    if (args.head_part2 != nullptr) args.head_part2[slot] = hp2;
  }
}

template <int BN>
struct FCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;  // bf16: one 128-byte swizzle row of K
  static constexpr int kABytes = BM * 128;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kEpiWarps = 8;
  static constexpr int kStgBytes = 32 * 128;  // per-warp staging box: 32 rows x 64 bf16
  static constexpr int kFixed = 1024 /*align*/ + 256 /*barriers*/ + kEpiWarps * kStgBytes;
  static constexpr int kStagesFit = (227 * 1024 - kFixed) / kStageBytes;
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  static constexpr int kThreads = 64 + 32 * kEpiWarps;
  static constexpr uint32_t kTmemCols = 2 * BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + kFixed;
  static_assert(kStages >= 3, "pipeline too shallow");
};

template <int BN, bool B_MN>
__global__ void __launch_bounds__(FCfg<BN>::kThreads, 1)
    umma_fwd_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC, const GemmArgs args, int tiles_m, int tiles_n) {
  using Cfg = FCfg<BN>;
  using namespace fwd_detail;
  constexpr int BM = Cfg::BM, BK = Cfg::BK, STAGES = Cfg::kStages, UK = 16;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*bf16*/, false, B_MN, BM, BN);
  constexpr int kHalf = BN / 2;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + STAGES * Cfg::kStageBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + Cfg::kEpiWarps * Cfg::kStgBytes);
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
    ptx::tma_prefetch_desc(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 32 * Cfg::kEpiWarps);
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
          ptx::tma_load_2d(sa, &tmA, &full_bar[stage], k0, m0);
          if constexpr (B_MN) {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) ptx::tma_load_2d(sb + c * (BK * 128), &tmB, &full_bar[stage], n0 + c * 64, k0);
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
        ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = ptx::sw128_desc(sa + kk * UK * 2, 16, 1024);
            const uint64_t bd = B_MN ? ptx::sw128_desc(sb + kk * args.mn_kstep, BK * 128, args.mn_sbo, args.mn_layout)
                                     : ptx::sw128_desc(sb + kk * UK * 2, 16, 1024);
            ptx::umma_f16(d, ad, bd, kIdesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // epilogue warps 2..9: TMEM lane quarter = warp % 4, column half = (warp - 2) / 4
    const int ew = int(warp) - 2;
    const int quarter = int(warp & 3);
    const int half = ew >> 2;
    uint8_t* stg = staging + ew * Cfg::kStgBytes;
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int acc = i & 1;
      const uint32_t use = uint32_t(i >> 1);
      const int m0 = (t % tiles_m) * BM, n_tile = t / tiles_m;
      ptx::mbar_wait(&tfull[acc], use & 1);
      ptx::tc_fence_after();
      const uint32_t t_acc = tmem_base + uint32_t(acc * BN + half * kHalf) + (uint32_t(quarter * 32) << 16);
      fwd_epi_tile<kHalf>(args, &tmC, stg, t_acc, m0, quarter, n_tile * BN + half * kHalf, 2 * n_tile + half, [&] {
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
      });
    }
    if (lane == 0) bulk_wait0();
    __syncwarp();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

}  // namespace moses
