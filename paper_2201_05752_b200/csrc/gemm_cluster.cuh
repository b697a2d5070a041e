// gemm_cluster.cuh — weight-resident, activation-multicast tcgen05 GEMM for the MLP's hidden layers.
//
// The cost-model GEMMs are tall and skinny in the weight: X [rows x K] * W^T with W only N x K =
// 512 x <=512 (<= 512 KB bf16). Streaming W per 128-row tile (the generic kernels) makes the weight
// the dominant L2->SM traffic (B re-read by every tile). Here a cluster of 4 CTAs splits N = 512
// into four 128-column slices that stay RESIDENT in shared memory (128 x K bf16 <= 128 KB per CTA),
// and every 128-row activation tile is TMA-multicast to the 4 CTAs (each CTA fetches one 32-row
// quarter for the whole cluster). Per layer the L2->SM traffic drops from
// tiles*(A + B_tile) to A + 4*B_slice*clusters.
//
//   warp 0      producer: resident B slice once, then A quarters multicast per K-block (ring of STAGES)
//   warp 1      MMA issuer: 128x128xK per tile into one of two TMEM accumulators; each smem stage is
//               released to all 4 producers with a multicast tcgen05.commit (empty barrier count 4)
//   warps 2..5  epilogue (gemm_persistent.cuh epilogue_tile), overlapping the next tile's MMAs
//
// Constraints: bf16, N % 512 == 0 handled as N == 4 * 128 (the hidden width), K <= 512.
#pragma once
#include "gemm_persistent.cuh"

namespace moses {

struct CCfg {
  static constexpr int BM = 128, BN = 128, BK = 64;  // bf16: one 128-byte swizzle row of K
  static constexpr int kCluster = 4;
  static constexpr int kMaxK = 512;
  static constexpr int kBSliceBytes = BN * 128;      // one K-block of the resident slice (16 KB)
  static constexpr int kABytes = BM * 128;           // one K-block of the activation tile (16 KB)
  static constexpr int kMaxStages = 12;
  static constexpr int kThreads = 192;
  static constexpr uint32_t kTmemCols = 2 * BN;
  static constexpr int kSmemLimit = 227 * 1024;
  // resident slice (num_kb x 16 KB) + as many 16 KB activation stages as fit (runtime: depends on K)
  static int stages_for(int num_kb) {
    const int s = (kSmemLimit - 1024 - 512 - num_kb * kBSliceBytes) / kABytes;
    return s > kMaxStages ? kMaxStages : s;
  }
  static int smem_bytes(int num_kb) { return num_kb * kBSliceBytes + stages_for(num_kb) * kABytes + 1024 + 512; }
};

template <bool B_MN, int EPI>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(192, 1)
    umma_gemm_cluster(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const GemmArgs args, int tiles_m, int STAGES) {
  using T = __nv_bfloat16;
  constexpr int BM = CCfg::BM, BN = CCfg::BN, BK = CCfg::BK;
  constexpr int UK = UmmaType<T>::kUmmaK;
  constexpr uint32_t kIdesc = ptx::umma_idesc(UmmaType<T>::kFormat, false, B_MN, BM, BN);
  constexpr uint16_t kAll = (1u << CCfg::kCluster) - 1;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int num_kb = (args.K + BK - 1) / BK;
  uint8_t* sB = smem;                                // num_kb x 16 KB resident slice
  uint8_t* sA = smem + num_kb * CCfg::kBSliceBytes;  // STAGES x 16 KB ring
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sA + STAGES * CCfg::kABytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* bfull = empty_bar + STAGES;
  uint64_t* tfull = bfull + 1;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const uint32_t rank = ptx::cluster_ctarank();
  const int cluster = blockIdx.x / CCfg::kCluster, clusters = gridDim.x / CCfg::kCluster;
  const int n0 = int(rank) * BN;
  ptx::pdl_launch_dependents();

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], CCfg::kCluster);  // one release per consumer CTA
    }
    ptx::mbar_init(bfull, 1);
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<CCfg::kTmemCols>(tmem_slot);
  ptx::pdl_wait();
  ptx::tc_fence_before();
  ptx::cluster_sync();  // peers' barriers are initialised before anyone multicasts into them
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // resident weight slice: N rows [n0, n0+128) x all K
      ptx::mbar_arrive_expect_tx(bfull, uint32_t(num_kb * CCfg::kBSliceBytes));
      for (int kb = 0; kb < num_kb; ++kb) {
        uint8_t* dst = sB + kb * CCfg::kBSliceBytes;
        if constexpr (B_MN) {
#pragma unroll
          for (int c = 0; c < BN / 64; ++c) ptx::tma_load_2d(dst + c * (BK * 128), &tmB, bfull, n0 + c * 64, kb * BK);
        } else {
          ptx::tma_load_2d(dst, &tmB, bfull, kb * BK, n0);
        }
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < tiles_m; t += clusters) {
        const int m0 = t * BM;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);  // all 4 CTAs released this stage
          uint8_t* sa = sA + stage * CCfg::kABytes;
          ptx::mbar_arrive_expect_tx(&full_bar[stage], CCfg::kABytes);
          // my 32-row quarter of the 128-row tile, written into every CTA's stage
          ptx::tma_load_2d_mc(sa + rank * (32 * 128), &tmA, &full_bar[stage], kb * BK, m0 + int(rank) * 32, kAll);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      ptx::mbar_wait(bfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int t = cluster; t < tiles_m; t += clusters, ++i) {
        const int acc = i & 1;
        const uint32_t use = uint32_t(i >> 1);
        ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(sA + stage * CCfg::kABytes);
          const uint32_t sb = ptx::smem_u32(sB + kb * CCfg::kBSliceBytes);
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = ptx::sw128_desc(sa + kk * UK * 2, 16, 1024);
            const uint64_t bd = B_MN ? ptx::sw128_desc(sb + kk * UK * 128, BK * 128, 1024)
                                     : ptx::sw128_desc(sb + kk * UK * 2, 16, 1024);
            ptx::umma_f16(d, ad, bd, kIdesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::umma_commit_mc(&empty_bar[stage], kAll);  // release this stage in all 4 CTAs
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
    for (int t = cluster; t < tiles_m; t += clusters, ++i) {
      const int acc = i & 1;
      const uint32_t use = uint32_t(i >> 1);
      ptx::mbar_wait(&tfull[acc], use & 1);
      ptx::tc_fence_after();
      const uint32_t t_acc = tmem_base + uint32_t(acc * BN) + (uint32_t(quarter * 32) << 16);
      epilogue_tile<T, BN, false, B_MN, EPI>(args, t_acc, t * BM, n0, int(rank), row);
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // no CTA leaves while peers may still multicast into it or release its stages
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CCfg::kTmemCols>(tmem_base);
  }
}

}  // namespace moses
