// gemm_fwd2.cuh — weight-resident CTA-pair forward layer for candidate-pool scoring (bf16, N = 512).
//
// Why: the one-CTA scoring layer (gemm_fwd.cuh) streams a 128 x 64 A block (16 KB) and a 256 x 64
// weight block (32 KB) per 512 MMA cycles; TMA delivers ~45 B/clk into one SM (tools/mma_bench.cu),
// so the tensor pipe idles half the time. Here a 2-CTA cluster runs tcgen05.mma.cta_group::2
// (M = 256: 128 rows per CTA, N = 256: 128 weight columns per CTA) and each CTA keeps its 128-column
// weight slice for ALL of K resident in shared memory (128 KB at K = 512), loaded once per launch.
// Only activations stream: 16 KB per CTA per 512 MMA cycles (~32 B/clk), under the TMA rate.
//
//   pair p: n-half (p % 2) of the 512 output columns; m tiles of 256 rows, p/2, p/2 + pairs/2, ...
//   CTA r of the pair: rows [256 i + 128 r, +128), weight columns [256 h + 128 r, +128)
//   leader (r = 0): issues the MMAs (one thread); both CTAs' TMA loads complete on the leader's
//   barriers (.cta_group::2 bulk tensor copies); MMA commits multicast to both CTAs' barriers;
//   each CTA drains its own TMEM (its 128 rows x 256 columns) with the gemm_fwd.cuh epilogue.
#pragma once
#include "gemm_fwd.cuh"

namespace moses {

namespace pair_detail {
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// TMA load into this CTA's shared memory, completing bytes on the barrier at cluster address `bar`
__device__ __forceinline__ void tma_load_2sm(void* smem_dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          ptx::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
// relaxed: these arrivals only count (data arrives through complete_tx, TMEM reads are ordered by
// tcgen05 fences); the default .release emits a GPU-scope MEMBAR per arrival (measured: it paced
// the producer at one stage per MEMBAR round trip)
__device__ __forceinline__ void arrive_remote(uint32_t bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void expect_tx_remote(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {  // arrive on `bar` in both CTAs of the pair
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          ptx::smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_result) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(smem_result)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
}  // namespace pair_detail

struct PairCfg {
  static constexpr int BM = 128;       // rows per CTA (pair tile: 256)
  static constexpr int BNC = 128;      // weight columns per CTA (pair N: 256)
  static constexpr int BK = 64;
  static constexpr int kMaxK = 512;
  static constexpr int kWBytes = kMaxK / BK * BNC * 128;  // resident weight slice: 128 KB
  static constexpr int kABytes = BM * 128;                // one 128 x 64 activation block
  static constexpr int kStages = 4;
  static constexpr int kEpiWarps = 8;
  static constexpr int kStgBytes = 32 * 128;
  static constexpr int kThreads = 64 + 32 * kEpiWarps;
  static constexpr uint32_t kTmemCols = 512;  // two 256-column accumulators
  static constexpr int kSmemBytes = kWBytes + kStages * kABytes + kEpiWarps * kStgBytes + 1024 + 256;
};

// B (weights) MN-major [K][N] (the flat parameter block), A K-major activations.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg::kThreads, 1)
    umma_fwd_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmC, const GemmArgs args, int tiles_m2) {
  using C = PairCfg;
  using namespace pair_detail;
  constexpr int BM = C::BM, BK = C::BK, S = C::kStages, UK = 16;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*bf16*/, false, true /*B MN-major*/, 2 * BM, 2 * C::BNC);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sA = sW + C::kWBytes;
  uint8_t* staging = sA + S * C::kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + C::kEpiWarps * C::kStgBytes);  // leader's are used
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull = empty_bar + S;
  uint64_t* tempty = tfull + 2;  // leader's are used
  uint64_t* wfull = tempty + 2;  // leader's is used
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wfull + 1);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = int(blockIdx.x >> 1), npairs = int(gridDim.x >> 1);
  const int n_half = pair & 1, pair_in_half = pair >> 1, pairs_per_half = npairs >> 1;
  const int num_kb = (args.K + BK - 1) / BK;
  ptx::pdl_launch_dependents();

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    ptx::tma_prefetch_desc(&tmC);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full_bar[s], 2);   // one arrival per CTA (+ both CTAs' bytes)
      ptx::mbar_init(&empty_bar[s], 1);  // the leader's multicast commit
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * C::kEpiWarps);  // one arrival per epilogue warp of both CTAs
    }
    ptx::mbar_init(wfull, 2);
    ptx::fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<C::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barrier inits and TMEM address visible pair-wide
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint32_t lw = mapa(ptx::smem_u32(wfull), 0);
      ptx::pdl_wait();  // weights / activations may come from the previous kernel
      // resident weight slice: columns [256 h + 128 r, +128), every K block
      const uint32_t wbytes = uint32_t(num_kb) * C::BNC * 128;
      expect_tx_remote(lw, wbytes);
      for (int kb = 0; kb < num_kb; ++kb) {
#pragma unroll
        for (int c = 0; c < C::BNC / 64; ++c)
          tma_load_2sm(sW + (kb * (C::BNC / 64) + c) * (BK * 128), &tmB, lw, n_half * 256 + int(rank) * C::BNC + c * 64,
                       kb * BK);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int i = pair_in_half; i < tiles_m2; i += pairs_per_half) {
        const int m0 = i * 2 * BM + int(rank) * BM;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          const uint32_t lf = mapa(ptx::smem_u32(&full_bar[stage]), 0);
          expect_tx_remote(lf, C::kABytes);
          tma_load_2sm(sA + stage * C::kABytes, &tmA, lf, kb * BK, m0);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (rank == 0 && lane == 0) {
      ptx::mbar_wait(wfull, 0);
      ptx::tc_fence_after();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      const uint32_t w0 = ptx::smem_u32(sW), a0 = ptx::smem_u32(sA);
      for (int i = pair_in_half; i < tiles_m2; i += pairs_per_half, ++it) {
        const int acc = it & 1;
        const uint32_t use = uint32_t(it >> 1);
        ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * 2 * C::BNC);
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = a0 + stage * C::kABytes;
          const uint32_t sb = w0 + kb * (C::BNC / 64) * (BK * 128);
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = ptx::sw128_desc(sa + kk * UK * 2, 16, 1024);
            const uint64_t bd = ptx::sw128_desc(sb + kk * args.mn_kstep, BK * 128, args.mn_sbo, args.mn_layout);
            umma_f16_pair(d, ad, bd, kIdesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          commit_pair(&empty_bar[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        commit_pair(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue warps 2..9 (both CTAs)
    const int ew = int(warp) - 2;
    const int quarter = int(warp & 3);
    const int half = ew >> 2;
    uint8_t* stg = staging + ew * C::kStgBytes;
    const uint32_t lt[2] = {mapa(ptx::smem_u32(&tempty[0]), 0), mapa(ptx::smem_u32(&tempty[1]), 0)};
    int it = 0;
    for (int i = pair_in_half; i < tiles_m2; i += pairs_per_half, ++it) {
      const int acc = it & 1;
      const uint32_t use = uint32_t(it >> 1);
      const int m0 = i * 2 * BM + int(rank) * BM;
      ptx::mbar_wait(&tfull[acc], use & 1);
      ptx::tc_fence_after();
      const uint32_t t_acc = tmem_base + uint32_t(acc * 2 * C::BNC + half * C::BNC) + (uint32_t(quarter * 32) << 16);
      fwd_epi_tile<C::BNC>(args, &tmC, stg, t_acc, m0, quarter, n_half * 256 + half * C::BNC, 2 * n_half + half, [&] {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_remote(lt[acc]);
      });
    }
    if (lane == 0) fwd_detail::bulk_wait0();
    __syncwarp();
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();  // no CTA leaves while its peer's MMAs / commits may still target it
  if (warp == 2) {
    ptx::tc_fence_after();
    tmem_dealloc_pair<C::kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------------------------
// Split-bf16 scoring layer (MOSES_PREC_BF16X3 at scoring sizes): the weight-resident CTA pair with every
// operand a hi / lo bf16 pair and each product formed as A_hi W_hi + A_hi W_lo + A_lo W_hi (the split
// chain's arithmetic, mlp_chain_split.cuh). A 128-column hi + lo weight slice would be 256 KB, so the
// pair covers N = 128 (64 weight columns per CTA, both planes resident: 128 KB) and four pair groups
// cover the 512 output columns. Activations stream in 32-column K-blocks (64B-swizzled, hi | lo = 16 KB
// per stage, 4 stages): the ring releases a stage every 6 MMAs (M = 256, N = 128, ~400 cycles), which
// keeps ~3 stages of loads ahead of the tensor core inside the 64 KB the resident weights leave (two
// 32 KB stages left the MMAs waiting on their data: tensor pipe 42-50%). The hi / lo outputs leave
// through TMA-stored staging boxes (fwd_epi_tile SPLIT).
//
//   pair p: output columns [128 (p % 4), +128), m tiles of 256 rows p/4, p/4 + pairs/4, ...
//   CTA r of the pair: rows [256 i + 128 r, +128), weight columns [128 (p % 4) + 64 r, +64)
struct PairSplitCfg {
  static constexpr int BM = 128;   // rows per CTA (pair tile: 256)
  static constexpr int BNC = 64;   // weight columns per CTA (pair N: 128)
  static constexpr int BKW = 64;   // K rows per resident weight box (SW128, MN-major)
  static constexpr int BKA = 32;   // K columns per activation block (64 B rows, SWIZZLE_64B)
  static constexpr int kMaxK = 512;
  static constexpr int kWPlane = kMaxK / BKW * BNC * 128;  // resident weight slice, one plane: 64 KB
  static constexpr int kWBytes = 2 * kWPlane;
  static constexpr int kAPlane = BM * BKA * 2;             // one 128 x 32 activation block: 8 KB
  static constexpr int kStageBytes = 2 * kAPlane;          // hi | lo
  // The activation ring is TMA-latency bound (an 8 KB x 2 block lands ~2-3K cycles after issue against 384
  // MMA cycles per block): 4 epilogue warps (each draining both 64-column halves of its lane quarter,
  // well inside a tile's MMA time) leave shared memory for a fifth stage.
  static constexpr int kStages = 5;
  static constexpr int kEpiWarps = 4;
  static constexpr int kStgBytes = 32 * 128;
  static constexpr int kThreads = 64 + 32 * kEpiWarps;
  static constexpr uint32_t kTmemCols = 256;  // two 128-column accumulators
  static constexpr int kSmemBytes = kWBytes + kStages * kStageBytes + kEpiWarps * kStgBytes + 1024 + 256;
};
static_assert(PairSplitCfg::kSmemBytes <= 232448, "split pair layer exceeds shared memory");

// K-block order of a fused-chain layer fed by the previous one (8 blocks of 64 from the four CTAs'
// 128-column slices, two 64-column halves each), for the CTA computing output column group q: its own
// two blocks first (the chain consumes them straight from its epilogue's staging), then the other
// CTAs' first halves, then their second halves (each half is signalled on its own).
__host__ __device__ __forceinline__ int chain_korder(int q, int i) {
  if (i < 2) return 2 * q + i;
  const int j = (i - 2) % 3, h = (i - 2) / 3;
  return 2 * (j + (j >= q ? 1 : 0)) + h;
}
// 32-column activation K-block at position i: the 64-column blocks in chain_korder order for column
// group q (kperm), each as its two 32-column halves
__device__ __forceinline__ int pair_kb(bool kperm, int q, int i) {
  return kperm ? chain_korder(q, i >> 1) * 2 + (i & 1) : i;
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairSplitCfg::kThreads, 1)
    umma_fwd_pair_split(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmA_lo,
                        const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmB_lo,
                        const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC_lo,
                        const GemmArgs args, int tiles_m2) {
  using C = PairSplitCfg;
  using namespace pair_detail;
  constexpr int BM = C::BM, S = C::kStages, UK = 16;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*bf16*/, false, true /*B MN-major*/, 2 * BM, 2 * C::BNC);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;  // hi plane [0, kWPlane), lo plane [kWPlane, 2 kWPlane)
  uint8_t* sA = sW + C::kWBytes;
  uint8_t* staging = sA + S * C::kStageBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + C::kEpiWarps * C::kStgBytes);  // leader's are used
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull = empty_bar + S;
  uint64_t* tempty = tfull + 2;  // leader's are used
  uint64_t* wfull = tempty + 2;  // leader's is used
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wfull + 1);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = int(blockIdx.x >> 1), npairs = int(gridDim.x >> 1);
  const int nq = pair & 3, pair_in_q = pair >> 2, pairs_per_q = npairs >> 2;
  const int num_kbw = (args.K + C::BKW - 1) / C::BKW;
  const int num_kba = (args.K + C::BKA - 1) / C::BKA;
  ptx::pdl_launch_dependents();

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmA_lo);
    ptx::tma_prefetch_desc(&tmB);
    ptx::tma_prefetch_desc(&tmB_lo);
    ptx::tma_prefetch_desc(&tmC);
    ptx::tma_prefetch_desc(&tmC_lo);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full_bar[s], 2);   // one arrival per CTA (+ both CTAs' bytes)
      ptx::mbar_init(&empty_bar[s], 1);  // the leader's multicast commit
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * C::kEpiWarps);  // one arrival per epilogue warp of both CTAs
    }
    ptx::mbar_init(wfull, 2);
    ptx::fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<C::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barrier inits and TMEM address visible pair-wide
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint32_t lw = mapa(ptx::smem_u32(wfull), 0);
      ptx::pdl_wait();  // weights / activations may come from the previous kernel
      // resident weight slice, both planes: columns [128 nq + 64 r, +64), every K block
      expect_tx_remote(lw, uint32_t(num_kbw) * C::BNC * 128 * 2);
      for (int kb = 0; kb < num_kbw; ++kb) {
        const int col = nq * 128 + int(rank) * C::BNC;
        tma_load_2sm(sW + kb * (C::BKW * 128), &tmB, lw, col, kb * C::BKW);
        tma_load_2sm(sW + C::kWPlane + kb * (C::BKW * 128), &tmB_lo, lw, col, kb * C::BKW);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int i = pair_in_q; i < tiles_m2; i += pairs_per_q) {
        const int m0 = i * 2 * BM + int(rank) * BM;
        for (int i = 0; i < num_kba; ++i) {
          const int kb = pair_kb(args.kperm != 0, nq, i);
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          const uint32_t lf = mapa(ptx::smem_u32(&full_bar[stage]), 0);
          expect_tx_remote(lf, C::kStageBytes);
          uint8_t* dst = sA + stage * C::kStageBytes;
          tma_load_2sm(dst, &tmA, lf, kb * C::BKA, m0);
          tma_load_2sm(dst + C::kAPlane, &tmA_lo, lf, kb * C::BKA, m0);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (rank == 0 && lane == 0) {
      ptx::mbar_wait(wfull, 0);
      ptx::tc_fence_after();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      const uint32_t w0 = ptx::smem_u32(sW), a0 = ptx::smem_u32(sA);
      for (int i = pair_in_q; i < tiles_m2; i += pairs_per_q, ++it) {
        const int acc = it & 1;
        const uint32_t use = uint32_t(it >> 1);
        ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * 2 * C::BNC);
        for (int i = 0; i < num_kba; ++i) {
          const int kb = pair_kb(args.kperm != 0, nq, i);
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sah = a0 + stage * C::kStageBytes, sal = sah + C::kAPlane;
          // the weight box holding these 32 K rows, and the 16-row step inside it
          const uint32_t sbh = w0 + (kb >> 1) * (C::BKW * 128), sbl = sbh + C::kWPlane;
#pragma unroll
          for (int kk = 0; kk < C::BKA / UK; ++kk) {
            // A: K-major 64-byte rows, SWIZZLE_64B (8-row groups 512 B apart; layout type 4)
            const uint64_t ah = ptx::sw128_desc(sah + kk * UK * 2, 16, 512, 4);
            const uint64_t al = ptx::sw128_desc(sal + kk * UK * 2, 16, 512, 4);
            const int ks = (kb & 1) * (C::BKA / UK) + kk;
            const uint64_t bh = ptx::sw128_desc(sbh + ks * args.mn_kstep, C::BKW * 128, args.mn_sbo, args.mn_layout);
            const uint64_t bl = ptx::sw128_desc(sbl + ks * args.mn_kstep, C::BKW * 128, args.mn_sbo, args.mn_layout);
            umma_f16_pair(d, ah, bh, kIdesc, (i > 0 || kk > 0) ? 1u : 0u);
            umma_f16_pair(d, ah, bl, kIdesc, 1u);
            umma_f16_pair(d, al, bh, kIdesc, 1u);
          }
          commit_pair(&empty_bar[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        commit_pair(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue warps 2..5 (both CTAs)
    // warp w: TMEM lane quarter w % 4, both 64-column halves of the accumulator in turn
    const int ew = int(warp) - 2;
    const int quarter = int(warp & 3);
    uint8_t* stg = staging + ew * C::kStgBytes;
    const uint32_t lt[2] = {mapa(ptx::smem_u32(&tempty[0]), 0), mapa(ptx::smem_u32(&tempty[1]), 0)};
    int it = 0;
    for (int i = pair_in_q; i < tiles_m2; i += pairs_per_q, ++it) {
      const int acc = it & 1;
      const uint32_t use = uint32_t(it >> 1);
      const int m0 = i * 2 * BM + int(rank) * BM;
      ptx::mbar_wait(&tfull[acc], use & 1);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        const uint32_t t_acc =
            tmem_base + uint32_t(acc * 2 * C::BNC + half * C::BNC) + (uint32_t(quarter * 32) << 16);
        fwd_epi_tile<C::BNC, true>(args, &tmC, stg, t_acc, m0, quarter, nq * 128 + half * C::BNC, 2 * nq + half,
                                   [&] {
                                     if (half == 1) {  // the whole accumulator is in registers / staged
                                       ptx::tc_fence_before();
                                       __syncwarp();
                                       if (lane == 0) arrive_remote(lt[acc]);
                                     }
                                   },
                                   &tmC_lo);
      }
    }
    if (lane == 0) fwd_detail::bulk_wait0();
    __syncwarp();
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();  // no CTA leaves while its peer's MMAs / commits may still target it
  if (warp == 2) {
    ptx::tc_fence_after();
    tmem_dealloc_pair<C::kTmemCols>(tmem_base);
  }
}

}  // namespace moses
