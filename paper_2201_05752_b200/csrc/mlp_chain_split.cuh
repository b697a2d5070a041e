// mlp_chain_split.cuh — the fused hidden-layer chain (mlp_chain.cuh) in split-bf16 precision
// (MOSES_PREC_BF16X3): every GEMM operand is a pair of bf16 planes, v = hi + lo with
// hi = rn_bf16(v), lo = rn_bf16(v - hi) (|v - hi - lo| <= 2^-18 |v|), and every product is formed
// as A_hi*W_hi + A_hi*W_lo + A_lo*W_hi on the bf16 tensor cores (the lo*lo term is below 2^-16 of
// the product). Predictions, losses and gradients then sit ~1e-5 from the fp64 reference instead
// of the ~5e-3 of single bf16 operands (tools/precision_probe.py), at 3x the MMA work of bf16.
//
// Decomposition as the bf16 chain: a 4-CTA cluster owns a 128-row block for all layers, CTA q
// computes output columns [128q, 128q+128). Two operand planes do not fit a resident 128 x 512
// activation tile next to a weight ring (2 x 128 KB), and a tile is read once per layer anyway, so
// every operand K-block streams (see the streamed form below). Measured and dropped: a resident hi
// tile + streamed lo plane (same step time, less in flight); 64-row blocks on all 148 SMs (slower:
// 2x the weight traffic, M = 64 MMAs, starved side-stream kernels).
#pragma once
#include "mlp_chain.cuh"
#include "gemm_fwd2.cuh"

namespace moses {

struct ChainSplitMaps {
  CUtensorMap in, in_lo;                 // chain input hi / lo planes [M][K0], box {64, 128}
  CUtensorMap w[kChainMaxLayers];        // as ChainMaps::w (hi shadow)
  CUtensorMap w_lo[kChainMaxLayers];     // the lo shadow, same boxes
  CUtensorMap out[kChainMaxLayers];      // hi outputs: TMA store + multicast reload, box {64, 128}
  CUtensorMap out_lo[kChainMaxLayers];   // lo outputs: the next layer's A_lo stream, box {64, 128}
};

namespace chain_detail {
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// one cluster-scope release fence, then relaxed arrivals on several peers' barriers (a .release arrive
// fences on every call)
__device__ __forceinline__ void fence_release_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAITC_%=;\n\t}\n" ::"r"(ptx::smem_u32(bar)),
      "r"(parity)
      : "memory");
}
}  // namespace chain_detail

// ---------------------------------------------------------------------------------------------
// Streamed form: no resident activation tile. Every operand K-block streams from L2 through a
// 3-stage ring of [W_hi | W_lo | A_hi | A_lo] (4 x 16 KB), twice the bytes in flight of the
// resident form (which spends 128 KB of shared memory on a tile each K-block of is read once per
// layer). The epilogue writes both planes of its 128 x 128 output slice to global memory; the four
// CTAs of the cluster signal each other through a remote arrive on every CTA's `ready` mbarrier
// (count 4, one phase per layer), after which the producers stream the next layer's A blocks. The
// next layer's first weight blocks are prefetched while the epilogue runs.
struct ChainSplitStreamCfg {
  static constexpr int BM = 128, BN = 128, BK = 64, kWidth = 512, kCluster = 4;
  static constexpr int kTile = BM * 128;                    // one 64-col K-block of a 128-row bf16 plane
  static constexpr int kStages = 3;
  static constexpr int kWBytes = BN * 128;                  // one K-block of one weight plane (16 KB)
  static constexpr int kStageBytes = 2 * kWBytes + 2 * kTile;  // W_hi | W_lo | A_hi | A_lo
  static constexpr int kParamFloats = kChainMaxLayers * BN + 2 * BN;  // bias slices + head_w / head_u slices
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256 + kParamFloats * 4;
  // warps 0-7 epilogue (warp w: TMEM lanes 32 (w % 4).., columns 64 (w / 4)..), 8 TMA producer of the
  // weight blocks, 9 MMA, 10 TMA producer of the activation blocks (two issuing warps: ~1.3x the per-SM
  // TMA ingest of one, profiles/r2/tma_ingest_bench.json)
  static constexpr int kEpiWarps = 8, kProducerWarp = 8, kMmaWarp = 9, kAProducerWarp = 10, kThreads = 352;
};
static_assert(ChainSplitStreamCfg::kSmemBytes <= 232448, "streamed split chain exceeds shared memory");

template <bool FWD>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(ChainSplitStreamCfg::kThreads, 1)
    mlp_chain_split_stream_kernel(const __grid_constant__ ChainSplitMaps maps, const __grid_constant__ ChainArgs args) {
  using namespace chain_detail;
  using C = ChainSplitStreamCfg;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, S = C::kStages;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*BF16*/, false, FWD /*B MN-major*/, BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sRing = smem;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(sRing + S * C::kStageBytes);
  uint64_t* wempty = wfull + S;
  uint64_t* acc_full = wempty + S;
  uint64_t* ready = acc_full + 1;  // [2]: half h (columns [64h, 64h+64) of every CTA's slice) is in global memory
  uint64_t* staged = ready + 2;    // this CTA's half-1 staging (in the ring's A areas) has been read out
  uint64_t* own_staged = staged + 1;  // both halves of this CTA's slice are staged (and TMEM is read out)
  uint64_t* own_done = own_staged + 1;  // the MMAs reading the staged slice as the next layer's A are done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(own_done + 1);
  float* s_bias = reinterpret_cast<float*>(sRing + S * C::kStageBytes + 256);  // [layer][BN] (FWD)
  float* s_head = s_bias + kChainMaxLayers * BN;                                // [2][BN] head_w, head_u

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const uint32_t q = ptx::cluster_ctarank();
  const int m0 = int(blockIdx.x / C::kCluster) * BM, n0 = int(q) * BN;
  const int L = args.n_layers;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&wfull[s], 2);  // weight producer + activation producer (each with its bytes)
      ptx::mbar_init(&wempty[s], 1);
    }
    ptx::mbar_init(acc_full, 1);
    ptx::mbar_init(&ready[0], C::kCluster);
    ptx::mbar_init(&ready[1], C::kCluster);
    ptx::mbar_init(staged, 1);
    ptx::mbar_init(own_staged, 2);
    ptx::mbar_init(own_done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<BN>(tmem_slot);
  ptx::pdl_wait();
  if (threadIdx.x == 0) CHAIN_TRACE(6, 0);
  if constexpr (FWD) {  // the slices of every layer's bias and of the head vectors, once
    for (int i = threadIdx.x; i < L * BN; i += blockDim.x) {
      const int l = i / BN, j = i - l * BN;
      s_bias[i] = args.bias[l] ? __ldg(args.bias[l] + n0 + j) : 0.f;
    }
    for (int j = threadIdx.x; j < BN; j += blockDim.x) {
      s_head[j] = args.head_w ? __ldg(args.head_w + n0 + j) : 0.f;
      s_head[BN + j] = args.head_u ? __ldg(args.head_u + n0 + j) : 0.f;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();      // CTA-level order of the inits / parameter slices (what compute-sanitizer tracks)
  ptx::cluster_sync();  // barrier inits visible cluster-wide before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == C::kProducerWarp) {
    // ------------------------------------------------------------ TMA producer: weight blocks
    // Runs ahead of the activation producer by up to the ring depth (the next layer's first weight
    // blocks land while this layer's MMAs / epilogue run). Position order per layer: chain_korder.
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int l = 0; l < L; ++l) {
        const int nkb = (args.K[l] + BK - 1) / BK;
        const bool perm = l > 0 && nkb == 2 * C::kCluster;
        for (int i = 0; i < nkb; ++i) {
          const int kb = perm ? chain_korder(int(q), i) : i;
          ptx::mbar_wait(&wempty[stage], phase ^ 1);
          uint8_t* dst = sRing + stage * C::kStageBytes;
          ptx::mbar_arrive_expect_tx(&wfull[stage], 2 * C::kWBytes);
          if constexpr (FWD) {
            ptx::tma_load_2d(dst, &maps.w[l], &wfull[stage], n0, kb * BK);
            ptx::tma_load_2d(dst + BK * 128, &maps.w[l], &wfull[stage], n0 + 64, kb * BK);
            ptx::tma_load_2d(dst + C::kWBytes, &maps.w_lo[l], &wfull[stage], n0, kb * BK);
            ptx::tma_load_2d(dst + C::kWBytes + BK * 128, &maps.w_lo[l], &wfull[stage], n0 + 64, kb * BK);
          } else {
            ptx::tma_load_2d(dst, &maps.w[l], &wfull[stage], kb * BK, n0);
            ptx::tma_load_2d(dst + C::kWBytes, &maps.w_lo[l], &wfull[stage], kb * BK, n0);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == C::kAProducerWarp) {
    // ------------------------------------------------------------ TMA producer: activation blocks
    // Layers fed by the previous one (chain_korder): positions 0-1 are this CTA's own slice, which the MMA
    // warp reads straight from the epilogue's staging (the ring stage only brings its weights: a plain
    // arrive); positions 2-4 are the other CTAs' first halves (ready[0]), 5-7 their second halves
    // (ready[1]). Before any load into the ring's A areas: the MMAs reading the staging are done
    // (own_done) and the epilogue's bulk stores have read it out (staged).
    if (lane == 0) {
      ptx::tma_prefetch_desc(&maps.in);
      ptx::tma_prefetch_desc(&maps.in_lo);
      int stage = 0;
      uint32_t phase = 0;
      for (int l = 0; l < L; ++l) {
        const int nkb = (args.K[l] + BK - 1) / BK;
        const bool perm = l > 0 && nkb == 2 * C::kCluster;
        const CUtensorMap* hi = l == 0 ? &maps.in : &maps.out[l - 1];
        const CUtensorMap* lo = l == 0 ? &maps.in_lo : &maps.out_lo[l - 1];
        if (l > 0 && !perm) {
          ptx::mbar_wait(staged, uint32_t(l - 1) & 1u);
          mbar_wait_cluster(&ready[0], uint32_t(l - 1) & 1u);
          mbar_wait_cluster(&ready[1], uint32_t(l - 1) & 1u);
          fence_proxy_async_global();
          CHAIN_TRACE(4, l);
        }
        for (int i = 0; i < nkb; ++i) {
          const int kb = perm ? chain_korder(int(q), i) : i;
          ptx::mbar_wait(&wempty[stage], phase ^ 1);
          if (perm && i < 2) {
            ptx::mbar_arrive(&wfull[stage]);  // own block: no activation bytes through the ring
          } else {
            if (perm && i == 2) {
              ptx::mbar_wait(own_done, uint32_t(l - 1) & 1u);
              ptx::mbar_wait(staged, uint32_t(l - 1) & 1u);
              mbar_wait_cluster(&ready[0], uint32_t(l - 1) & 1u);
              fence_proxy_async_global();
              CHAIN_TRACE(4, l);
            }
            if (perm && i == 5) {
              mbar_wait_cluster(&ready[1], uint32_t(l - 1) & 1u);
              fence_proxy_async_global();
            }
            uint8_t* dst = sRing + stage * C::kStageBytes + 2 * C::kWBytes;
            ptx::mbar_arrive_expect_tx(&wfull[stage], 2 * C::kTile);
            ptx::tma_load_2d(dst, hi, &wfull[stage], kb * BK, m0);
            ptx::tma_load_2d(dst + C::kTile, lo, &wfull[stage], kb * BK, m0);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == C::kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    for (int l = 0; l < L; ++l) {
      if (lane == 0) {
        const int nkb = (args.K[l] + BK - 1) / BK;
        const bool perm = l > 0 && nkb == 2 * C::kCluster;
        const uint32_t r0 = ptx::smem_u32(sRing);
        for (int kb = 0; kb < nkb; ++kb) {
          if (perm && kb == 0) {  // this CTA's slice of the previous layer is staged: its blocks first
            ptx::mbar_wait(own_staged, uint32_t(l - 1) & 1u);
            ptx::tc_fence_after();
          }
          ptx::mbar_wait(&wfull[stage], phase);
          ptx::tc_fence_after();
          if (kb == 0) CHAIN_TRACE(0, l);
          const uint32_t sb = r0 + stage * C::kStageBytes, sbl = sb + C::kWBytes;
          // own blocks (positions 0-1): half kb of the staged slice, hi in stage 0's A areas, lo in stage 1's
          const uint32_t sah = (perm && kb < 2) ? r0 + 2 * C::kWBytes + kb * C::kTile : sb + 2 * C::kWBytes;
          const uint32_t sal = (perm && kb < 2) ? r0 + C::kStageBytes + 2 * C::kWBytes + kb * C::kTile : sah + C::kTile;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ah = ptx::sw128_desc(sah + kk * 32, 16, 1024);
            const uint64_t al = ptx::sw128_desc(sal + kk * 32, 16, 1024);
            const uint64_t bh = FWD ? ptx::sw128_desc(sb + kk * 2048, BK * 128, 1024, 2)
                                    : ptx::sw128_desc(sb + kk * 32, 16, 1024);
            const uint64_t bl = FWD ? ptx::sw128_desc(sbl + kk * 2048, BK * 128, 1024, 2)
                                    : ptx::sw128_desc(sbl + kk * 32, 16, 1024);
            ptx::umma_f16(tmem, ah, bh, kIdesc, (kb > 0 || kk > 0) ? 1u : 0u);
            ptx::umma_f16(tmem, ah, bl, kIdesc, 1u);
            ptx::umma_f16(tmem, al, bh, kIdesc, 1u);
          }
          ptx::umma_commit(&wempty[stage]);
          if (perm && kb == 1) ptx::umma_commit(own_done);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(acc_full);
        CHAIN_TRACE(1, l);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue warps 0-7
    // warp w: rows 32 (w % 4).. of the block, columns [64h, 64h + 64) of the slice (h = w / 4); the
    // four warps of half h stage it, and one of them stores and signals it (ready[h])
    const int h = int(warp) >> 2;
    const int row = int(warp & 3) * 32 + int(lane);
    const int m = m0 + row;
    const bool row_ok = m < args.M;
    const uint32_t t_row = tmem + ((uint32_t(warp & 3) * 32u) << 16) + uint32_t(h * 64);
    const bool issuer = (threadIdx.x & 127) == 0;  // thread 0 of warp 4h
    for (int l = 0; l < L; ++l) {
      const bool last = l + 1 == L;
      uint4 mk[2][4];
      if constexpr (!FWD) {
        if (row_ok) {
          const uint4* src = reinterpret_cast<const uint4*>(args.mask[l] + (long long)m * args.ldm[l] + n0 + h * 64);
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int v = 0; v < 4; ++v) mk[c][v] = __ldg(src + c * 4 + v);
        }
      }
      ptx::mbar_wait(acc_full, uint32_t(l) & 1u);
      ptx::tc_fence_after();
      if (threadIdx.x == 0) CHAIN_TRACE(2, l);
      const bool store = !last || args.out[l] != nullptr;
      // the output slice is staged in the A areas of ring stages 0 (hi) and 1 (lo) — free while the
      // epilogue runs: this layer's MMAs are complete and the next layer's A loads wait for `staged` /
      // `ready` — in the TMA store boxes' SW128 layout (half h = box h), then leaves in bulk stores
      uint8_t* st_hi = sRing + 2 * C::kWBytes + h * C::kTile;
      uint8_t* st_lo = sRing + C::kStageBytes + 2 * C::kWBytes + h * C::kTile;
      float hp = 0.f, hp2 = 0.f;
      uint32_t rr[2][32];  // both 32-column chunks of the half in flight
      ptx::tmem_ld_32x32b_x32(t_row, rr[0]);
      ptx::tmem_ld_32x32b_x32(t_row + 32, rr[1]);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[c][j]);
        if constexpr (FWD) {
          const float* sb = s_bias + l * BN + h * 64 + c * 32;
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j] + sb[j], 0.f);
          if (last) {
            if (args.head_w != nullptr) {
#pragma unroll
              for (int j = 0; j < 32; ++j) hp = fmaf(v[j], s_head[h * 64 + c * 32 + j], hp);
            }
            if (args.head_u != nullptr) {
#pragma unroll
              for (int j = 0; j < 32; ++j) hp2 = fmaf(v[j], s_head[BN + h * 64 + c * 32 + j], hp2);
            }
          }
        } else {
          const __nv_bfloat16* mv = reinterpret_cast<const __nv_bfloat16*>(mk[c]);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __bfloat162float(mv[j]) > 0.f ? v[j] : 0.f;
        }
        if (store) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 ph, pl;
            uint32_t* hw = reinterpret_cast<uint32_t*>(&ph);
            uint32_t* lw = reinterpret_cast<uint32_t*>(&pl);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[j + 2 * e], v[j + 2 * e + 1]);
              const __nv_bfloat162 l2 = __floats2bfloat162_rn(v[j + 2 * e] - __low2float(h2),
                                                              v[j + 2 * e + 1] - __high2float(h2));
              hw[e] = *reinterpret_cast<const uint32_t*>(&h2);
              lw[e] = *reinterpret_cast<const uint32_t*>(&l2);
            }
            const int col = c * 32 + j;  // within the half
            const int off = row * 128 + (((col >> 3) ^ (row & 7)) << 4);
            *reinterpret_cast<uint4*>(st_hi + off) = ph;
            *reinterpret_cast<uint4*>(st_lo + off) = pl;
          }
        }
      }
      if (FWD && last && row_ok) {  // per-64-column head partials (8 per row), as the scoring pair layers
        if (args.head_part != nullptr) args.head_part[(long long)(2 * q + h) * args.head_ld + m] = hp;
        if (args.head_part2 != nullptr) args.head_part2[(long long)(2 * q + h) * args.head_ld + m] = hp2;
      }
      if (store) {
        ptx::tc_fence_before();
        fence_proxy_async_smem();
        bar_sync(2 + h, 128);
        if (issuer) {
          if (!last) ptx::mbar_arrive(own_staged);  // the next layer's MMAs may read this half (and TMEM is free)
          tma_store_2d(&maps.out[l], st_hi, n0 + 64 * h, m0);
          tma_store_2d(&maps.out_lo[l], st_lo, n0 + 64 * h, m0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          if (h == 1) ptx::mbar_arrive(staged);  // half 0's areas are covered by this CTA's ready[0] arrival
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          if (h == 1) CHAIN_TRACE(3, l);
          if (!last) {
            const uint32_t local = ptx::smem_u32(&ready[h]);
#pragma unroll
            fence_release_cluster();
            for (uint32_t p = 0; p < uint32_t(C::kCluster); ++p) mbar_arrive_cluster_relaxed(mapa(local, p));
          }
        }
        bar_sync(2 + h, 128);  // the staging areas are reusable (next layer's epilogue)
      } else if (h == 1 && issuer) {
        ptx::mbar_arrive(staged);  // nothing staged: keep the phase count per layer
      }
    }
    if (threadIdx.x == 0) CHAIN_TRACE(7, 0);
    ptx::pdl_launch_dependents();
  }

  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();  // no CTA leaves while a remote arrive into it could still be in flight
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<BN>(tmem);
  }
}


// ---------------------------------------------------------------------------------------------
// CTA-pair form (moses_debug_set_chain_pair; not the default): tcgen05.mma.cta_group::2. Built on the
// hypothesis that the streamed form's K-blocks (~1.16K cycles against 768 of MMA) are bound by the smem
// port, which a cta_group::1 M = 128 MMA saturates (8 KB of operand reads per 64-cycle N = 128 MMA).
// Measured: no faster. The per-position trace (tools/chain_trace.py) shows the ring is TMA-latency
// bound instead — an activation block lands ~1.9 us after it is issued, and 3-4 positions in flight
// cover only ~3K MMA cycles — and at cfg5 the 8-CTA clusters do not all fit at once. Here an 8-CTA cluster owns
// 256 rows: CTA c = 2q + r computes rows [128 r, +128) of the block and columns [128 q, +128); the
// pair (2q, 2q+1) issues M = 256, N = 128 MMAs from its leader, each CTA supplying its own 128 rows of
// A and half (64 columns) of the weight slice: 6 KB of operand reads per MMA per SM, and half the
// weight stream. Per element the MMA sequence (K order, hi*hi, hi*lo, lo*hi) is the streamed form's,
// so results are bit-identical to it. The four CTAs of a row block exchange their slices as there
// (ready[h] counts the four CTAs with the same r).
struct ChainPairCfg {
  static constexpr int BM = 128, BN = 128, BK = 64, kWidth = 512, kCluster = 8;
  static constexpr int kTile = BM * 128;                       // one 64-col K-block of a 128-row plane
  static constexpr int kWHalf = 64 * 128;                      // one K-block of one weight plane's half (8 KB)
  static constexpr int kStages = 4;
  static constexpr int kStageBytes = 2 * kWHalf + 2 * kTile;   // W_hi | W_lo (halves) | A_hi | A_lo: 48 KB
  static constexpr int kParamFloats = kChainMaxLayers * BN + 2 * BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256 + kParamFloats * 4;
  static constexpr int kEpiWarps = 8, kProducerWarp = 8, kMmaWarp = 9, kAProducerWarp = 10, kThreads = 352;
};
static_assert(ChainPairCfg::kSmemBytes <= 232448, "pair split chain exceeds shared memory");

namespace chain_detail {
__device__ __forceinline__ void commit_pair_mask(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          ptx::smem_u32(bar)),
      "h"(mask)
      : "memory");
}
}  // namespace chain_detail

#define CHAIN_TRACE_P(ev, l)                                                                           \
  do {                                                                                                 \
    if (args.trace != nullptr && blockIdx.x < 4)                                                       \
      args.trace[(int(blockIdx.x) * kChainMaxLayers + (l)) * 8 + (ev)] = chain_detail::clk();          \
  } while (0)

template <bool FWD>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(ChainPairCfg::kThreads, 1)
    mlp_chain_split_pair_kernel(const __grid_constant__ ChainSplitMaps maps, const __grid_constant__ ChainArgs args) {
  using namespace chain_detail;
  using pair_detail::tma_load_2sm;
  using pair_detail::expect_tx_remote;
  using pair_detail::umma_f16_pair;
  using pair_detail::tmem_alloc_pair;
  using pair_detail::tmem_dealloc_pair;
  using C = ChainPairCfg;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, S = C::kStages;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*BF16*/, false, FWD /*B MN-major*/, 2 * BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sRing = smem;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(sRing + S * C::kStageBytes);  // the leader's are used
  uint64_t* wempty = wfull + S;
  uint64_t* acc_full = wempty + S;
  uint64_t* ready = acc_full + 1;  // [2]
  uint64_t* staged = ready + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(staged + 1);
  float* s_bias = reinterpret_cast<float*>(sRing + S * C::kStageBytes + 256);
  float* s_head = s_bias + kChainMaxLayers * BN;

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const uint32_t c = ptx::cluster_ctarank();
  const uint32_t q = c >> 1, r = c & 1u;  // column slice, row block of the pair
  const int m0 = int(blockIdx.x / C::kCluster) * 2 * BM + int(r) * BM, n0 = int(q) * BN;
  const int wc0 = n0 + int(r) * 64;  // this CTA's half of the pair's weight columns
  const int L = args.n_layers;
  const uint16_t pair_mask = uint16_t(3u << (2 * q));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&wfull[s], 4);  // both CTAs' weight and activation producers (each with its bytes)
      ptx::mbar_init(&wempty[s], 1);
    }
    ptx::mbar_init(acc_full, 1);
    ptx::mbar_init(&ready[0], 4);
    ptx::mbar_init(&ready[1], 4);
    ptx::mbar_init(staged, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_pair<BN>(tmem_slot);
  ptx::pdl_wait();
  if (threadIdx.x == 0) CHAIN_TRACE_P(6, 0);
  if constexpr (FWD) {
    for (int i = threadIdx.x; i < L * BN; i += blockDim.x) {
      const int l = i / BN, j = i - l * BN;
      s_bias[i] = args.bias[l] ? __ldg(args.bias[l] + n0 + j) : 0.f;
    }
    for (int j = threadIdx.x; j < BN; j += blockDim.x) {
      s_head[j] = args.head_w ? __ldg(args.head_w + n0 + j) : 0.f;
      s_head[BN + j] = args.head_u ? __ldg(args.head_u + n0 + j) : 0.f;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == C::kProducerWarp) {
    // ------------------------------------------------------------ weight half blocks (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int l = 0; l < L; ++l) {
        const int nkb = (args.K[l] + BK - 1) / BK;
        const bool perm = l > 0 && nkb == 8;
        for (int i = 0; i < nkb; ++i) {
          const int kb = perm ? chain_korder(int(q), i) : i;
          ptx::mbar_wait(&wempty[stage], phase ^ 1);
          if (l == 1 && i < 8 && args.trace != nullptr && blockIdx.x == 0)
            args.trace[(0 * kChainMaxLayers + 5) * 8 + i] = chain_detail::clk();
          uint8_t* dst = sRing + stage * C::kStageBytes;
          const uint32_t lf = mapa(ptx::smem_u32(&wfull[stage]), c & ~1u);
          expect_tx_remote(lf, 2 * C::kWHalf);
          if constexpr (FWD) {
            tma_load_2sm(dst, &maps.w[l], lf, wc0, kb * BK);
            tma_load_2sm(dst + C::kWHalf, &maps.w_lo[l], lf, wc0, kb * BK);
          } else {
            tma_load_2sm(dst, &maps.w[l], lf, kb * BK, wc0);
            tma_load_2sm(dst + C::kWHalf, &maps.w_lo[l], lf, kb * BK, wc0);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == C::kAProducerWarp) {
    // ------------------------------------------------------------ activation blocks (both CTAs)
    if (lane == 0) {
      ptx::tma_prefetch_desc(&maps.in);
      ptx::tma_prefetch_desc(&maps.in_lo);
      int stage = 0;
      uint32_t phase = 0;
      for (int l = 0; l < L; ++l) {
        const int nkb = (args.K[l] + BK - 1) / BK;
        const bool perm = l > 0 && nkb == 8;
        const CUtensorMap* hi = l == 0 ? &maps.in : &maps.out[l - 1];
        const CUtensorMap* lo = l == 0 ? &maps.in_lo : &maps.out_lo[l - 1];
        if (l > 0) {
          ptx::mbar_wait(staged, uint32_t(l - 1) & 1u);
          mbar_wait_cluster(&ready[0], uint32_t(l - 1) & 1u);
          mbar_wait_cluster(&ready[1], uint32_t(l - 1) & 1u);  // own blocks come first, from global here
          fence_proxy_async_global();
          if (r == 0) CHAIN_TRACE_P(4, l);
        }
        for (int i = 0; i < nkb; ++i) {
          const int kb = perm ? chain_korder(int(q), i) : i;
          ptx::mbar_wait(&wempty[stage], phase ^ 1);
          if (l == 1 && i < 8 && args.trace != nullptr && blockIdx.x == 0)
            args.trace[(0 * kChainMaxLayers + 6) * 8 + i] = chain_detail::clk();
          uint8_t* dst = sRing + stage * C::kStageBytes + 2 * C::kWHalf;
          const uint32_t lf = mapa(ptx::smem_u32(&wfull[stage]), c & ~1u);
          expect_tx_remote(lf, 2 * C::kTile);
          tma_load_2sm(dst, hi, lf, kb * BK, m0);
          tma_load_2sm(dst + C::kTile, lo, lf, kb * BK, m0);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == C::kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    if (r == 0 && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t r0 = ptx::smem_u32(sRing);
      for (int l = 0; l < L; ++l) {
        const int nkb = (args.K[l] + BK - 1) / BK;
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait(&wfull[stage], phase);
          ptx::tc_fence_after();
          if (kb == 0) CHAIN_TRACE_P(0, l);
          if (l == 1 && kb < 8 && args.trace != nullptr && blockIdx.x == 0)
            args.trace[(0 * kChainMaxLayers + 4) * 8 + kb] = chain_detail::clk();
          const uint32_t sb = r0 + stage * C::kStageBytes, sbl = sb + C::kWHalf;
          const uint32_t sah = sb + 2 * C::kWHalf, sal = sah + C::kTile;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ah = ptx::sw128_desc(sah + kk * 32, 16, 1024);
            const uint64_t al = ptx::sw128_desc(sal + kk * 32, 16, 1024);
            const uint64_t bh = FWD ? ptx::sw128_desc(sb + kk * 2048, C::kWHalf, 1024, 2)
                                    : ptx::sw128_desc(sb + kk * 32, 16, 1024);
            const uint64_t bl = FWD ? ptx::sw128_desc(sbl + kk * 2048, C::kWHalf, 1024, 2)
                                    : ptx::sw128_desc(sbl + kk * 32, 16, 1024);
            umma_f16_pair(tmem, ah, bh, kIdesc, (kb > 0 || kk > 0) ? 1u : 0u);
            umma_f16_pair(tmem, ah, bl, kIdesc, 1u);
            umma_f16_pair(tmem, al, bh, kIdesc, 1u);
          }
          commit_pair_mask(&wempty[stage], pair_mask);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        commit_pair_mask(acc_full, pair_mask);
        CHAIN_TRACE_P(1, l);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue warps 0-7 (as the streamed form)
    const int h = int(warp) >> 2;
    const int row = int(warp & 3) * 32 + int(lane);
    const int m = m0 + row;
    const bool row_ok = m < args.M;
    const uint32_t t_row = tmem + ((uint32_t(warp & 3) * 32u) << 16) + uint32_t(h * 64);
    const bool issuer = (threadIdx.x & 127) == 0;
    for (int l = 0; l < L; ++l) {
      const bool last = l + 1 == L;
      uint4 mk[2][4];
      if constexpr (!FWD) {
        if (row_ok) {
          const uint4* src = reinterpret_cast<const uint4*>(args.mask[l] + (long long)m * args.ldm[l] + n0 + h * 64);
#pragma unroll
          for (int cc = 0; cc < 2; ++cc)
#pragma unroll
            for (int v = 0; v < 4; ++v) mk[cc][v] = __ldg(src + cc * 4 + v);
        }
      }
      ptx::mbar_wait(acc_full, uint32_t(l) & 1u);
      ptx::tc_fence_after();
      if (threadIdx.x == 0) CHAIN_TRACE_P(2, l);
      const bool store = !last || args.out[l] != nullptr;
      uint8_t* st_hi = sRing + 2 * C::kWHalf + h * C::kTile;                   // stage 0's A areas
      uint8_t* st_lo = sRing + C::kStageBytes + 2 * C::kWHalf + h * C::kTile;  // stage 1's A areas
      float hp = 0.f, hp2 = 0.f;
      uint32_t rr[2][32];
      ptx::tmem_ld_32x32b_x32(t_row, rr[0]);
      ptx::tmem_ld_32x32b_x32(t_row + 32, rr[1]);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[cc][j]);
        if constexpr (FWD) {
          const float* sbias = s_bias + l * BN + h * 64 + cc * 32;
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j] + sbias[j], 0.f);
          if (last) {
            if (args.head_w != nullptr) {
#pragma unroll
              for (int j = 0; j < 32; ++j) hp = fmaf(v[j], s_head[h * 64 + cc * 32 + j], hp);
            }
            if (args.head_u != nullptr) {
#pragma unroll
              for (int j = 0; j < 32; ++j) hp2 = fmaf(v[j], s_head[BN + h * 64 + cc * 32 + j], hp2);
            }
          }
        } else {
          const __nv_bfloat16* mv = reinterpret_cast<const __nv_bfloat16*>(mk[cc]);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __bfloat162float(mv[j]) > 0.f ? v[j] : 0.f;
        }
        if (store) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 ph, pl;
            uint32_t* hw = reinterpret_cast<uint32_t*>(&ph);
            uint32_t* lw = reinterpret_cast<uint32_t*>(&pl);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[j + 2 * e], v[j + 2 * e + 1]);
              const __nv_bfloat162 l2 = __floats2bfloat162_rn(v[j + 2 * e] - __low2float(h2),
                                                              v[j + 2 * e + 1] - __high2float(h2));
              hw[e] = *reinterpret_cast<const uint32_t*>(&h2);
              lw[e] = *reinterpret_cast<const uint32_t*>(&l2);
            }
            const int col = cc * 32 + j;
            const int off = row * 128 + (((col >> 3) ^ (row & 7)) << 4);
            *reinterpret_cast<uint4*>(st_hi + off) = ph;
            *reinterpret_cast<uint4*>(st_lo + off) = pl;
          }
        }
      }
      if (FWD && last && row_ok) {
        if (args.head_part != nullptr) args.head_part[(long long)(2 * q + h) * args.head_ld + m] = hp;
        if (args.head_part2 != nullptr) args.head_part2[(long long)(2 * q + h) * args.head_ld + m] = hp2;
      }
      if (store) {
        ptx::tc_fence_before();
        fence_proxy_async_smem();
        bar_sync(2 + h, 128);
        if (issuer) {
          tma_store_2d(&maps.out[l], st_hi, n0 + 64 * h, m0);
          tma_store_2d(&maps.out_lo[l], st_lo, n0 + 64 * h, m0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          if (h == 1) ptx::mbar_arrive(staged);
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          if (h == 1) CHAIN_TRACE_P(3, l);
          if (!last) {  // the four CTAs holding the same rows
            const uint32_t local = ptx::smem_u32(&ready[h]);
#pragma unroll
            fence_release_cluster();
            for (uint32_t p = 0; p < 4; ++p) mbar_arrive_cluster_relaxed(mapa(local, 2 * p + r));
          }
        }
        bar_sync(2 + h, 128);
      } else if (h == 1 && issuer) {
        ptx::mbar_arrive(staged);
      }
    }
    if (threadIdx.x == 0) CHAIN_TRACE_P(7, 0);
    ptx::pdl_launch_dependents();
  }

  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 0) {
    ptx::tc_fence_after();
    tmem_dealloc_pair<BN>(tmem);
  }
}
}  // namespace moses
