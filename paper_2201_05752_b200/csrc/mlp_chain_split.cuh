// mlp_chain_split.cuh — the fused hidden-layer chain (mlp_chain.cuh) in split-bf16 precision
// (MOSES_PREC_BF16X3): every GEMM operand is a pair of bf16 planes, v = hi + lo with
// hi = rn_bf16(v), lo = rn_bf16(v - hi) (|v - hi - lo| <= 2^-18 |v|), and every product is formed
// as A_hi*W_hi + A_hi*W_lo + A_lo*W_hi on the bf16 tensor cores (the lo*lo term is below 2^-16 of
// the product). Predictions, losses and gradients then sit ~1e-5 from the fp64 reference instead
// of the ~5e-3 of single bf16 operands (tools/precision_probe.py), at 3x the MMA work of bf16.
//
// Same decomposition as the bf16 chain: a 4-CTA cluster owns a 128-row block for all layers, CTA q
// computes output columns [128q, 128q+128), the layer's 128 x 512 hi activation tile stays in
// shared memory (exchanged through a TMA store + L2 multicast) — but the lo tile (another 128 KB)
// does not fit next to it. It streams from L2 instead, one 64-column K-block per pipeline stage
// together with that K-block's W_hi and W_lo slices (3 x 16 KB per stage, 2 stages):
//
//   stage s: [ W_hi(kb) 16 KB | W_lo(kb) 16 KB | A_lo(kb) 16 KB ]   one mbarrier, 48 KB expected
//
// The epilogue writes its lo slice straight to global memory; once all four CTAs' slices are there
// (fence.proxy.async + a remote arrive on every CTA's `lo_ready` mbarrier, count 4), the producer
// issues the next layer's A_lo loads. W loads of the next layer's first stages are still prefetched
// during the exchange (the stage's mbarrier expects all 48 KB, the A_lo part lands later).
#pragma once
#include "mlp_chain.cuh"

namespace moses {

struct ChainSplitMaps {
  CUtensorMap in, in_lo;                 // chain input hi / lo planes [M][K0], box {64, 128}
  CUtensorMap w[kChainMaxLayers];        // as ChainMaps::w (hi shadow)
  CUtensorMap w_lo[kChainMaxLayers];     // the lo shadow, same boxes
  CUtensorMap out[kChainMaxLayers];      // hi outputs: TMA store + multicast reload, box {64, 128}
  CUtensorMap out_lo[kChainMaxLayers];   // lo outputs: the next layer's A_lo stream, box {64, 128}
};

struct ChainSplitCfg {
  static constexpr int BM = 128, BN = 128, BK = 64, kWidth = 512, kCluster = 4;
  static constexpr int kTile = BM * 128;                    // one 64-col K-block of a 128-row bf16 tile
  static constexpr int kActBytes = (kWidth / BK) * kTile;   // 128 KB hi tile
  static constexpr int kStages = 2;
  static constexpr int kWBytes = BN * 128;                  // one K-block of one weight plane (16 KB)
  static constexpr int kStageBytes = 2 * kWBytes + kTile;   // W_hi | W_lo | A_lo
  static constexpr int kSmemBytes = kActBytes + kStages * kStageBytes + 1024 + 256;
};
static_assert(ChainSplitCfg::kSmemBytes <= 232448, "split chain exceeds the 227 KB shared-memory limit");

namespace chain_detail {
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
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

template <bool FWD>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(192, 1)
    mlp_chain_split_kernel(const __grid_constant__ ChainSplitMaps maps, const __grid_constant__ ChainArgs args) {
  using namespace chain_detail;
  using C = ChainSplitCfg;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, S = C::kStages;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*BF16*/, false, FWD /*B MN-major*/, BM, BN);
  constexpr uint16_t kAll = 0xF;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sAct = smem;
  uint8_t* sRing = smem + C::kActBytes;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(sRing + S * C::kStageBytes);
  uint64_t* wempty = wfull + S;
  uint64_t* act_full = wempty + S;
  uint64_t* acc_full = act_full + 1;
  uint64_t* slice_free = acc_full + 1;  // this CTA's outgoing TMA store finished reading its slice
  uint64_t* lo_ready = slice_free + 1;  // all four CTAs' lo slices of the layer are in global memory
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lo_ready + 1);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const uint32_t q = ptx::cluster_ctarank();
  const int m0 = int(blockIdx.x / C::kCluster) * BM, n0 = int(q) * BN;
  const int L = args.n_layers;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&wfull[s], 1);
      ptx::mbar_init(&wempty[s], 1);
    }
    ptx::mbar_init(act_full, 1);
    ptx::mbar_init(acc_full, 1);
    ptx::mbar_init(slice_free, 1);
    ptx::mbar_init(lo_ready, C::kCluster);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<BN>(tmem_slot);
  ptx::pdl_wait();  // every global read below may depend on the previous kernel
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barrier inits + TMEM address visible cluster-wide before any multicast / remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    int pend_n = 0;                 // K-blocks of the current layer whose W was issued before its A_lo
    int pend_stage[S];
    // W_hi + W_lo of (layer l, K-block kb) into the next stage; the stage also expects its A_lo block
    auto load_w = [&](int l, int kb) -> int {
      ptx::mbar_wait(&wempty[stage], phase ^ 1);
      uint8_t* dst = sRing + stage * C::kStageBytes;
      ptx::mbar_arrive_expect_tx(&wfull[stage], C::kStageBytes);
      if constexpr (FWD) {
        ptx::tma_load_2d(dst, &maps.w[l], &wfull[stage], n0, kb * BK);
        ptx::tma_load_2d(dst + BK * 128, &maps.w[l], &wfull[stage], n0 + 64, kb * BK);
        ptx::tma_load_2d(dst + C::kWBytes, &maps.w_lo[l], &wfull[stage], n0, kb * BK);
        ptx::tma_load_2d(dst + C::kWBytes + BK * 128, &maps.w_lo[l], &wfull[stage], n0 + 64, kb * BK);
      } else {
        ptx::tma_load_2d(dst, &maps.w[l], &wfull[stage], kb * BK, n0);
        ptx::tma_load_2d(dst + C::kWBytes, &maps.w_lo[l], &wfull[stage], kb * BK, n0);
      }
      const int s = stage;
      if (++stage == S) { stage = 0; phase ^= 1; }
      return s;
    };
    auto load_alo = [&](int l, int kb, int s) {
      const CUtensorMap* src = l == 0 ? &maps.in_lo : &maps.out_lo[l - 1];
      ptx::tma_load_2d(sRing + s * C::kStageBytes + 2 * C::kWBytes, src, &wfull[s], kb * BK, m0);
    };
    if (lane == 0) {
      ptx::tma_prefetch_desc(&maps.in);
      ptx::tma_prefetch_desc(&maps.in_lo);
      const int nkb0 = (args.K[0] + BK - 1) / BK;
      ptx::mbar_arrive_expect_tx(act_full, nkb0 * C::kTile);
      for (int kb = int(q); kb < nkb0; kb += C::kCluster)
        ptx::tma_load_2d_mc(sAct + kb * C::kTile, &maps.in, act_full, kb * BK, m0, kAll);
    }
    for (int l = 0; l < L; ++l) {
      const int nkb = (args.K[l] + BK - 1) / BK;
      if (lane == 0) {
        if (l > 0) {
          // every CTA's lo slice of layer l-1 is in global memory: stream the A_lo blocks
          mbar_wait_cluster(lo_ready, uint32_t(l - 1) & 1u);
          fence_proxy_async_global();
        }
        for (int i = 0; i < pend_n; ++i) load_alo(l, i, pend_stage[i]);
        for (int kb = pend_n; kb < nkb; ++kb) load_alo(l, kb, load_w(l, kb));
      }
      pend_n = 0;
      if (l + 1 < L) {
        __syncwarp();
        cl_arrive();
        if (lane == 0) {  // prefetch the next layer's first weight blocks while the exchange runs
          const int nn = (args.K[l + 1] + BK - 1) / BK;
          pend_n = nn < S ? nn : S;
          for (int kb = 0; kb < pend_n; ++kb) pend_stage[kb] = load_w(l + 1, kb);
        }
        pend_n = __shfl_sync(0xffffffffu, pend_n, 0);
#pragma unroll
        for (int i = 0; i < S; ++i) pend_stage[i] = __shfl_sync(0xffffffffu, pend_stage[i], 0);
        bar_sync(1, 160);  // this CTA's hi slice is in its own activation tile and fenced
        if (lane == 0) {
          tma_store_2d(&maps.out[l], sAct + (2 * q) * C::kTile, n0, m0);
          tma_store_2d(&maps.out[l], sAct + (2 * q + 1) * C::kTile, n0 + 64, m0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // slice is in global (L2)
          ptx::mbar_arrive(slice_free);
        }
        __syncwarp();
        cl_wait();  // every CTA's MMAs of layer l are done: activation tiles are free
        if (lane == 0) {
          constexpr uint32_t kSlice = 2 * C::kTile;
          const uint16_t peers = uint16_t(kAll & ~(1u << q));
          ptx::mbar_arrive_expect_tx(act_full, (C::kCluster - 1) * kSlice);  // the 3 peer slices
          ptx::tma_load_2d_mc(sAct + (2 * q) * C::kTile, &maps.out[l], act_full, n0, m0, peers);
          ptx::tma_load_2d_mc(sAct + (2 * q + 1) * C::kTile, &maps.out[l], act_full, n0 + 64, m0, peers);
        }
        __syncwarp();
      } else if (args.out[l] != nullptr) {  // last layer: coalesced TMA store of the hi output slice
        bar_sync(1, 160);
        if (lane == 0) {
          tma_store_2d(&maps.out[l], sAct + (2 * q) * C::kTile, n0, m0);
          tma_store_2d(&maps.out[l], sAct + (2 * q + 1) * C::kTile, n0 + 64, m0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
        __syncwarp();
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    for (int l = 0; l < L; ++l) {
      if (lane == 0) {
        ptx::mbar_wait(act_full, uint32_t(l) & 1u);
        ptx::tc_fence_after();
        const int nkb = (args.K[l] + BK - 1) / BK;
        const uint32_t a0 = ptx::smem_u32(sAct), r0 = ptx::smem_u32(sRing);
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait(&wfull[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sb = r0 + stage * C::kStageBytes, sbl = sb + C::kWBytes, sal = sb + 2 * C::kWBytes;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ah = ptx::sw128_desc(a0 + kb * C::kTile + kk * 32, 16, 1024);
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
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(acc_full);
      }
      __syncwarp();
      if (l + 1 < L) {
        cl_arrive();
        cl_wait();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps 0-3
    const int row = int(warp) * 32 + int(lane);
    const int m = m0 + row;
    const bool row_ok = m < args.M;
    const uint32_t t_row = tmem + ((warp * 32u) << 16);
    for (int l = 0; l < L; ++l) {
      const bool last = l + 1 == L;
      uint4 mk[BN / 32][4];
      if constexpr (!FWD) {
        if (row_ok) {
          const uint4* src = reinterpret_cast<const uint4*>(args.mask[l] + (long long)m * args.ldm[l] + n0);
#pragma unroll
          for (int c = 0; c < BN / 32; ++c)
#pragma unroll
            for (int v = 0; v < 4; ++v) mk[c][v] = __ldg(src + c * 4 + v);
        }
      }
      ptx::mbar_wait(acc_full, uint32_t(l) & 1u);
      ptx::tc_fence_after();
      if (!last) cl_arrive();
      const bool store = !last || args.out[l] != nullptr;
      if (store && l >= 1) ptx::mbar_wait(slice_free, uint32_t(l - 1) & 1u);
      __nv_bfloat16* lo_row = (store && row_ok) ? args.out_lo[l] + (long long)m * args.ldo[l] + n0 : nullptr;
      float hp = 0.f, hp2 = 0.f;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
        ptx::tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if constexpr (FWD) {
          const float* bias = args.bias[l] ? args.bias[l] + n0 + c * 32 : nullptr;
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j] + (bias ? __ldg(bias + j) : 0.f), 0.f);
          if (last) {
            if (args.head_w != nullptr) {
#pragma unroll
              for (int j = 0; j < 32; ++j) hp = fmaf(v[j], __ldg(args.head_w + n0 + c * 32 + j), hp);
            }
            if (args.head_u != nullptr) {
#pragma unroll
              for (int j = 0; j < 32; ++j) hp2 = fmaf(v[j], __ldg(args.head_u + n0 + c * 32 + j), hp2);
            }
          }
        } else {
          uint4 cur[4];
#pragma unroll
          for (int cc = 0; cc < BN / 32; ++cc)
            if (cc == c)
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) cur[q4] = mk[cc][q4];
          const __nv_bfloat16* mv = reinterpret_cast<const __nv_bfloat16*>(cur);
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
            const int col = n0 + c * 32 + j;
            const int chunk = ((col & 63) >> 3) ^ (row & 7);
            *reinterpret_cast<uint4*>(sAct + (col >> 6) * C::kTile + row * 128 + chunk * 16) = ph;
            if (lo_row != nullptr) *reinterpret_cast<uint4*>(lo_row + c * 32 + j) = pl;
          }
        }
      }
      if (FWD && last && row_ok) {
        if (args.head_part != nullptr) args.head_part[(long long)q * args.head_ld + m] = hp;
        if (args.head_part2 != nullptr) args.head_part2[(long long)q * args.head_ld + m] = hp2;
      }
      if (store) {
        ptx::tc_fence_before();
        fence_proxy_async_smem();  // generic st.shared -> async-proxy readers (TMA store, tensor core)
        bar_arrive(1, 160);
      }
      if (!last) {
        // lo slice -> every CTA's lo_ready: generic global stores made visible to the async proxy
        // (the peers' TMA loads), then one release arrive per CTA of the cluster
        fence_proxy_async_global();
        bar_sync(2, 128);
        if (threadIdx.x == 0) {
          const uint32_t local = ptx::smem_u32(lo_ready);
#pragma unroll
          for (uint32_t p = 0; p < uint32_t(C::kCluster); ++p) mbar_arrive_cluster(mapa(local, p));
        }
        cl_wait();
      }
    }
    ptx::pdl_launch_dependents();
  }

  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();  // no CTA leaves while a multicast / remote arrive into it could still be in flight
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<BN>(tmem);
  }
}

}  // namespace moses
