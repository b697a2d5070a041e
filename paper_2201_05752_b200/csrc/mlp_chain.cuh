// mlp_chain.cuh — the whole hidden-layer chain of one 128-row block in ONE kernel (bf16).
//
// The cost-model step at batch 512 programs (~2.3K statement rows) is latency-bound: every
// per-layer GEMM launch pays ~5 us of fixed cost (launch, prologue, first TMA round trip,
// teardown) for ~1 us of tensor work (tools/gemm_latency.py). Rows are independent through the
// forward pass (and through the dZ chain of the backward pass), so a 4-CTA cluster owns a
// 128-row block for ALL layers:
//
//   CTA q of the cluster computes output columns [128q, 128q+128) of every layer;
//   the layer's full 128 x 512 bf16 activation tile (the next layer's A operand, 8 SW128
//   K-blocks = 128 KB) lives in shared memory of every CTA;
//   after a layer, CTA q's epilogue writes its 128 x 128 slice straight into its OWN activation
//   tile (swizzled st.shared; its MMAs of the layer are complete); the producer TMA-stores the
//   two K-blocks to global (coalesced; the backward pass needs them anyway) and, once the store
//   has landed, TMA-MULTICASTS them from L2 into the 3 peer tiles. (Pushing the 96 KB per CTA
//   through DSMEM instead is bound by its ~18 B/clk ports: measured 2.8 us vs 1.3 us per layer.)
//   weights (16 KB per K-block) stream through a 4-stage TMA ring that prefetches the next
//   layer while the exchange runs.
//
// Two instances:
//   FWD:  out_l = relu(A_l W_l + b_l), W_l MN-major [K][512]; last layer: per-slice head dots
//         (head_part[q][row], fixed-order partials as the per-layer kernels) — identical math
//         and MMA order to umma_gemm_cluster, so the results are bitwise equal.
//   DGRAD: dz_l = (dz_{l+1} W_l^T) * [act_l > 0], W_l K-major [512][512].
//
// Cluster barrier protocol per exchange (every thread arrives/waits once per exchange):
//   arrive#  epilogue: after the layer's accumulator is complete (=> this CTA's MMAs no longer
//            read the activation tile); producer/MMA warps: after issuing the layer
//   wait#    producer: before multicasting into the other CTAs' tiles.
// TMEM: one 128-column fp32 accumulator; the next layer's MMAs start only after the exchange,
// which follows the epilogue's TMEM reads.
#pragma once
#include "gemm.cuh"

namespace moses {

constexpr int kChainMaxLayers = 8;

struct ChainMaps {
  CUtensorMap in;                        // chain input [M][K0] (x0 or dz_last), box {64, 128}
  CUtensorMap w[kChainMaxLayers];        // FWD: [K][512] box {64, 64}; DGRAD: [512 n][512 k] box {64, 128}
  CUtensorMap out[kChainMaxLayers];      // outputs [M][512] box {64, 128}: TMA store + multicast reload
};

struct ChainArgs {
  int M;
  int n_layers;
  int K[kChainMaxLayers];
  const float* bias[kChainMaxLayers];    // FWD
  __nv_bfloat16* out[kChainMaxLayers];
  long long ldo[kChainMaxLayers];
  const __nv_bfloat16* mask[kChainMaxLayers];  // DGRAD: relu' source (act_l)
  long long ldm[kChainMaxLayers];
  const float* head_w;  // FWD last layer
  const float* head_u;
  float* head_part;
  float* head_part2;
  long long head_ld;
  unsigned long long* trace;  // optional phase timestamps of cluster 0 (tools/chain_trace.py)
  __nv_bfloat16* out_lo[kChainMaxLayers];  // split chain: lo planes of the outputs (row stride ldo)
};

struct ChainCfg {
  static constexpr int BM = 128, BN = 128, BK = 64, kWidth = 512, kCluster = 4;
  static constexpr int kTile = BM * 128;                // one 64-col K-block of a 128-row bf16 tile
  static constexpr int kActBytes = (kWidth / BK) * kTile;  // 128 KB
  static constexpr int kStages = 5;
  static constexpr int kWBytes = BN * 128;              // one K-block of the weight slice (16 KB)
  static constexpr int kSmemBytes = kActBytes + kStages * kWBytes + 1024 + 256 + kChainMaxLayers * BN * 4;
};

namespace chain_detail {
// relaxed: the barrier only orders tensor-core reads (signalled through mbarriers) against the
// peers' later bulk copies; a .release arrive would emit a GPU-scope MEMBAR behind the epilogue's
// global stores.
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory"); }
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// async bulk copy own smem -> a peer CTA's smem, completing on the peer's mbarrier
__device__ __forceinline__ void bulk_to_peer(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t mbar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src), "r"(bytes), "r"(mbar_cluster)
               : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire;" ::: "memory"); }
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// trace slots: [q][layer][event]; events: 0 mma start, 1 mma issued, 2 acc seen, 3 stores fenced,
// 4 cluster wait passed (producer), 5 multicast issued, 6 kernel start, 7 kernel end
#define CHAIN_TRACE(ev, l)                                                                             \
  do {                                                                                                 \
    if (args.trace != nullptr && blockIdx.x < 4)                                                       \
      args.trace[(q * kChainMaxLayers + (l)) * 8 + (ev)] = chain_detail::clk();                        \
  } while (0)
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
}  // namespace chain_detail

template <bool FWD>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(192, 1)
    mlp_chain_kernel(const __grid_constant__ ChainMaps maps, const __grid_constant__ ChainArgs args) {
  using namespace chain_detail;
  using C = ChainCfg;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, S = C::kStages;
  constexpr uint32_t kIdesc = ptx::umma_idesc(1 /*BF16*/, false, FWD /*B MN-major*/, BM, BN);
  constexpr uint16_t kAll = 0xF;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sAct = smem;
  uint8_t* sW = smem + C::kActBytes;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(sW + S * C::kWBytes);
  uint64_t* wempty = wfull + S;
  uint64_t* act_full = wempty + S;
  uint64_t* acc_full = act_full + 1;
  uint64_t* slice_free = acc_full + 1;  // this CTA's outgoing bulk copies finished reading its slice
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(slice_free + 1);
  float* s_bias = reinterpret_cast<float*>(sW + S * C::kWBytes + 256);

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
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<BN>(tmem_slot);
  ptx::pdl_wait();  // every global read below may depend on the previous kernel
  if (threadIdx.x == 0) CHAIN_TRACE(6, 0);
  if constexpr (FWD) {
    for (int i = threadIdx.x; i < L * BN; i += blockDim.x) {
      const int l = i / BN, j = i - l * BN;
      s_bias[i] = args.bias[l] ? __ldg(args.bias[l] + n0 + j) : 0.f;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();      // CTA-level order of the inits / parameter slices (what compute-sanitizer tracks)
  ptx::cluster_sync();  // barrier inits + TMEM address visible cluster-wide before any multicast
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    int issued_next = 0;  // weight K-blocks of layer l already issued as prefetch
    auto load_w = [&](int l, int kb) {
      ptx::mbar_wait(&wempty[stage], phase ^ 1);
      uint8_t* dst = sW + stage * C::kWBytes;
      ptx::mbar_arrive_expect_tx(&wfull[stage], C::kWBytes);
      if constexpr (FWD) {
        ptx::tma_load_2d(dst, &maps.w[l], &wfull[stage], n0, kb * BK);
        ptx::tma_load_2d(dst + BK * 128, &maps.w[l], &wfull[stage], n0 + 64, kb * BK);
      } else {
        ptx::tma_load_2d(dst, &maps.w[l], &wfull[stage], kb * BK, n0);
      }
      if (++stage == S) { stage = 0; phase ^= 1; }
    };
    if (lane == 0) {
      ptx::tma_prefetch_desc(&maps.in);
      const int nkb0 = (args.K[0] + BK - 1) / BK;
      ptx::mbar_arrive_expect_tx(act_full, nkb0 * C::kTile);
      for (int kb = int(q); kb < nkb0; kb += C::kCluster)
        ptx::tma_load_2d_mc(sAct + kb * C::kTile, &maps.in, act_full, kb * BK, m0, kAll);
    }
    for (int l = 0; l < L; ++l) {
      const int nkb = (args.K[l] + BK - 1) / BK;
      if (lane == 0)
        for (int kb = issued_next; kb < nkb; ++kb) load_w(l, kb);
      issued_next = 0;
      if (l + 1 < L) {
        __syncwarp();
        cl_arrive();
        if (lane == 0) {  // prefetch the next layer's first weight blocks while the exchange runs
          const int nn = (args.K[l + 1] + BK - 1) / BK;
          issued_next = nn < S ? nn : S;
          for (int kb = 0; kb < issued_next; ++kb) load_w(l + 1, kb);
        }
        issued_next = __shfl_sync(0xffffffffu, issued_next, 0);
        bar_sync(1, 160);  // this CTA's slice is in its own activation tile and fenced
        if (lane == 0) {
          CHAIN_TRACE(5, l);
          tma_store_2d(&maps.out[l], sAct + (2 * q) * C::kTile, n0, m0);
          tma_store_2d(&maps.out[l], sAct + (2 * q + 1) * C::kTile, n0 + 64, m0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // slice is in global (L2)
          ptx::mbar_arrive(slice_free);
        }
        __syncwarp();
        cl_wait();  // every CTA's MMAs of layer l are done: activation tiles are free
        if (lane == 0) {
          CHAIN_TRACE(4, l);
          constexpr uint32_t kSlice = 2 * C::kTile;
          const uint16_t peers = uint16_t(kAll & ~(1u << q));
          ptx::mbar_arrive_expect_tx(act_full, (C::kCluster - 1) * kSlice);  // the 3 peer slices
          ptx::tma_load_2d_mc(sAct + (2 * q) * C::kTile, &maps.out[l], act_full, n0, m0, peers);
          ptx::tma_load_2d_mc(sAct + (2 * q + 1) * C::kTile, &maps.out[l], act_full, n0 + 64, m0, peers);
        }
        __syncwarp();
      } else if (args.out[l] != nullptr) {  // last layer: coalesced TMA store of the output slice
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
        CHAIN_TRACE(0, l);
        const int nkb = (args.K[l] + BK - 1) / BK;
        const uint32_t a0 = ptx::smem_u32(sAct), w0 = ptx::smem_u32(sW);
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait(&wfull[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sb = w0 + stage * C::kWBytes;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = ptx::sw128_desc(a0 + kb * C::kTile + kk * 32, 16, 1024);
            const uint64_t bd = FWD ? ptx::sw128_desc(sb + kk * 2048, BK * 128, 1024, 2)
                                    : ptx::sw128_desc(sb + kk * 32, 16, 1024);
            ptx::umma_f16(tmem, ad, bd, kIdesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::umma_commit(&wempty[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(acc_full);
        CHAIN_TRACE(1, l);
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
      uint4 mk[BN / 32][4];  // DGRAD: relu' source of all four 32-column chunks, loaded before the
                             // accumulator wait so the L2 latency hides behind the layer's MMAs
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
      if (threadIdx.x == 0) CHAIN_TRACE(2, l);
      if (!last) cl_arrive();
      const bool store = !last || args.out[l] != nullptr;  // slice goes through the own tile
      if (store && l >= 1) ptx::mbar_wait(slice_free, uint32_t(l - 1) & 1u);
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
          const float* sb = s_bias + l * BN + c * 32;
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j] + sb[j], 0.f);
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
          for (int cc = 0; cc < BN / 32; ++cc)  // static register indexing of the chunk
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
            uint4 pk;
            __nv_bfloat162 p0 = __floats2bfloat162_rn(v[j], v[j + 1]);
            __nv_bfloat162 p1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
            __nv_bfloat162 p2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]);
            __nv_bfloat162 p3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
            pk.x = *reinterpret_cast<uint32_t*>(&p0);
            pk.y = *reinterpret_cast<uint32_t*>(&p1);
            pk.z = *reinterpret_cast<uint32_t*>(&p2);
            pk.w = *reinterpret_cast<uint32_t*>(&p3);
            // own activation tile (next layer's A operand / TMA-store source): SW128 K-major,
            // 16-byte chunk (col%64)/8 ^ (row%8)
            const int col = n0 + c * 32 + j;
            const int chunk = ((col & 63) >> 3) ^ (row & 7);
            *reinterpret_cast<uint4*>(sAct + (col >> 6) * C::kTile + row * 128 + chunk * 16) = pk;
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
        if (threadIdx.x == 0) CHAIN_TRACE(3, l);
        bar_arrive(1, 160);
      }
      if (!last) cl_wait();
    }
    if (threadIdx.x == 0) CHAIN_TRACE(7, 0);
    ptx::pdl_launch_dependents();
  }

  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();  // no CTA leaves while a multicast into it could still be in flight
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<BN>(tmem);
  }
}

}  // namespace moses
