// gemm.cuh — tcgen05 (UMMA) GEMM for the cost-model MLP on sm_100a.
//
//   C[m][n] = sum_k A(m,k) * B(n,k)        BM = 128 rows per CTA, BN in {64,128,256}
//
// One CTA = one 128 x BN output tile; K is streamed through a STAGES-deep ring
// of 128-byte-swizzled shared-memory tiles filled by TMA (warp 0, one lane),
// consumed by tcgen05.mma issued from a single thread (warp 1), accumulated in
// TMEM (BN fp32 columns x 128 lanes). All four warps then drain TMEM with
// tcgen05.ld (one output row per thread) through a fused epilogue:
//
//   Epi::Fwd      H = act(acc + bias) stored as the next layer's operand, plus
//                 optional per-row dot products with the head vector(s) (the
//                 scalar output layer and the discriminator logit folded in,
//                 written as per-N-tile partials so the sum stays deterministic).
//   Epi::Dgrad    dZ_prev = acc * [H_prev > 0]   (ReLU' from the stored activation)
//   Epi::StoreF32 fp32 store (weight+bias gradients in the reference flat layout)
//
// Operands may be K-major or MN-major (the flat parameter block [in][out]
// is MN-major for the forward pass and K-major for the data-gradient pass;
// the wgrad pass reads both activations MN-major), selected per template.
// T = __nv_bfloat16 (kind::f16) or float (kind::tf32).
#pragma once
#include <cuda_bf16.h>

#include "ptx.cuh"

namespace moses {

enum class Epi : int { Fwd = 0, Dgrad = 1, StoreF32 = 2 };

struct GemmArgs {
  int M, N, K;
  void* out;            // T* (Fwd, Dgrad) or float* (StoreF32)
  long long ldo;        // output row stride (elements)
  const float* bias;    // Fwd: [N] or null
  int relu;             // Fwd
  const float* head_w;  // Fwd: optional [N] -> head_part[tile_n * head_ld + m]
  const float* head_u;  // Fwd: optional [N] -> head_part2[...]
  float* head_part;
  float* head_part2;
  long long head_ld;
  const void* mask;     // Dgrad: T*, ReLU' source H_prev[m * ldm + n]
  long long ldm;
  int mn_layout;        // descriptor layout type for MN-major operands (2 = SW128, 1 = SW128_BASE32B)
  int mn_sbo;           // SBO bytes for MN-major operands
  int mn_kstep;         // bytes advanced per MMA K step for MN-major operands
  int round_out;        // fp32 Fwd/Dgrad outputs rounded to tf32 (next GEMM operand)
  void* out_lo;         // 3xTF32 (gemm_split.cuh): low half of the Fwd/Dgrad output
  int kperm;            // umma_fwd_pair_split: K-blocks in the fused chain's order (chain_korder)
};

__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

template <typename T>
struct UmmaType;
template <>
struct UmmaType<__nv_bfloat16> {
  static constexpr uint32_t kFormat = 1;  // BF16
  static constexpr int kUmmaK = 16;
};
template <>
struct UmmaType<float> {
  static constexpr uint32_t kFormat = 2;  // TF32
  static constexpr int kUmmaK = 8;
};

template <typename T, int BN>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 128 / int(sizeof(T));  // one 128-byte swizzle row of K
  static constexpr int kABytes = BM * 128;         // 16 KB
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (200 * 1024 / kStageBytes) > 6 ? 6 : (200 * 1024 / kStageBytes);
  static constexpr int kMNChunk = 128 / int(sizeof(T));  // elements per 128-byte MN row
  static constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  static constexpr int kVecBytes = 3 * BN * 4;  // bias / head_w / head_u slices of this CTA's N range
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/ + kVecBytes;
};

template <typename T, int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(128, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmArgs args) {
  using Cfg = GemmCfg<T, BN>;
  constexpr int BM = Cfg::BM, BK = Cfg::BK, STAGES = Cfg::kStages;
  constexpr int UK = UmmaType<T>::kUmmaK;
  constexpr uint32_t kIdesc = ptx::umma_idesc(UmmaType<T>::kFormat, A_MN, B_MN, BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* accum_bar = empty_bar + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_bar + 1);
  float* s_bias = reinterpret_cast<float*>(smem + STAGES * Cfg::kStageBytes + 256);
  float* s_hw = s_bias + BN;
  float* s_hu = s_hw + BN;

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int num_kb = (args.K + BK - 1) / BK;
  ptx::pdl_launch_dependents();

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    ptx::mbar_init(accum_bar, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  // everything above overlaps the previous kernel's tail (PDL); operands/params are read below
  ptx::pdl_wait();
  if constexpr (EPI == int(Epi::Fwd)) {
    for (int j = threadIdx.x; j < BN; j += 128) {
      const int n = n0 + j;
      const bool ok = n < args.N;
      s_bias[j] = (ok && args.bias) ? __ldg(args.bias + n) : 0.f;
      s_hw[j] = (ok && args.head_w) ? __ldg(args.head_w + n) : 0.f;
      s_hu[j] = (ok && args.head_u) ? __ldg(args.head_u + n) : 0.f;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
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
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (single thread)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
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
          const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
          if constexpr (sizeof(T) == 2) ptx::umma_f16(tmem_base, ad, bd, kIdesc, acc);
          else ptx::umma_tf32(tmem_base, ad, bd, kIdesc, acc);
        }
        ptx::umma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs retire
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      ptx::umma_commit(accum_bar);  // accumulator complete
    }
    __syncwarp();
  }

  // ---------------- epilogue: all 4 warps, one accumulator row per thread
  const int row = warp * 32 + lane;
  const int m = m0 + row;
  const bool row_ok = m < args.M;
  const uint32_t t_row = tmem_base + ((warp * 32u) << 16);
  float hp = 0.f, hp2 = 0.f;
  // ReLU' source for the Dgrad epilogue: 16-byte vector loads, chunk 0 prefetched while the MMAs run
  constexpr int kMaskVec = 32 * int(sizeof(T)) / 16;
  uint4 mk[kMaskVec];
  auto load_mask = [&](int c) {
    if constexpr (EPI == int(Epi::Dgrad)) {
      const int nb = n0 + c * 32;
      if (row_ok && nb + 32 <= args.N) {
        const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(args.mask) + (long long)m * args.ldm + nb);
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
  ptx::mbar_wait(accum_bar, 0);
  ptx::tc_fence_after();

#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
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
      const float* sb = s_bias + c * 32;
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += sb[j];
      if (args.relu) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
      }
      if (args.head_w != nullptr) {
        const float* hw = s_hw + c * 32;
#pragma unroll
        for (int j = 0; j < 32; ++j) hp = fmaf(v[j], hw[j], hp);
      }
      if (args.head_u != nullptr) {
        const float* hu = s_hu + c * 32;
#pragma unroll
        for (int j = 0; j < 32; ++j) hp2 = fmaf(v[j], hu[j], hp2);
      }
    }

    if constexpr (EPI == int(Epi::StoreF32)) {
      float* orow = reinterpret_cast<float*>(args.out) + (long long)m * args.ldo + nb;
      if (nvalid == 32 && (args.ldo % 4) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(orow + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
        #pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nvalid) orow[j] = v[j];
      }
    } else {
      T* orow = reinterpret_cast<T*>(args.out) + (long long)m * args.ldo + nb;
      if (args.out == nullptr) continue;
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
          for (int j = 0; j < 32; ++j) v[j] = tf32_round(v[j]);  // next layer's kind::tf32 operand
        }
        if (nvalid == 32) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(orow + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
          #pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nvalid) orow[j] = v[j];
        }
      }
    }
  }
  if constexpr (EPI == int(Epi::Fwd)) {
    if (row_ok && args.head_part != nullptr) args.head_part[(long long)blockIdx.y * args.head_ld + m] = hp;
    if (row_ok && args.head_part2 != nullptr) args.head_part2[(long long)blockIdx.y * args.head_ld + m] = hp2;
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

}  // namespace moses
