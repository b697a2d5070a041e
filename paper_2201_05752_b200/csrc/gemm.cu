// gemm.cu — host side of the tcgen05 GEMM: TMA descriptor encoding (driver
// entry point fetched through the runtime, so the library needs no -lcuda),
// N-tile selection for the 148-SM grid, and the template instantiations.
#include <mutex>
#include <unordered_map>
#include <type_traits>

#include "common.cuh"
#include "gemm.cuh"
#include "gemm_persistent.cuh"
#include "gemm_fwd.cuh"
#include "gemm_fwd2.cuh"
#include "gemm_gram.cuh"
#include "gemm_cluster.cuh"
#include "gemm_split.cuh"
#include "mlp_chain.cuh"
#include "mlp_chain_split.cuh"
#include "gemm_group.cuh"
#include "gemm_wgrad_sk.cuh"

namespace moses {
// MN-major operand encoding (index 0 = bf16, 1 = tf32). 16-bit operands use the plain 128-byte
// swizzle (8 K-rows per 1024-B atom). 32-bit MN-major operands need the 32-byte-atom variant: TMA
// SWIZZLE_128B_ATOM_32B on the load side and descriptor layout SWIZZLE_128B_BASE32B (type 1) with
// 4-row (512-B) K atoms on the MMA side — the plain 128-B swizzle makes kind::tf32 read zeros
// (measured on B200, tools/debug_tf32mn.py).
int g_mn_swz[2] = {int(CU_TENSOR_MAP_SWIZZLE_128B), int(CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)};
int g_mn_layout[2] = {2, 1};
int g_mn_sbo[2] = {1024, 512};
int g_mn_kstep[2] = {16 * 128, 8 * 128};
extern int g_num_sms;
extern int g_cluster;
extern unsigned long long* g_chain_trace;
namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) fail(MOSES_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D tiled map over a row-major matrix: `inner` contiguous elements per row,
// `outer` rows, row stride `ld` elements; box = box_inner x box_outer, 128-B swizzle.
// Encoded maps are memoised per host thread: a map is a pure function of its arguments, and an eager
// call (gradients, the Moses step, predict) encodes tens of them on the host before its first launch.
struct MapKey {
  const void* base;
  long long inner, outer, ld;
  int elem, box_inner, box_outer, swz;
  bool operator==(const MapKey& o) const {
    return base == o.base && inner == o.inner && outer == o.outer && ld == o.ld && elem == o.elem &&
           box_inner == o.box_inner && box_outer == o.box_outer && swz == o.swz;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    uint64_t h = reinterpret_cast<uintptr_t>(k.base) * 0x9e3779b97f4a7c15ull;
    for (long long v : {k.inner, k.outer, k.ld, (long long)k.elem, (long long)k.box_inner, (long long)k.box_outer,
                        (long long)k.swz})
      h = (h ^ uint64_t(v)) * 0x100000001b3ull;
    return size_t(h ^ (h >> 29));
  }
};
CUtensorMap encode_map(const void* base, int elem, long long inner, long long outer, long long ld, int box_inner,
                       int box_outer, CUtensorMapSwizzle swz);
CUtensorMap make_map(const void* base, int elem, long long inner, long long outer, long long ld, int box_inner,
                     int box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  const MapKey key{base, inner, outer, ld, elem, box_inner, box_outer, int(swz)};
  const auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() >= 4096) cache.clear();  // bounded: callers passing ever-new buffers
  const CUtensorMap m = encode_map(base, elem, inner, outer, ld, box_inner, box_outer, swz);
  cache.emplace(key, m);
  return m;
}
CUtensorMap encode_map(const void* base, int elem, long long inner, long long outer, long long ld, int box_inner,
                       int box_outer, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * elem};
  const cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_outer)};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * elem) & 15))
    fail(MOSES_ERR_INVALID_ARG, "TMA operand must be 16-byte aligned with a 16-byte row stride");
  const CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(MOSES_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

// operand map: rows of the GEMM dimension `mn` (size MN), K along the other axis
CUtensorMap operand_map(const Operand& o, int elem, long long MN, long long K, int tile_mn) {
  const int chunk = 128 / elem;  // elements in one 128-B swizzle row
  if (o.mn_major)
    return make_map(o.ptr, elem, MN, K, o.ld, chunk, chunk /* BK */, CUtensorMapSwizzle(g_mn_swz[elem == 4]));
  return make_map(o.ptr, elem, K, MN, o.ld, chunk, tile_mn);
}

template <typename T, int BN, bool AMN, bool BMN, int EPI>
void launch_t(const GemmCall& c, cudaStream_t s) {
  using Cfg = GemmCfg<T, BN>;
  auto kern = umma_gemm_kernel<T, BN, AMN, BMN, EPI>;
  static bool configured = false;
  if (!configured) {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
    configured = true;
  }
  constexpr int elem = sizeof(T);
  const CUtensorMap ta = operand_map(c.A, elem, c.M, c.K, Cfg::BM);
  const CUtensorMap tb = operand_map(c.B, elem, c.N, c.K, BN);
  GemmArgs a{};
  a.M = c.M;
  a.N = c.N;
  a.K = c.K;
  a.out = c.out;
  a.ldo = c.ldo;
  a.bias = c.bias;
  a.relu = c.relu;
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.mask = c.mask;
  a.ldm = c.ldm;
  a.mn_layout = g_mn_layout[elem == 4];
  a.mn_sbo = g_mn_sbo[elem == 4];
  a.mn_kstep = g_mn_kstep[elem == 4];
  a.round_out = c.round_out;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ceil_div(c.M, Cfg::BM), ceil_div(c.N, BN));
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: prologue overlaps the previous kernel
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, a));
}

template <typename T, int BN, bool AMN, bool BMN, int EPI>
void launch_p(const GemmCall& c, cudaStream_t s) {
  using Cfg = PCfg<T, BN>;
  auto kern = umma_gemm_persistent<T, BN, AMN, BMN, EPI>;
  static bool configured = false;
  if (!configured) {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
    configured = true;
  }
  constexpr int elem = sizeof(T);
  const CUtensorMap ta = operand_map(c.A, elem, c.M, c.K, Cfg::BM);
  const CUtensorMap tb = operand_map(c.B, elem, c.N, c.K, BN);
  GemmArgs a{};
  a.M = c.M;
  a.N = c.N;
  a.K = c.K;
  a.out = c.out;
  a.ldo = c.ldo;
  a.bias = c.bias;
  a.relu = c.relu;
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.mask = c.mask;
  a.ldm = c.ldm;
  a.mn_layout = g_mn_layout[elem == 4];
  a.mn_sbo = g_mn_sbo[elem == 4];
  a.mn_kstep = g_mn_kstep[elem == 4];
  a.round_out = c.round_out;
  const int tm = ceil_div(c.M, Cfg::BM), tn = ceil_div(c.N, BN);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(tm * tn, g_num_sms));
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, a, tm, tn));
}

// scoring-shape forward layer (gemm_fwd.cuh): bf16, A K-major, TMA-stored activations
template <int BN, bool BMN>
void launch_f(const GemmCall& c, cudaStream_t s) {
  using Cfg = FCfg<BN>;
  auto kern = umma_fwd_persistent<BN, BMN>;
  static std::once_flag once;
  std::call_once(once, [&] {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
  });
  const CUtensorMap ta = operand_map(c.A, 2, c.M, c.K, Cfg::BM);
  const CUtensorMap tb = operand_map(c.B, 2, c.N, c.K, BN);
  // output boxes of 32 rows x 64 columns; the map's extent (N x M) clips ragged edges, so the
  // activation buffer's constant-1 column at index N is never touched
  const CUtensorMap tc = c.out ? make_map(c.out, 2, c.N, c.M, c.ldo, 64, 32) : ta;
  GemmArgs a{};
  a.M = c.M;
  a.N = c.N;
  a.K = c.K;
  a.out = c.out;
  a.ldo = c.ldo;
  a.bias = c.bias;
  a.relu = c.relu;
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.mn_layout = g_mn_layout[0];
  a.mn_sbo = g_mn_sbo[0];
  a.mn_kstep = g_mn_kstep[0];
  const int tm = ceil_div(c.M, Cfg::BM), tn = ceil_div(c.N, BN);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(tm * tn, g_num_sms));
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, a, tm, tn));
}

// scoring hidden layers, N = 512: weight-resident CTA pairs (gemm_fwd2.cuh)
void launch_pair(const GemmCall& c, cudaStream_t s) {
  using Cfg = PairCfg;
  auto kern = umma_fwd_pair;
  static std::once_flag once;
  std::call_once(once, [&] {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
  });
  const CUtensorMap ta = operand_map(c.A, 2, c.M, c.K, Cfg::BM);
  const CUtensorMap tb = operand_map(c.B, 2, c.N, c.K, 64);
  const CUtensorMap tc = c.out ? make_map(c.out, 2, c.N, c.M, c.ldo, 64, 32) : ta;
  GemmArgs a{};
  a.M = c.M;
  a.N = c.N;
  a.K = c.K;
  a.out = c.out;
  a.ldo = c.ldo;
  a.bias = c.bias;
  a.relu = c.relu;
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.mn_layout = g_mn_layout[0];
  a.mn_sbo = g_mn_sbo[0];
  a.mn_kstep = g_mn_kstep[0];
  const int tiles_m2 = ceil_div(c.M, 2 * Cfg::BM);
  int pairs = std::min(g_num_sms / 2, 2 * tiles_m2);
  pairs -= pairs & 1;  // both n-halves get the same number of pairs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, a, tiles_m2));
}

// split-bf16 scoring layers, N % 128 == 0, K <= 512 (gemm_fwd2.cuh umma_fwd_pair_split)
void launch_pair_split(const GemmCall& c, cudaStream_t s) {
  using Cfg = PairSplitCfg;
  auto kern = umma_fwd_pair_split;
  static std::once_flag once;
  std::call_once(once, [&] {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
  });
  if (c.out != nullptr && c.out_lo == nullptr) fail(MOSES_ERR_INVALID_ARG, "split pair layer output without a lo plane");
  const Operand alo{c.A.lo, c.A.ld, c.A.mn_major}, blo{c.B.lo, c.B.ld, c.B.mn_major};
  // activations: 32-column K-blocks with 64-byte rows (SWIZZLE_64B), see PairSplitCfg
  const CUtensorMap ta = make_map(c.A.ptr, 2, c.K, c.M, c.A.ld, Cfg::BKA, Cfg::BM, CU_TENSOR_MAP_SWIZZLE_64B);
  const CUtensorMap ta_lo = make_map(alo.ptr, 2, c.K, c.M, c.A.ld, Cfg::BKA, Cfg::BM, CU_TENSOR_MAP_SWIZZLE_64B);
  const CUtensorMap tb = operand_map(c.B, 2, c.N, c.K, 64);
  const CUtensorMap tb_lo = operand_map(blo, 2, c.N, c.K, 64);
  const CUtensorMap tc = c.out ? make_map(c.out, 2, c.N, c.M, c.ldo, 64, 32) : ta;
  const CUtensorMap tc_lo = c.out ? make_map(c.out_lo, 2, c.N, c.M, c.ldo, 64, 32) : ta;
  GemmArgs a{};
  a.M = c.M;
  a.N = c.N;
  a.K = c.K;
  a.out = c.out;
  a.ldo = c.ldo;
  a.bias = c.bias;
  a.relu = c.relu;
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.mn_layout = g_mn_layout[0];
  a.mn_sbo = g_mn_sbo[0];
  a.mn_kstep = g_mn_kstep[0];
  a.kperm = c.kperm && c.K == 512;
  const int tiles_m2 = ceil_div(c.M, 2 * Cfg::BM);
  const int groups = c.N / 128;  // pair groups per m tile (4 at N = 512)
  if (groups != 4) fail(MOSES_ERR_INVALID_ARG, "split pair layer: N = 512");
  int pairs = std::min(g_num_sms / 2, groups * tiles_m2);
  pairs -= pairs % groups;  // every column quarter gets the same number of pairs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, ta_lo, tb, tb_lo, tc, tc_lo, a, tiles_m2));
}

template <bool BMN, int EPI>
void launch_c(const GemmCall& c, cudaStream_t s) {
  auto kern = umma_gemm_cluster<BMN, EPI>;
  static bool configured = false;
  if (!configured) {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CCfg::kSmemLimit));
    configured = true;
  }
  const int num_kb = ceil_div(c.K, CCfg::BK);
  // A: 32-row quarters (multicast), B: resident 128-column slices
  const CUtensorMap ta = make_map(c.A.ptr, 2, c.K, c.M, c.A.ld, 64, 32);
  const CUtensorMap tb = operand_map(c.B, 2, c.N, c.K, CCfg::BN);
  GemmArgs a{};
  a.M = c.M;
  a.N = c.N;
  a.K = c.K;
  a.out = c.out;
  a.ldo = c.ldo;
  a.bias = c.bias;
  a.relu = c.relu;
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.mask = c.mask;
  a.ldm = c.ldm;
  a.round_out = c.round_out;
  const int tm = ceil_div(c.M, CCfg::BM);
  const int clusters = std::max(1, std::min(tm, g_num_sms / CCfg::kCluster));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * CCfg::kCluster);
  cfg.blockDim = dim3(CCfg::kThreads);
  cfg.dynamicSmemBytes = CCfg::smem_bytes(num_kb);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, a, tm, CCfg::stages_for(num_kb)));
}

template <bool FWD>
void launch_chain_t(const ChainCall& c, cudaStream_t s) {
  auto kern = mlp_chain_kernel<FWD>;
  static std::once_flag once;
  std::call_once(once, [&] {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ChainCfg::kSmemBytes));
  });
  ChainMaps maps;
  ChainArgs a{};
  a.M = c.M;
  a.n_layers = c.n_layers;
  maps.in = make_map(c.in, 2, c.K[0], c.M, c.ld_in, 64, 128);
  for (int l = 0; l < c.n_layers; ++l) {
    a.K[l] = c.K[l];
    a.bias[l] = c.bias[l];
    a.out[l] = static_cast<__nv_bfloat16*>(c.out[l]);
    a.ldo[l] = c.ldo[l];
    a.mask[l] = static_cast<const __nv_bfloat16*>(c.mask[l]);
    a.ldm[l] = c.ldm[l];
    maps.w[l] = FWD ? make_map(c.w[l], 2, ChainCfg::kWidth, c.K[l], ChainCfg::kWidth, 64, 64)
                    : make_map(c.w[l], 2, ChainCfg::kWidth, ChainCfg::kWidth, ChainCfg::kWidth, 64, 128);
    if (c.out[l] != nullptr) maps.out[l] = make_map(c.out[l], 2, ChainCfg::kWidth, c.M, c.ldo[l], 64, 128);
  }
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.trace = c.trace ? c.trace : g_chain_trace;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ChainCfg::kCluster * ceil_div(c.M, ChainCfg::BM));
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = ChainCfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, maps, a));
}

template <bool UPDATE, bool SPLIT>
void launch_group_t(const WgradGroupCall& c, cudaStream_t s) {
  using Cfg = std::conditional_t<SPLIT, GroupSplitCfg, GroupCfg>;
  static std::once_flag once;
  std::call_once(once, [&] {
    if constexpr (SPLIT)
      MOSES_CUDA(cudaFuncSetAttribute(wgrad_group_split_kernel<UPDATE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cfg::kSmemBytes));
    else
      MOSES_CUDA(cudaFuncSetAttribute(wgrad_group_kernel<UPDATE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cfg::kSmemBytes));
  });
  GroupMapsSplit maps;
  GroupArgs a{};
  a.n = c.n;
  a.K = c.K;
  int tiles = 0;
  for (int l = 0; l < c.n; ++l) {
    maps.a[l] = make_map(c.a[l], 2, c.M[l], c.K, c.lda[l], 64, Cfg::BK);
    maps.b[l] = make_map(c.b[l], 2, c.N[l], c.K, c.ldb[l], 64, Cfg::BK);
    if constexpr (SPLIT) {
      if (!c.a_lo[l] || !c.b_lo[l] || (UPDATE && !c.shadow_lo[l]))
        fail(MOSES_ERR_INVALID_ARG, "split grouped wgrad needs the lo planes");
      maps.a_lo[l] = make_map(c.a_lo[l], 2, c.M[l], c.K, c.lda[l], 64, Cfg::BK);
      maps.b_lo[l] = make_map(c.b_lo[l], 2, c.N[l], c.K, c.ldb[l], 64, Cfg::BK);
      a.shadow_lo[l] = static_cast<__nv_bfloat16*>(c.shadow_lo[l]);
    }
    a.tile_begin[l] = tiles;
    a.tiles_n[l] = ceil_div(c.N[l], GroupCfg::BN);
    a.M[l] = c.M[l];
    a.N[l] = c.N[l];
    a.g[l] = c.g[l];
    a.w[l] = c.w[l];
    a.mom[l] = c.mom[l];
    a.shadow[l] = static_cast<__nv_bfloat16*>(c.shadow[l]);
    tiles += ceil_div(c.M[l], GroupCfg::BM) * a.tiles_n[l];
  }
  a.tile_begin[c.n] = tiles;
  a.lr = c.lr;
  a.mu = c.mu;
  a.counter = c.counter;
  a.loss_src = c.loss_src;
  a.loss_acc = c.loss_acc;
  a.loss_copy = c.loss_copy;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles);
  cfg.blockDim = dim3(SPLIT ? 192 : 128);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if constexpr (SPLIT)
    MOSES_CUDA(cudaLaunchKernelEx(&cfg, wgrad_group_split_kernel<UPDATE>, maps, a));
  else
    MOSES_CUDA(cudaLaunchKernelEx(&cfg, wgrad_group_kernel<UPDATE>, static_cast<const GroupMaps&>(maps), a));
}

// Split-bf16 weight gradients split over the batch rows in clusters of S CTAs (gemm_wgrad_sk.cuh).
// S is the largest cluster width in 1..8 that still fits every CTA in one wave (the occupancy API's
// active-cluster count for this kernel) and minimises the 128-row chunks per CTA.
template <bool UPDATE>
void launch_wgrad_sk_t(const WgradGroupCall& c, cudaStream_t s) {
  using C = WgskCfg;
  auto kern = wgrad_sk_kernel<UPDATE>;
  static std::once_flag once;
  static int max_clusters[9] = {};
  std::call_once(once, [&] {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
    for (int S = 1; S <= 8; ++S) {
      cudaLaunchConfig_t q{};
      q.gridDim = dim3(S * 16);
      q.blockDim = dim3(C::kThreads);
      q.dynamicSmemBytes = C::kSmemBytes;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = unsigned(S);
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.attrs = at;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess) {
        (void)cudaGetLastError();
        n = 0;
      }
      max_clusters[S] = n;
    }
  });
  GroupMapsSplit maps;
  WgskArgs a{};
  GroupArgs& ga = a.ga;
  ga.n = c.n;
  ga.K = c.K;
  int tiles = 0;
  for (int l = 0; l < c.n; ++l) {
    if (!c.a_lo[l] || !c.b_lo[l] || (c.update && !c.shadow_lo[l]))
      fail(MOSES_ERR_INVALID_ARG, "split wgrad needs the lo planes");
    maps.a[l] = make_map(c.a[l], 2, c.M[l], c.K, c.lda[l], 64, C::BK);
    maps.b[l] = make_map(c.b[l], 2, c.N[l], c.K, c.ldb[l], 64, C::BK);
    maps.a_lo[l] = make_map(c.a_lo[l], 2, c.M[l], c.K, c.lda[l], 64, C::BK);
    maps.b_lo[l] = make_map(c.b_lo[l], 2, c.N[l], c.K, c.ldb[l], 64, C::BK);
    const int dims = c.M[l] - 1;  // the last G row is the bias (ones column of act_l)
    a.bias_sep[l] = (dims % C::BM) == 0;
    a.Mg[l] = a.bias_sep[l] ? dims : c.M[l];
    a.bias_row[l] = dims;
    {  // bias columns per m-tile: spread over the level's m-tiles when they divide the tile evenly
      const int mt = ceil_div(a.Mg[l], C::BM);
      a.bias_w[l] = (C::BN % (2 * mt) == 0) ? C::BN / mt : C::BN;
    }
    ga.tile_begin[l] = tiles;
    ga.tiles_n[l] = ceil_div(c.N[l], C::BN);
    ga.M[l] = c.M[l];
    ga.N[l] = c.N[l];
    ga.g[l] = c.g[l];
    ga.w[l] = c.w[l];
    ga.mom[l] = c.mom[l];
    ga.shadow[l] = static_cast<__nv_bfloat16*>(c.shadow[l]);
    ga.shadow_lo[l] = static_cast<__nv_bfloat16*>(c.shadow_lo[l]);
    tiles += ceil_div(a.Mg[l], C::BM) * ga.tiles_n[l];
  }
  ga.tile_begin[c.n] = tiles;
  ga.lr = c.lr;
  ga.mu = c.mu;
  ga.counter = c.counter;
  ga.loss_src = c.loss_src;
  ga.loss_acc = c.loss_acc;
  ga.loss_copy = c.loss_copy;
  a.kc = g_wgrad_sk_kc > 0 ? g_wgrad_sk_kc : C::kChunkKb;
  a.trace = g_wgrad_sk_trace;
  const int chunks = ceil_div(c.K, C::BK * a.kc);
  int S = 1, best = chunks;
  const int budget = c.max_ctas > 0 ? std::min(c.max_ctas, kWgskMaxCtas) : kWgskMaxCtas;
  for (int cand = 2; cand <= std::min(8, c.max_split); ++cand) {
    if (cand > chunks || (long long)tiles > (long long)max_clusters[cand] || (long long)tiles * cand > budget) continue;
    const int per = ceil_div(chunks, cand);
    if (per < best) {
      best = per;
      S = cand;
    }
  }
  if (g_wgrad_sk_splits > 0) S = std::min(g_wgrad_sk_splits, std::max(1, chunks));
  if (S > 1 && (c.sk_ws == nullptr || (long long)tiles * S > kWgskMaxCtas)) S = 1;
  a.S = S;
  a.ws = c.sk_ws;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles * S);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = unsigned(S);
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, maps, a));
}

template <typename T, int BN>
void dispatch_persistent(const GemmCall& c, cudaStream_t s) {
  const bool am = c.A.mn_major, bm = c.B.mn_major;
  switch (c.epi) {
    case EpiKind::Fwd:
      if (!am && bm) return launch_p<T, BN, false, true, int(Epi::Fwd)>(c, s);
      if (!am && !bm) return launch_p<T, BN, false, false, int(Epi::Fwd)>(c, s);
      break;
    case EpiKind::Dgrad:
      if (!am && !bm) return launch_p<T, BN, false, false, int(Epi::Dgrad)>(c, s);
      break;
    case EpiKind::StoreF32:
      if (am && bm) return launch_p<T, BN, true, true, int(Epi::StoreF32)>(c, s);
      if (!am && !bm) return launch_p<T, BN, false, false, int(Epi::StoreF32)>(c, s);
      if (!am && bm) return launch_p<T, BN, false, true, int(Epi::StoreF32)>(c, s);
      break;
  }
  fail(MOSES_ERR_INVALID_ARG, "unsupported persistent GEMM combination");
}

// 3xTF32 (fp32 parity mode): gemm_split.cuh, 128 x 64 tiles
template <bool AMN, bool BMN, int EPI>
void launch_s(const GemmCall& c, cudaStream_t s) {
  constexpr int BN = 64;
  using Cfg = SCfg<BN>;
  auto kern = umma_gemm_split<BN, AMN, BMN, EPI>;
  static std::once_flag once;
  std::call_once(once, [&] {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
  });
  const CUtensorMap ta = operand_map(c.A, 4, c.M, c.K, Cfg::BM);
  const CUtensorMap tb = operand_map(c.B, 4, c.N, c.K, BN);
  const CUtensorMap tal = operand_map({c.A.lo, c.A.ld, c.A.mn_major}, 4, c.M, c.K, Cfg::BM);
  const CUtensorMap tbl = operand_map({c.B.lo, c.B.ld, c.B.mn_major}, 4, c.N, c.K, BN);
  GemmArgs a{};
  a.M = c.M;
  a.N = c.N;
  a.K = c.K;
  a.out = c.out;
  a.ldo = c.ldo;
  a.bias = c.bias;
  a.relu = c.relu;
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.mask = c.mask;
  a.ldm = c.ldm;
  a.mn_layout = g_mn_layout[1];
  a.mn_sbo = g_mn_sbo[1];
  a.mn_kstep = g_mn_kstep[1];
  a.round_out = c.round_out;
  a.out_lo = c.out_lo;
  kern<<<dim3(ceil_div(c.M, Cfg::BM), ceil_div(c.N, BN)), 192, Cfg::kSmemBytes, s>>>(ta, tb, tal, tbl, a);
  MOSES_CUDA(cudaGetLastError());
}

void dispatch_split(const GemmCall& c, cudaStream_t s) {
  const bool am = c.A.mn_major, bm = c.B.mn_major;
  switch (c.epi) {
    case EpiKind::Fwd:
      if (!am && bm) return launch_s<false, true, int(Epi::Fwd)>(c, s);
      break;
    case EpiKind::Dgrad:
      if (!am && !bm) return launch_s<false, false, int(Epi::Dgrad)>(c, s);
      break;
    case EpiKind::StoreF32:
      if (am && bm) return launch_s<true, true, int(Epi::StoreF32)>(c, s);
      break;
  }
  fail(MOSES_ERR_INVALID_ARG, "unsupported 3xTF32 GEMM combination");
}

template <typename T, int BN>
void dispatch_major(const GemmCall& c, cudaStream_t s) {
  const bool am = c.A.mn_major, bm = c.B.mn_major;
  switch (c.epi) {
    case EpiKind::Fwd:
      if (!am && bm) return launch_t<T, BN, false, true, int(Epi::Fwd)>(c, s);
      if (!am && !bm) return launch_t<T, BN, false, false, int(Epi::Fwd)>(c, s);
      break;
    case EpiKind::Dgrad:
      if (!am && !bm) return launch_t<T, BN, false, false, int(Epi::Dgrad)>(c, s);
      break;
    case EpiKind::StoreF32:
      if (am && bm) return launch_t<T, BN, true, true, int(Epi::StoreF32)>(c, s);
      if (!am && !bm) return launch_t<T, BN, false, false, int(Epi::StoreF32)>(c, s);
      if (!am && bm) return launch_t<T, BN, false, true, int(Epi::StoreF32)>(c, s);
      break;
  }
  fail(MOSES_ERR_INVALID_ARG, "unsupported GEMM operand-major / epilogue combination");
}

template <typename T>
void dispatch_bn(const GemmCall& c, int bn, cudaStream_t s) {
  switch (bn) {
    case 64: return dispatch_major<T, 64>(c, s);
    case 128: return dispatch_major<T, 128>(c, s);
    default: return dispatch_major<T, 256>(c, s);
  }
}

}  // namespace

// Largest N tile that still gives at least one full wave of CTAs on 148 SMs;
// small problems fall back to BN=64 for parallelism.
int gemm_pick_bn(int M, int N) {
  const int mt = ceil_div(M, 128);
  for (int bn : {256, 128}) {
    if (N >= bn && (long long)mt * ceil_div(N, bn) >= 148) return bn;
  }
  return 64;
}

int g_num_sms = 148;
int g_persistent = 1;  // persistent kernel for problems with more tiles than SMs
int g_fwd = 1;  // scoring-shape forward kernel (gemm_fwd.cuh)
int g_pair = 1;  // weight-resident CTA-pair forward kernel (gemm_fwd2.cuh)
int g_cluster = 1;     // weight-resident cluster kernel for the 512-wide hidden layers

int g_chain = 1;
unsigned long long* g_chain_trace = nullptr;
int g_group = 1;
int g_wgrad_sk = 1;          // split-bf16 wgrad split over K in clusters (gemm_wgrad_sk.cuh)
int g_wgrad_sk_splits = 0;   // > 0: force the cluster width (tests)
int g_chain_pair = 0;        // split chain on CTA pairs (mlp_chain_split_pair_kernel; measured no faster)
int g_wgrad_early = 1;       // split bf16: last hidden level's wgrad beside the dZ chain
int g_wgrad_sk_kc = 0;       // > 0: k-blocks per TMEM promotion chunk (experiments)
unsigned long long* g_wgrad_sk_trace = nullptr;
int g_rank_fused = 1;
size_t wgrad_sk_ws_bytes() { return size_t(kWgskMaxCtas) * kSlotFloats * sizeof(float); }
void launch_wgrad_group(const WgradGroupCall& c, cudaStream_t s) {
  if (c.K <= 0 || c.n <= 0) return;
  if (c.n > kGroupMax) fail(MOSES_ERR_INVALID_ARG, "too many levels for the grouped wgrad");
  if (c.split && g_wgrad_sk) {
    if (c.update) launch_wgrad_sk_t<true>(c, s);
    else launch_wgrad_sk_t<false>(c, s);
  } else if (c.split) {
    if (c.update) launch_group_t<true, true>(c, s);
    else launch_group_t<false, true>(c, s);
  } else {
    if (c.update) launch_group_t<true, false>(c, s);
    else launch_group_t<false, false>(c, s);
  }
}
template <bool FWD>
void launch_chain_split_t(const ChainCall& c, cudaStream_t s) {
  auto kern = mlp_chain_split_stream_kernel<FWD>;
  static std::once_flag once;
  std::call_once(once, [&] {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    ChainSplitStreamCfg::kSmemBytes));
  });
  if (c.in_lo == nullptr) fail(MOSES_ERR_INVALID_ARG, "split chain needs the input lo plane");
  ChainSplitMaps maps;
  ChainArgs a{};
  a.M = c.M;
  a.n_layers = c.n_layers;
  maps.in = make_map(c.in, 2, c.K[0], c.M, c.ld_in, 64, 128);
  maps.in_lo = make_map(c.in_lo, 2, c.K[0], c.M, c.ld_in, 64, 128);
  constexpr int W = ChainSplitStreamCfg::kWidth;
  for (int l = 0; l < c.n_layers; ++l) {
    a.K[l] = c.K[l];
    a.bias[l] = c.bias[l];
    a.out[l] = static_cast<__nv_bfloat16*>(c.out[l]);
    a.out_lo[l] = static_cast<__nv_bfloat16*>(c.out_lo[l]);
    a.ldo[l] = c.ldo[l];
    a.mask[l] = static_cast<const __nv_bfloat16*>(c.mask[l]);
    a.ldm[l] = c.ldm[l];
    if (c.w_lo[l] == nullptr) fail(MOSES_ERR_INVALID_ARG, "split chain needs the weight lo planes");
    maps.w[l] = FWD ? make_map(c.w[l], 2, W, c.K[l], W, 64, 64) : make_map(c.w[l], 2, W, W, W, 64, 128);
    maps.w_lo[l] = FWD ? make_map(c.w_lo[l], 2, W, c.K[l], W, 64, 64) : make_map(c.w_lo[l], 2, W, W, W, 64, 128);
    if (c.out[l] != nullptr) {
      if (c.out_lo[l] == nullptr) fail(MOSES_ERR_INVALID_ARG, "split chain output without a lo plane");
      maps.out[l] = make_map(c.out[l], 2, W, c.M, c.ldo[l], 64, 128);
      maps.out_lo[l] = make_map(c.out_lo[l], 2, W, c.M, c.ldo[l], 64, 128);
    }
  }
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.trace = c.trace ? c.trace : g_chain_trace;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ChainSplitStreamCfg::kCluster * ceil_div(c.M, ChainSplitStreamCfg::BM));
  cfg.blockDim = dim3(ChainSplitStreamCfg::kThreads);
  cfg.dynamicSmemBytes = ChainSplitStreamCfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, maps, a));
}

// split chain on CTA pairs (mlp_chain_split_pair_kernel), 8-CTA clusters of 256 rows
template <bool FWD>
void launch_chain_pair_t(const ChainCall& c, cudaStream_t s) {
  auto kern = mlp_chain_split_pair_kernel<FWD>;
  static std::once_flag once;
  std::call_once(once, [&] {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    ChainPairCfg::kSmemBytes));
  });
  if (c.in_lo == nullptr) fail(MOSES_ERR_INVALID_ARG, "split chain needs the input lo plane");
  ChainSplitMaps maps;
  ChainArgs a{};
  a.M = c.M;
  a.n_layers = c.n_layers;
  maps.in = make_map(c.in, 2, c.K[0], c.M, c.ld_in, 64, 128);
  maps.in_lo = make_map(c.in_lo, 2, c.K[0], c.M, c.ld_in, 64, 128);
  constexpr int W = ChainPairCfg::kWidth;
  for (int l = 0; l < c.n_layers; ++l) {
    a.K[l] = c.K[l];
    a.bias[l] = c.bias[l];
    a.out[l] = static_cast<__nv_bfloat16*>(c.out[l]);
    a.out_lo[l] = static_cast<__nv_bfloat16*>(c.out_lo[l]);
    a.ldo[l] = c.ldo[l];
    a.mask[l] = static_cast<const __nv_bfloat16*>(c.mask[l]);
    a.ldm[l] = c.ldm[l];
    if (c.w_lo[l] == nullptr) fail(MOSES_ERR_INVALID_ARG, "split chain needs the weight lo planes");
    maps.w[l] = FWD ? make_map(c.w[l], 2, W, c.K[l], W, 64, 64) : make_map(c.w[l], 2, W, W, W, 64, 64);
    maps.w_lo[l] = FWD ? make_map(c.w_lo[l], 2, W, c.K[l], W, 64, 64) : make_map(c.w_lo[l], 2, W, W, W, 64, 64);
    if (c.out[l] != nullptr) {
      if (c.out_lo[l] == nullptr) fail(MOSES_ERR_INVALID_ARG, "split chain output without a lo plane");
      maps.out[l] = make_map(c.out[l], 2, W, c.M, c.ldo[l], 64, 128);
      maps.out_lo[l] = make_map(c.out_lo[l], 2, W, c.M, c.ldo[l], 64, 128);
    }
  }
  a.head_w = c.head_w;
  a.head_u = c.head_u;
  a.head_part = c.head_part;
  a.head_part2 = c.head_part2;
  a.head_ld = c.head_ld;
  a.trace = c.trace ? c.trace : g_chain_trace;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ChainPairCfg::kCluster * ceil_div(c.M, 2 * ChainPairCfg::BM));
  cfg.blockDim = dim3(ChainPairCfg::kThreads);
  cfg.dynamicSmemBytes = ChainPairCfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOSES_CUDA(cudaLaunchKernelEx(&cfg, kern, maps, a));
}

void launch_chain(const ChainCall& c, cudaStream_t s) {
  if (c.M <= 0) return;
  if (c.n_layers < 1 || c.n_layers > kChainMaxLayers) fail(MOSES_ERR_INVALID_ARG, "chain depth");
  if (c.split) {
    if (g_chain_pair) {
      if (c.fwd) launch_chain_pair_t<true>(c, s);
      else launch_chain_pair_t<false>(c, s);
    } else {
      if (c.fwd) launch_chain_split_t<true>(c, s);
      else launch_chain_split_t<false>(c, s);
    }
    return;
  }
  if (c.fwd) launch_chain_t<true>(c, s);
  else launch_chain_t<false>(c, s);
}

int launch_gemm(int elem, const GemmCall& c, cudaStream_t s) {
  if (c.M <= 0 || c.N <= 0) return 0;
  if (c.K <= 0) fail(MOSES_ERR_INVALID_ARG, "GEMM with K == 0");
  static bool sm_init = false;
  if (!sm_init) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      g_num_sms = n;
    sm_init = true;
  }
  if (elem == 2 && (c.A.lo != nullptr || c.B.lo != nullptr)) {  // split bf16: the weight-resident pair layer
    if (!c.A.lo || !c.B.lo || c.epi != EpiKind::Fwd || c.A.mn_major || !c.B.mn_major || c.N != 512 ||
        c.K > PairSplitCfg::kMaxK || (c.ldo * 2) % 16 != 0)
      fail(MOSES_ERR_INVALID_ARG, "split-bf16 GEMMs: forward layers of width 512 with K <= 512");
    launch_pair_split(c, s);
    return 64;  // head partials per 64-column slice
  }
  if (c.A.lo != nullptr || c.B.lo != nullptr) {  // 3xTF32: both operands split, non-persistent kernel
    if (elem != 4 || !c.A.lo || !c.B.lo) fail(MOSES_ERR_INVALID_ARG, "3xTF32 needs fp32 hi/lo operands");
    dispatch_split(c, s);
    return 64;
  }
  // Hidden layers (bf16, N = 512, K <= 512, A K-major): weight-resident 4-CTA cluster kernel.
  // Measured on B200: wins at training sizes (M ~ 2.3K statement rows: 18 m-tiles); at scoring sizes
  // (64K-row chunks) its N=128 SS-MMA is shared-memory-bandwidth bound and the persistent BN=256
  // kernel is 1.7x faster (tools/gemm_sweep.py), so it is limited to M <= 16K rows.
  if (g_cluster && !c.bn && elem == 2 && c.M <= 16384 && c.N == 4 * CCfg::BN && c.K <= CCfg::kMaxK && !c.A.mn_major &&
      (c.epi == EpiKind::Fwd || c.epi == EpiKind::Dgrad) && (c.A.ld * 2) % 16 == 0) {
    if (c.epi == EpiKind::Fwd) {
      if (c.B.mn_major) launch_c<true, int(Epi::Fwd)>(c, s);
      else launch_c<false, int(Epi::Fwd)>(c, s);
    } else {
      if (c.B.mn_major) launch_c<true, int(Epi::Dgrad)>(c, s);
      else launch_c<false, int(Epi::Dgrad)>(c, s);
    }
    return CCfg::BN;
  }
  // Large problems: persistent kernel with double-buffered TMEM accumulators, BN = 256 (or 128).
  const int mt = ceil_div(c.M, 128);
  if (g_persistent && !c.bn && c.N >= 128) {
    const int pbn = c.N >= 256 ? 256 : 128;
    if ((long long)mt * ceil_div(c.N, pbn) >= 2LL * g_num_sms) {
      if (g_pair && elem == 2 && c.epi == EpiKind::Fwd && !c.A.mn_major && c.B.mn_major && c.N == 512 &&
          c.K <= PairCfg::kMaxK && (c.ldo * 2) % 16 == 0 && g_num_sms >= 4) {
        launch_pair(c, s);
        return 128;  // head partials per 128-column quarter
      }
      if (g_fwd && elem == 2 && c.epi == EpiKind::Fwd && !c.A.mn_major && (c.ldo * 2) % 16 == 0) {
        if (pbn == 256) c.B.mn_major ? launch_f<256, true>(c, s) : launch_f<256, false>(c, s);
        else c.B.mn_major ? launch_f<128, true>(c, s) : launch_f<128, false>(c, s);
        return pbn / 2;  // head partials per half tile
      }
      if (elem == 2) {
        if (pbn == 256) dispatch_persistent<__nv_bfloat16, 256>(c, s);
        else dispatch_persistent<__nv_bfloat16, 128>(c, s);
      } else {
        if (pbn == 256) dispatch_persistent<float, 256>(c, s);
        else dispatch_persistent<float, 128>(c, s);
      }
      return pbn;
    }
  }
  const int bn = c.bn ? c.bn : gemm_pick_bn(c.M, c.N);
  if (elem == 2) dispatch_bn<__nv_bfloat16>(c, bn, s);
  else dispatch_bn<float>(c, bn, s);
  return bn;
}

// ---------------------------------------------------------------- MMD^2 on the tensor cores
namespace {
// one warp per row: tf32 (RNA) copy into a 16-B-aligned padded row + squared norm of the rounded row
__global__ void gram_prep_kernel(const float* __restrict__ X, long long rows, int W, long long ld,
                                 float* __restrict__ Xp, long long ldp, float* __restrict__ norms) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    float acc = 0.f;
    for (int j = lane; j < ldp; j += 32) {
      const float v = j < W ? tf32_round(X[r * ld + j]) : 0.f;
      Xp[r * ldp + j] = v;
      acc = fmaf(v, v, acc);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) norms[r] = acc;
  }
}
__global__ void __launch_bounds__(1024) gram_sum_kernel(const double* p, long long n, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += 1024) s += p[i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = sh[threadIdx.x];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
  }
}
long long gram_tiles(long long M, long long N, bool sym) {
  const long long tm = (M + 127) / 128, tn = (N + 127) / 128;
  return sym ? tm * (tm + 1) / 2 : tm * tn;
}
}  // namespace

size_t mmd_ws_bytes(long long m, long long n, int W) {
  const long long ldp = (W + 3) / 4 * 4;
  const long long tiles = std::max(gram_tiles(m, m, true), std::max(gram_tiles(n, n, true), gram_tiles(m, n, false)));
  return size_t(m + n) * ldp * 4 + size_t(m + n) * 4 + size_t(tiles) * 4 * 8 + 64 + 4 * 256;
}

// Gram reduction S(X, Y) into *out (device double); X, Y: tf32-rounded rows with stride ldp.
static void gram_sum(const float* X, long long M, const float* nx, const float* Y, long long N, const float* ny, int W,
                     long long ldp, float c, bool sym, double* part, double* out, cudaStream_t s) {
  auto kern = umma_gram_kernel;
  static std::once_flag once;
  std::call_once(once, [&] {
    MOSES_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GCfg::kSmemBytes));
  });
  const CUtensorMap ta = make_map(X, 4, W, M, ldp, 32, 128);
  const CUtensorMap tb = make_map(Y, 4, W, N, ldp, 32, 128);
  GramArgs g{};
  g.M = int(M);
  g.N = int(N);
  g.K = W;
  g.nx = nx;
  g.ny = ny;
  g.c = c;
  g.sym = sym ? 1 : 0;
  g.part = part;
  const long long tiles = gram_tiles(M, N, sym);
  const int grid = int(std::min<long long>(tiles, g_num_sms));
  kern<<<grid, GCfg::kThreads, GCfg::kSmemBytes, s>>>(ta, tb, g, ceil_div(M, 128), tiles);
  gram_sum_kernel<<<1, 1024, 0, s>>>(part, tiles * 4, out);
  MOSES_CUDA(cudaGetLastError());
}

// Biased MMD^2 (oracle mmd2): S(s,s)/m^2 + S(t,t)/n^2 - 2 S(s,t)/(m n); rows of xs / xt with stride ld.
double mmd2_tc(const float* xs, long long m, const float* xt, long long n, int W, long long ld, float sigma, void* ws,
               cudaStream_t s, int* launches) {
  if (g_num_sms <= 0) g_num_sms = 148;
  const long long ldp = (W + 3) / 4 * 4;
  uint8_t* p = static_cast<uint8_t*>(ws);
  float* Xp = reinterpret_cast<float*>(p);
  float* norms = Xp + (m + n) * ldp;
  double* sums = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(norms) + ((m + n) * 4 + 255) / 256 * 256);
  double* part = sums + 8;
  gram_prep_kernel<<<int(std::min<long long>((m + 7) / 8, 4096)), 256, 0, s>>>(xs, m, W, ld, Xp, ldp, norms);
  gram_prep_kernel<<<int(std::min<long long>((n + 7) / 8, 4096)), 256, 0, s>>>(xt, n, W, ld, Xp + m * ldp, ldp,
                                                                               norms + m);
  const float c = float(1.4426950408889634 / (2.0 * double(sigma) * double(sigma)));
  const float* Xs = Xp;
  const float* Xt = Xp + m * ldp;
  gram_sum(Xs, m, norms, Xs, m, norms, W, ldp, c, true, part, sums + 0, s);
  gram_sum(Xt, n, norms + m, Xt, n, norms + m, W, ldp, c, true, part, sums + 1, s);
  gram_sum(Xs, m, norms, Xt, n, norms + m, W, ldp, c, false, part, sums + 2, s);
  double h[3];
  MOSES_CUDA(cudaMemcpyAsync(h, sums, sizeof(h), cudaMemcpyDeviceToHost, s));
  MOSES_CUDA(cudaStreamSynchronize(s));
  if (launches) *launches = 8;
  return h[0] / (double(m) * double(m)) + h[1] / (double(n) * double(n)) - 2.0 * h[2] / (double(m) * double(n));
}

}  // namespace moses
