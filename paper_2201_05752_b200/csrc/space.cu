// space.cu — candidate generation on the device: the knob-space helpers
// of the reference's scorer input path, so a candidate pool never crosses PCIe.
//
//   enumerate_configs (space.cpp:168-191): config `index` of the lexicographic enumeration, last
//     knob fastest = the mixed-radix digits of the index over the knob domain sizes;
//   encode_features (space.cpp:140-159): the 16-d feature row (10 live entries, 6 zero) in double,
//     rounded once to the model's operand type and written as a packed model row;
//   config_hash (space.cpp:193-197): FNV-1a over each value's 8 little-endian bytes — the identity
//     select_batch dedups on (search.cpp:82-95).
// One thread per configuration; the task-level entries (f7..f9) are computed on the host exactly
// like the reference (std::log10 / std::clamp) and passed in.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace moses {

constexpr int kSpaceMaxKnobs = 8;
constexpr int kSpaceMaxValues = 256;

struct SpaceArgs {
  double bytes_per_unit;
  double f7, f8, f9;  // task-level entries
  int nk;
  int sizes[kSpaceMaxKnobs], offs[kSpaceMaxKnobs], roles[kSpaceMaxKnobs];
  long long domains[kSpaceMaxValues];
  // Table path: f0..f6 are functions of the template knobs' domain indices only, so the host
  // evaluates them once per value (the reference's own expressions, std::log2 in double) and the
  // kernel gathers: t[r] = table of role r (f0..f4), t5 over (tile_x, tile_y), t6 over
  // (tile_x, tile_y, unroll). role_knob[r] = knob index of role r (-1: absent, index 0).
  const double* tab;  // null: evaluate on the device
  int tab_off[7], role_knob[5], role_size[5];
};

namespace {

template <typename T>
__device__ __forceinline__ T cvt_out(double v);
template <>
__device__ __forceinline__ float cvt_out<float>(double v) { return float(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(double v) { return __float2bfloat16_rn(float(v)); }
template <>
__device__ __forceinline__ double cvt_out<double>(double v) { return v; }

template <typename T>
__global__ void __launch_bounds__(256) encode_configs_kernel(const __grid_constant__ SpaceArgs a,
                                                             unsigned long long first, long long n, T* __restrict__ feat,
                                                             long long ld, int D, unsigned long long* __restrict__ hash,
                                                             long long* __restrict__ values_out,
                                                             const unsigned long long* __restrict__ idx_list) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long idx = idx_list ? idx_list[i] : first + (unsigned long long)i;
    long long v[kSpaceMaxKnobs];
    unsigned digit[kSpaceMaxKnobs];
    if (idx >> 32) {  // mixed-radix digits, last knob fastest
#pragma unroll
      for (int k = kSpaceMaxKnobs - 1; k >= 0; --k) {
        digit[k] = 0;
        if (k >= a.nk) continue;
        const unsigned long long s = (unsigned long long)a.sizes[k];
        digit[k] = unsigned(idx % s);
        idx /= s;
      }
    } else {  // 32-bit division is several times cheaper
      unsigned i32 = unsigned(idx);
#pragma unroll
      for (int k = kSpaceMaxKnobs - 1; k >= 0; --k) {
        digit[k] = 0;
        if (k >= a.nk) continue;
        const unsigned s = unsigned(a.sizes[k]);
        digit[k] = i32 % s;
        i32 /= s;
      }
    }
#pragma unroll
    for (int k = 0; k < kSpaceMaxKnobs; ++k) v[k] = k < a.nk ? a.domains[a.offs[k] + int(digit[k])] : 0;
    long long kv[5] = {1, 1, 0, 1, 1};  // knob_view fallbacks (space.cpp:132-136)
    unsigned seen = 0;                    // find_knob takes the first knob of a name
    unsigned long long h = 0xcbf29ce484222325ull;
#pragma unroll
    for (int k = 0; k < kSpaceMaxKnobs; ++k) {
      if (k >= a.nk) continue;
      const int r = a.roles[k];
      if (r >= 0 && r < 5 && !(seen & (1u << r))) {
        kv[r] = v[k];
        seen |= 1u << r;
      }
      const unsigned long long u = (unsigned long long)v[k];
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        h ^= (u >> (8 * b)) & 0xffull;
        h *= 0x100000001b3ull;
      }
      if (values_out) values_out[i * a.nk + k] = v[k];
    }
    if (hash) hash[i] = h;
    if (feat == nullptr) continue;
    double f[10];
    if (a.tab != nullptr) {
      int ri[5];
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        const int k = a.role_knob[r];
        ri[r] = 0;
#pragma unroll
        for (int kk = 0; kk < kSpaceMaxKnobs; ++kk)
          if (kk == k) ri[r] = int(digit[kk]);
      }
#pragma unroll
      for (int r = 0; r < 5; ++r) f[r] = __ldg(a.tab + a.tab_off[r] + ri[r]);
      const int txy = ri[0] * a.role_size[1] + ri[1];
      f[5] = __ldg(a.tab + a.tab_off[5] + txy);
      f[6] = __ldg(a.tab + a.tab_off[6] + txy * a.role_size[2] + ri[2]);
    } else {
      const double tx = double(kv[0]), ty = double(kv[1]), un = double(kv[2]);
      const double footprint = a.bytes_per_unit * tx * ty * fmax(1.0, un);
      f[0] = log2(tx) / 6.0;
      f[1] = log2(ty) / 6.0;
      f[2] = log2(1.0 + un) / 10.0;
      f[3] = log2(double(kv[3])) / 4.0;
      f[4] = log2(double(kv[4])) / 8.0;
      f[5] = log2(tx * ty) / 12.0;
      f[6] = log2(footprint) / 24.0;
    }
    f[7] = a.f7;
    f[8] = a.f8;
    f[9] = a.f9;
    T* row = feat + i * ld;
    if constexpr (sizeof(T) == 2) {
      if (ld % 8 == 0 && ld <= 32 && D + 1 <= ld && ((reinterpret_cast<uintptr_t>(feat) & 15) == 0)) {  // 16-B rows
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += 8) {  // ld <= 32 on this path
          if (c0 >= ld) break;
          uint4 pk;
          T* pe = reinterpret_cast<T*>(&pk);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int j = c0 + q;
            pe[q] = cvt_out<T>(j < 10 ? f[j < 10 ? j : 0] : (j == D ? 1.0 : 0.0));  // zero beyond D
          }
          *reinterpret_cast<uint4*>(row + c0) = pk;
        }
        continue;
      }
    }
    for (int j = 0; j < D; ++j) row[j] = cvt_out<T>(j < 10 ? f[j] : 0.0);
    if (ld > D) row[D] = cvt_out<T>(1.0);  // the packed layout's constant column (gradients' bias row)
  }
}

}  // namespace

// validate the knob space (space.cpp:41-66, build_space) into `a`; returns the space size
static unsigned long long fill_space(SpaceArgs& a, const long long* domains, const int* sizes, const int* roles,
                                     int nk) {
  if (nk <= 0 || nk > kSpaceMaxKnobs) fail(MOSES_ERR_INVALID_ARG, "knob count must lie in [1, 8]");
  a.nk = nk;
  int off = 0;
  unsigned long long space = 1;
  for (int k = 0; k < nk; ++k) {
    if (sizes[k] <= 0) fail(MOSES_ERR_INVALID_TASK, "knob domain must be non-empty");
    for (int j = 1; j < sizes[k]; ++j)
      if (domains[off + j - 1] >= domains[off + j]) fail(MOSES_ERR_INVALID_TASK, "knob domain must be strictly increasing");
    a.sizes[k] = sizes[k];
    a.offs[k] = off;
    a.roles[k] = roles[k];
    off += sizes[k];
    if (off > kSpaceMaxValues) fail(MOSES_ERR_INVALID_ARG, "knob domains exceed 256 values in total");
    if (space > ~0ull / (unsigned long long)sizes[k]) fail(MOSES_ERR_SPACE_TOO_LARGE, "knob space overflows 64 bits");
    space *= (unsigned long long)sizes[k];
  }
  std::copy(domains, domains + off, a.domains);
  return space;
}

static int encode_impl(const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                       unsigned long long first, const unsigned long long* idx_list, long long n, int out_kind,
                       void* feat, long long ld, int D, unsigned long long* hash, long long* values_out,
                       cudaStream_t st) {
  SpaceArgs a{};
  const unsigned long long space = fill_space(a, domains, sizes, roles, nk);
  if (n < 0 || (idx_list == nullptr && (first > space || (unsigned long long)n > space - first)))
    fail(MOSES_ERR_SHAPE_MISMATCH, "config range exceeds the knob space");
  a.bytes_per_unit = task4[1];
  a.f7 = std::clamp(std::log10(task4[0]) / 3.0, 0.0, 1.0);  // space.cpp:154
  a.f8 = task4[2] / 16.0;
  a.f9 = task4[3] / 10.0;
  if (feat != nullptr && (D < 10 || ld < D)) fail(MOSES_ERR_INVALID_ARG, "feature rows need D >= 10 and ld >= D");
  if (n == 0) return 0;
  // per-value tables of f0..f6 (host, the reference's expressions in double)
  std::vector<double> dom_r[5];
  const long long fallback[5] = {1, 1, 0, 1, 1};  // knob_view fallbacks (space.cpp:132-136)
  for (int r = 0; r < 5; ++r) {
    a.role_knob[r] = -1;
    for (int k = 0; k < nk; ++k)
      if (roles[k] == r && a.role_knob[r] < 0) a.role_knob[r] = k;
    if (a.role_knob[r] >= 0)
      for (int j = 0; j < sizes[a.role_knob[r]]; ++j) dom_r[r].push_back(double(domains[a.offs[a.role_knob[r]] + j]));
    else
      dom_r[r].push_back(double(fallback[r]));
    a.role_size[r] = int(dom_r[r].size());
  }
  const size_t n5 = dom_r[0].size() * dom_r[1].size(), n6 = n5 * dom_r[2].size();
  std::vector<double> tab;
  if (n6 <= (1u << 20)) {
    auto put = [&](int slot) { a.tab_off[slot] = int(tab.size()); };
    const double div[5] = {6.0, 6.0, 10.0, 4.0, 8.0};
    for (int r = 0; r < 5; ++r) {
      put(r);
      for (double x : dom_r[r]) tab.push_back(r == 2 ? std::log2(1.0 + x) / div[r] : std::log2(x) / div[r]);
    }
    put(5);
    for (double tx : dom_r[0])
      for (double ty : dom_r[1]) tab.push_back(std::log2(tx * ty) / 12.0);
    put(6);
    for (double tx : dom_r[0])
      for (double ty : dom_r[1])
        for (double un : dom_r[2]) tab.push_back(std::log2(task4[1] * tx * ty * std::max<double>(1.0, un)) / 24.0);
  }
  // per-call table, stream-ordered on `st`: callers encode on different streams, so a shared buffer
  // could be overwritten while an earlier encode kernel still reads it
  double* dtab = nullptr;
  if (!tab.empty()) {
    MOSES_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dtab), tab.size() * sizeof(double), st));
    MOSES_CUDA(cudaMemcpyAsync(dtab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    a.tab = dtab;
  }
  const int grid = int(std::min<long long>((n + 255) / 256, 148LL * 16));
  if (out_kind == 1)
    encode_configs_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(a, first, n, static_cast<__nv_bfloat16*>(feat), ld, D,
                                                              hash, values_out, idx_list);
  else if (out_kind == 2)
    encode_configs_kernel<double><<<grid, 256, 0, st>>>(a, first, n, static_cast<double*>(feat), ld, D, hash, values_out,
                                                       idx_list);
  else
    encode_configs_kernel<float><<<grid, 256, 0, st>>>(a, first, n, static_cast<float*>(feat), ld, D, hash, values_out,
                                                      idx_list);
  MOSES_CUDA(cudaGetLastError());
  if (dtab) MOSES_CUDA(cudaFreeAsync(dtab, st));
  return 1;
}
int encode_configs(const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                   unsigned long long first, long long n, int out_kind, void* feat, long long ld, int D,
                   unsigned long long* hash, long long* values_out, cudaStream_t st) {
  return encode_impl(task4, domains, sizes, roles, nk, first, nullptr, n, out_kind, feat, ld, D, hash, values_out, st);
}
int encode_configs_idx(const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                       const unsigned long long* idx_dev, long long n, int out_kind, void* feat, long long ld, int D,
                       cudaStream_t st) {
  return encode_impl(task4, domains, sizes, roles, nk, 0, idx_dev, n, out_kind, feat, ld, D, nullptr, nullptr, st);
}

// ---------------------------------------------------------------- simulated hardware (oracle.cpp:33-105)
// The label generator of the synthetic TenSet-style data: the closed-form
// response model per configuration, keyed Gaussian measurement noise, and the exhaustive
// noise-free optimum (true_best) as an argmin over (latency, enumeration index) — the
// lexicographically first configuration on exact ties, like the reference's strict <.
struct SimArgs {
  SpaceArgs sp;
  double peak, units, lanes, cache, overhead, noise_std, work, bytes, ideal_tiles, ideal_unroll;
  int repeats;
  unsigned long long key0;  // FNV-1a state after (seed, device id, task id)
};

namespace {

__device__ __forceinline__ void sim_decode(const SpaceArgs& a, unsigned long long idx, long long kv[5],
                                           unsigned long long* chash) {
  long long v[kSpaceMaxKnobs];
#pragma unroll
  for (int k = kSpaceMaxKnobs - 1; k >= 0; --k) {
    v[k] = 0;
    if (k >= a.nk) continue;
    const unsigned long long s = (unsigned long long)a.sizes[k];
    v[k] = a.domains[a.offs[k] + int(idx % s)];
    idx /= s;
  }
  kv[0] = 1; kv[1] = 1; kv[2] = 0; kv[3] = 1; kv[4] = 1;
  unsigned seen = 0;
  unsigned long long h = 0xcbf29ce484222325ull;
#pragma unroll
  for (int k = 0; k < kSpaceMaxKnobs; ++k) {
    if (k >= a.nk) continue;
    const int r = a.roles[k];
    if (r >= 0 && r < 5 && !(seen & (1u << r))) {
      kv[r] = v[k];
      seen |= 1u << r;
    }
    const unsigned long long u = (unsigned long long)v[k];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      h ^= (u >> (8 * b)) & 0xffull;
      h *= 0x100000001b3ull;
    }
  }
  *chash = h;
}

__device__ __forceinline__ double sim_clean_throughput(const SimArgs& s, const long long kv[5]) {
  // shared_factor (oracle.cpp:33-41)
  const double log_tiles = log2(double(kv[0] * kv[1]));
  const double dt = log_tiles - s.ideal_tiles;
  const double tile_term = exp(-(dt * dt) / 8.0);  // std::pow(x, 2.0) is correctly rounded: = fl(x * x)
  const double du = log2(1.0 + double(kv[2])) - s.ideal_unroll;
  const double unroll_term = 0.8 + 0.2 * exp(-(du * du) / 4.0);
  // device_factor (oracle.cpp:43-56)
  const double p = double(kv[4]), vec = double(kv[3]);
  const double parallel_term = fmin(p / s.units, s.units / p);
  const double vector_term = sqrt(fmin(vec / s.lanes, s.lanes / vec));
  const double footprint = s.bytes * double(kv[0]) * double(kv[1]) * fmax(1.0, double(kv[2]));
  const double cache_term = footprint <= s.cache ? 1.0 : s.cache / footprint;
  return s.peak * (tile_term * unroll_term) * (parallel_term * vector_term * cache_term);
}

__device__ __forceinline__ unsigned long long sm64(unsigned long long& st) {
  st += 0x9e3779b97f4a7c15ull;
  unsigned long long z = st;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) measure_configs_kernel(const __grid_constant__ SimArgs s,
                                                              unsigned long long first, long long n,
                                                              double* __restrict__ clean_ms, double* __restrict__ thr,
                                                              double* __restrict__ lat, double* __restrict__ wall,
                                                              float* __restrict__ label,
                                                              const unsigned long long* __restrict__ idx_list) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    long long kv[5];
    unsigned long long ch;
    sim_decode(s.sp, idx_list ? idx_list[i] : first + (unsigned long long)i, kv, &ch);
    const double clean_thr = sim_clean_throughput(s, kv);
    if (clean_ms) clean_ms[i] = s.work / clean_thr * 1000.0;  // clean_latency_ms (oracle.cpp:58-63)
    if (thr == nullptr && lat == nullptr && wall == nullptr && label == nullptr) continue;
    // measure (oracle.cpp:65-88): RngStream(KeyBuilder(seed, device, task, config_hash)).gaussian()
    unsigned long long key = s.key0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      key ^= (ch >> (8 * b)) & 0xffull;
      key *= 0x100000001b3ull;
    }
    unsigned long long st = key;
    const double u1 = double((sm64(st) >> 11) + 1) * 0x1.0p-53;
    const double u2 = double(sm64(st) >> 11) * 0x1.0p-53;
    const double g = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
    const double noise = fmax(0.05, 1.0 + g * s.noise_std);
    const double t = clean_thr * noise;
    const double l = s.work / t * 1000.0;
    if (thr) thr[i] = t;
    if (lat) lat[i] = l;
    if (wall) wall[i] = s.overhead + double(s.repeats) * l;
    if (label) label[i] = float(t);
  }
}

struct BestItem {
  double lat;
  unsigned long long idx;
};
__device__ __forceinline__ bool better(const BestItem& a, const BestItem& b) {
  return a.lat < b.lat || (a.lat == b.lat && a.idx < b.idx);
}

__global__ void __launch_bounds__(256) true_best_kernel(const __grid_constant__ SimArgs s, unsigned long long space,
                                                        BestItem* __restrict__ part) {
  BestItem best{__longlong_as_double(0x7ff0000000000000ll), ~0ull};
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < space; i += gridDim.x * 256ull) {
    long long kv[5];
    unsigned long long ch;
    sim_decode(s.sp, i, kv, &ch);
    const BestItem c{s.work / sim_clean_throughput(s, kv) * 1000.0, i};
    if (better(c, best)) best = c;
  }
  __shared__ BestItem sh[256];
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o && better(sh[threadIdx.x + o], sh[threadIdx.x])) sh[threadIdx.x] = sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(256) true_best_final_kernel(BestItem* part, int nparts) {
  __shared__ BestItem sh[256];
  BestItem best{__longlong_as_double(0x7ff0000000000000ll), ~0ull};
  for (int i = threadIdx.x; i < nparts; i += 256)
    if (better(part[i], best)) best = part[i];
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o && better(sh[threadIdx.x + o], sh[threadIdx.x])) sh[threadIdx.x] = sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[0] = sh[0];
}

}  // namespace

static SimArgs make_sim(const double* dev6, int repeats, const double* task4, const long long* domains, const int* sizes,
                        const int* roles, int nk, unsigned long long* space) {
  SimArgs s{};
  *space = fill_space(s.sp, domains, sizes, roles, nk);
  for (int i = 0; i < 4; ++i)
    if (!(dev6[i] > 0.0) || !std::isfinite(dev6[i])) fail(MOSES_ERR_INVALID_CONFIG, "device parameters must be positive");
  if (dev6[4] < 0.0 || dev6[5] < 0.0 || repeats < 1) fail(MOSES_ERR_INVALID_CONFIG, "invalid device");  // oracle.cpp:15-31
  s.peak = dev6[0];
  s.units = dev6[1];
  s.lanes = dev6[2];
  s.cache = dev6[3];
  s.overhead = dev6[4];
  s.noise_std = dev6[5];
  s.repeats = repeats;
  s.work = task4[0];
  s.bytes = task4[1];
  s.ideal_tiles = task4[2];
  s.ideal_unroll = task4[3];
  return s;
}

static void fnv_add_u64(unsigned long long& h, unsigned long long v) {
  for (int b = 0; b < 8; ++b) {
    h ^= (v >> (8 * b)) & 0xffull;
    h *= 0x100000001b3ull;
  }
}
static void fnv_add_str(unsigned long long& h, const char* s) {  // KeyBuilder::add(string): bytes + NUL
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001b3ull;
  }
  h ^= 0;
  h *= 0x100000001b3ull;
}

static int measure_impl(const double* dev6, int repeats, const char* device_id, const char* task_id,
                        const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                        unsigned long long seed, unsigned long long first, const unsigned long long* idx_list,
                        long long n, double* clean_ms, double* thr, double* lat, double* wall, float* label,
                        cudaStream_t st) {
  unsigned long long space;
  SimArgs s = make_sim(dev6, repeats, task4, domains, sizes, roles, nk, &space);
  if (n < 0 || (idx_list == nullptr && (first > space || (unsigned long long)n > space - first)))
    fail(MOSES_ERR_SHAPE_MISMATCH, "config range exceeds the knob space");
  unsigned long long h = 0xcbf29ce484222325ull;
  fnv_add_u64(h, seed);
  fnv_add_str(h, device_id ? device_id : "");
  fnv_add_str(h, task_id ? task_id : "");
  s.key0 = h;
  if (n == 0) return 0;
  const int grid = int(std::min<long long>((n + 255) / 256, 148LL * 16));
  measure_configs_kernel<<<grid, 256, 0, st>>>(s, first, n, clean_ms, thr, lat, wall, label, idx_list);
  MOSES_CUDA(cudaGetLastError());
  return 1;
}
int measure_configs(const double* dev6, int repeats, const char* device_id, const char* task_id, const double* task4,
                    const long long* domains, const int* sizes, const int* roles, int nk, unsigned long long seed,
                    unsigned long long first, long long n, double* clean_ms, double* thr, double* lat, double* wall,
                    float* label, cudaStream_t st) {
  return measure_impl(dev6, repeats, device_id, task_id, task4, domains, sizes, roles, nk, seed, first, nullptr, n,
                      clean_ms, thr, lat, wall, label, st);
}

int measure_configs_idx(const double* dev6, int repeats, const char* device_id, const char* task_id,
                        const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                        unsigned long long seed, const unsigned long long* idx_dev, long long n, double* thr,
                        double* lat, double* wall, cudaStream_t st) {
  return measure_impl(dev6, repeats, device_id, task_id, task4, domains, sizes, roles, nk, seed, 0, idx_dev, n, nullptr,
                      thr, lat, wall, nullptr, st);
}
int true_best(const double* dev6, const double* task4, const long long* domains, const int* sizes, const int* roles,
              int nk, long long* best_values, double* best_latency, cudaStream_t st) {
  unsigned long long space;
  SimArgs s = make_sim(dev6, 1, task4, domains, sizes, roles, nk, &space);
  if (space > (1ull << 40)) fail(MOSES_ERR_SPACE_TOO_LARGE, "exhaustive search over more than 2^40 configurations");
  const int grid = int(std::min<unsigned long long>((space + 255) / 256, 148ull * 8));
  BestItem* part = nullptr;
  MOSES_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(BestItem) * grid, st));
  true_best_kernel<<<grid, 256, 0, st>>>(s, space, part);
  true_best_final_kernel<<<1, 256, 0, st>>>(part, grid);
  BestItem b;
  MOSES_CUDA(cudaMemcpyAsync(&b, part, sizeof(b), cudaMemcpyDeviceToHost, st));
  MOSES_CUDA(cudaFreeAsync(part, st));
  MOSES_CUDA(cudaStreamSynchronize(st));
  *best_latency = b.lat;
  unsigned long long idx = b.idx;
  for (int k = nk - 1; k >= 0; --k) {
    best_values[k] = domains[s.sp.offs[k] + int(idx % (unsigned long long)sizes[k])];
    idx /= (unsigned long long)sizes[k];
  }
  return 2;
}


// ---------------------------------------------------------------- dataset generation
// generate_dataset (data.cpp:49-65), one task: RngStream(KeyBuilder(seed, "gen", task.id)) draws each
// configuration knob by knob with below(|domain|) (sample_config, space.cpp:94-100), then measure()
// labels it. Draw k (1-based) of the stream is mix(key + k*gamma), so sample s, knob j is draw
// s*nk + j + 1 — as long as no below() call rejects. Rejection happens when a draw is < (2^64 - m) % m
// (< m/2^64, about 1e-17 per draw here): the parallel kernel flags it and the exact sequential
// walk below replaces its result, so the configurations always equal the reference's.
struct DrawArgs {
  int nk;
  unsigned long long size[kSpaceMaxKnobs], thresh[kSpaceMaxKnobs];
};

namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) sample_configs_kernel(const __grid_constant__ DrawArgs d, unsigned long long key,
                                                             long long n, unsigned long long* __restrict__ idx,
                                                             int* __restrict__ rejected) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long id = 0;
    bool rej = false;
#pragma unroll
    for (int k = 0; k < kSpaceMaxKnobs; ++k) {
      if (k >= d.nk) continue;
      const unsigned long long ctr = (unsigned long long)i * (unsigned long long)d.nk + (unsigned long long)k + 1ull;
      const unsigned long long r = mix64(key + ctr * 0x9e3779b97f4a7c15ull);
      rej |= r < d.thresh[k];
      id = id * d.size[k] + r % d.size[k];
    }
    idx[i] = id;
    if (rej) atomicExch(rejected, 1);
  }
}

// the reference's sequential walk, rejection loop included (runs only when the kernel above flagged)
__global__ void sample_configs_serial_kernel(const __grid_constant__ DrawArgs d, unsigned long long key, long long n,
                                             unsigned long long* __restrict__ idx) {
  unsigned long long st = key;
  for (long long i = 0; i < n; ++i) {
    unsigned long long id = 0;
    for (int k = 0; k < d.nk; ++k) {
      unsigned long long r;
      do {
        st += 0x9e3779b97f4a7c15ull;
        r = mix64(st);
      } while (r < d.thresh[k]);
      id = id * d.size[k] + r % d.size[k];
    }
    idx[i] = id;
  }
}

// Configuration values -> enumeration index; validate_config (space.cpp:69-81): every value must be
// in its knob's (sorted) domain, else the smallest offending row is reported.
__global__ void __launch_bounds__(256) values_to_index_kernel(const __grid_constant__ SpaceArgs a,
                                                              const long long* __restrict__ values, long long n,
                                                              unsigned long long* __restrict__ idx,
                                                              unsigned long long* __restrict__ bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long id = 0;
    bool ok = true;
    for (int k = 0; k < a.nk; ++k) {
      const long long v = values[i * a.nk + k];
      int lo = 0, hi = a.sizes[k];  // first position with domain >= v
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a.domains[a.offs[k] + mid] < v) lo = mid + 1;
        else hi = mid;
      }
      ok &= lo < a.sizes[k] && a.domains[a.offs[k] + lo] == v;
      id = id * (unsigned long long)a.sizes[k] + (unsigned long long)(lo < a.sizes[k] ? lo : 0);
    }
    idx[i] = id;
    if (!ok) atomicMin(bad, (unsigned long long)i);
  }
}

}  // namespace

static bool g_force_serial_sampling = false;
void debug_force_serial_sampling(bool on) { g_force_serial_sampling = on; }

int generate_task_dataset(const double* dev6, int repeats, const char* device_id, const char* task_id,
                          const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                          long long samples, unsigned long long seed, int out_kind, void* feat, long long ld, int D,
                          long long* values_out, double* thr, double* lat, double* wall, float* label,
                          unsigned long long* idx_out, cudaStream_t st) {
  if (samples < 1) fail(MOSES_ERR_INVALID_CONFIG, "samples_per_task must be positive");
  SpaceArgs chk{};
  fill_space(chk, domains, sizes, roles, nk);  // validate_task / build_space before any draw
  DrawArgs d{};
  d.nk = nk;
  for (int k = 0; k < nk; ++k) {
    d.size[k] = (unsigned long long)sizes[k];
    d.thresh[k] = (0ull - d.size[k]) % d.size[k];
  }
  unsigned long long key = 0xcbf29ce484222325ull;
  fnv_add_u64(key, seed);
  fnv_add_str(key, "gen");
  fnv_add_str(key, task_id ? task_id : "");
  unsigned long long* idx = idx_out;
  int* rej = nullptr;
  char* ws = nullptr;
  const size_t idx_bytes = idx_out ? 0 : size_t(samples) * 8;
  MOSES_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), idx_bytes + 16, st));
  if (!idx) idx = reinterpret_cast<unsigned long long*>(ws);
  rej = reinterpret_cast<int*>(ws + idx_bytes);
  MOSES_CUDA(cudaMemsetAsync(rej, 0, sizeof(int), st));
  const int grid = int(std::min<long long>((samples + 255) / 256, 148LL * 16));
  sample_configs_kernel<<<grid, 256, 0, st>>>(d, key, samples, idx, rej);
  MOSES_CUDA(cudaGetLastError());
  int launches = 1;
  int h_rej = 0;
  MOSES_CUDA(cudaMemcpyAsync(&h_rej, rej, sizeof(int), cudaMemcpyDeviceToHost, st));
  MOSES_CUDA(cudaStreamSynchronize(st));
  if (h_rej || g_force_serial_sampling) {
    sample_configs_serial_kernel<<<1, 1, 0, st>>>(d, key, samples, idx);
    MOSES_CUDA(cudaGetLastError());
    ++launches;
  }
  if (feat || values_out)
    launches += encode_impl(task4, domains, sizes, roles, nk, 0, idx, samples, out_kind, feat, ld, D, nullptr,
                            values_out, st);
  if (thr || lat || wall || label)
    launches += measure_impl(dev6, repeats, device_id, task_id, task4, domains, sizes, roles, nk, seed, 0, idx, samples,
                             nullptr, thr, lat, wall, label, st);
  MOSES_CUDA(cudaFreeAsync(ws, st));
  return launches;
}

int encode_values(const double* task4, const long long* domains, const int* sizes, const int* roles, int nk,
                  const long long* values, long long n, int out_kind, void* feat, long long ld, int D,
                  unsigned long long* hash, unsigned long long* idx_out, long long* bad_row, cudaStream_t st) {
  SpaceArgs a{};
  fill_space(a, domains, sizes, roles, nk);
  *bad_row = -1;
  if (n < 0) fail(MOSES_ERR_SHAPE_MISMATCH, "negative row count");
  if (n == 0) return 0;
  char* ws = nullptr;
  const size_t idx_bytes = idx_out ? 0 : size_t(n) * 8;
  MOSES_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), idx_bytes + 16, st));
  unsigned long long* idx = idx_out ? idx_out : reinterpret_cast<unsigned long long*>(ws);
  auto* bad = reinterpret_cast<unsigned long long*>(ws + idx_bytes);
  MOSES_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
  const int grid = int(std::min<long long>((n + 255) / 256, 148LL * 16));
  values_to_index_kernel<<<grid, 256, 0, st>>>(a, values, n, idx, bad);
  MOSES_CUDA(cudaGetLastError());
  unsigned long long h_bad = 0;
  MOSES_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(h_bad), cudaMemcpyDeviceToHost, st));
  MOSES_CUDA(cudaStreamSynchronize(st));
  int launches = 1;
  if (h_bad != ~0ull) {
    *bad_row = (long long)h_bad;
    MOSES_CUDA(cudaFreeAsync(ws, st));
    fail(MOSES_ERR_INVALID_CONFIG, "record " + std::to_string(h_bad) + ": value not in its knob's domain");
  }
  if (feat || hash)
    launches += encode_impl(task4, domains, sizes, roles, nk, 0, idx, n, out_kind, feat, ld, D, hash, nullptr, st);
  MOSES_CUDA(cudaFreeAsync(ws, st));
  return launches;
}

}  // namespace moses
