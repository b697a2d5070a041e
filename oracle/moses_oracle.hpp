// moses_oracle.hpp — CPU ORACLE (test infrastructure only).
//
// A formula-for-formula C++20 restatement of the reference's cost-model hot
// path (moseslab, /root/reference/proj) used ONLY by tests/, by
// __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
// leg, as the checker and as the timed CPU baseline. It is never linked into
// the product library and never used as a fallback.
//
// Parity pinning: the reference cannot be built here (it needs Eigen3 and the
// vendored doctest/CLI11, none of which exist in the image).
// This restatement is therefore pinned against every known-answer test the
// reference ships for the path (tests/test_oracle_kat.py): the SplitMix64 /
// FNV-1a vectors (test_rng.cpp:14-72), the golden init+forward predictions
// (test_model.cpp:387-398, tests/golden/README.md:8-12), the ranking-loss hand
// cases (test_model.cpp:155-203), finite-difference gradients
// (test_model.cpp:225-256, acceptance.cpp:77-127), update arithmetic
// (test_model.cpp:267-326), the lottery suite incl. canonical ratio popcounts
// and tie-break (test_lottery.cpp:47-263), discriminator (:265-323) and the
// select_batch cases (test_search.cpp:161-187).
//
// Flat parameter order (lottery.hpp:13-14): per level, the weight array in
// Eigen column-major storage order — element (o,i) of the dims[l+1] x dims[l]
// matrix at off + i*out + o — then the bias. Viewed row-major that block is
// W^T, i.e. [in][out]; the device uses the identical flat layout.
//
// Everything is templated on the real type R so the same formulas run in fp64
// (reference precision) and in fp32 ("identical inputs in identical precision"
// for the bit-exact stages). Compiled with -ffp-contract=off like the
// reference (CMakeLists.txt:14-16); GEMMs use explicit FMA like Eigen does.
#pragma once

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#if defined(__AVX2__) && defined(__FMA__)
#include <immintrin.h>
#define ORACLE_AVX2 1
#endif

namespace oracle {

// ---------------------------------------------------------------- errors
// Ordinals follow moseslab::ErrorCode (errors.hpp:10-36).
enum class Err : int {
  InvalidTask = 0, InvalidConfig, SpaceTooLarge, ImmutableSpace, BadDims, DimMismatch,
  ShapeMismatch, VersionMismatch, CorruptStream, EmptyDataset, InvalidRatio,
  UnnormalizedThreshold, AdversaryDisabled, UnstableDecay, InfeasibleSplit, ZeroMean,
  InsufficientBatches, BudgetInfeasible, MissingReferenceStrategy, MismatchedRuns, EmptyRows,
  ParseError, MissingField, IoError, UsageError
};

struct Error : std::runtime_error {
  Err code;
  Error(Err c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(Err c, const std::string& m) { throw Error(c, m); }

// ---------------------------------------------------------------- rng (rng.hpp:16-80)
inline constexpr std::uint64_t kFnvOffset = 0xcbf29ce484222325ull;
inline constexpr std::uint64_t kFnvPrime = 0x100000001b3ull;

struct KeyBuilder {
  std::uint64_t h = kFnvOffset;
  void step(unsigned char b) { h ^= b; h *= kFnvPrime; }
  KeyBuilder& add(std::uint64_t v) {
    for (int i = 0; i < 8; ++i) step(static_cast<unsigned char>(v >> (8 * i)));
    return *this;
  }
  KeyBuilder& add(std::string_view s) {
    for (unsigned char c : s) step(c);
    step(0);
    return *this;
  }
  std::uint64_t value() const { return h; }
};

struct RngStream {
  std::uint64_t state;
  explicit RngStream(std::uint64_t s) : state(s) {}
  std::uint64_t next_u64() {
    state += 0x9e3779b97f4a7c15ull;
    std::uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  std::uint64_t below(std::uint64_t n) {
    const std::uint64_t threshold = (0 - n) % n;
    for (;;) {
      const std::uint64_t r = next_u64();
      if (r >= threshold) return r % n;
    }
  }
  double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double gaussian() {
    const double u1 = static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53;
    const double u2 = uniform01();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
  }
};

// Counter-based view of the same stream: draw k (1-based) of stream `key`.
// Identical to constructing RngStream(key) and calling next_u64() k times
// (rng.hpp:51-57), so any row of a synthetic set can be produced independently.
inline std::uint64_t splitmix_at(std::uint64_t key, std::uint64_t k) {
  std::uint64_t z = key + k * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline double u01_of(std::uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

// ---------------------------------------------------------------- model shape
inline void check_dims(const std::vector<int>& dims, bool strict) {
  // model.cpp:20-25. strict = the reference's exact 4-level rule; the
  // depth-generic extension (a17) accepts >= 3 levels ({D, h1..hL, 1}).
  if (strict ? dims.size() != 4 : dims.size() < 3)
    fail(Err::BadDims, "expected 4 levels, got " + std::to_string(dims.size()));
  for (int d : dims)
    if (d <= 0) fail(Err::BadDims, "non-positive level width");
  if (dims.back() != 1) fail(Err::BadDims, "output width must be 1");
}

inline std::int64_t level_offset(const std::vector<int>& dims, int l) {
  std::int64_t off = 0;
  for (int k = 0; k < l; ++k) off += std::int64_t(dims[k]) * dims[k + 1] + dims[k + 1];
  return off;
}
inline std::int64_t param_count(const std::vector<int>& dims) {  // model.cpp:141-145
  return level_offset(dims, int(dims.size()) - 1);
}

template <class R>
struct Params {
  std::vector<int> dims;
  std::vector<R> w;    // flat θ (weights+biases, reference flat order)
  std::vector<R> mom;  // flat momentum, same order (mw/mb)
  int levels() const { return int(dims.size()) - 1; }
  R* W(int l) { return w.data() + level_offset(dims, l); }
  const R* W(int l) const { return w.data() + level_offset(dims, l); }
  R* B(int l) { return W(l) + std::int64_t(dims[l]) * dims[l + 1]; }
  const R* B(int l) const { return W(l) + std::int64_t(dims[l]) * dims[l + 1]; }
};

// model.cpp:147-167: per level stream KeyBuilder(seed,"init",l); weights in
// column-major storage order = flat order; biases and momentum zero.
inline Params<double> init_random(const std::vector<int>& dims, std::uint64_t seed, bool strict = true) {
  check_dims(dims, strict);
  Params<double> p;
  p.dims = dims;
  const std::int64_t P = param_count(dims);
  p.w.assign(P, 0.0);
  p.mom.assign(P, 0.0);
  for (int l = 0; l + 1 < int(dims.size()); ++l) {
    const int fan_in = dims[l], fan_out = dims[l + 1];
    const double bound = std::sqrt(6.0 / static_cast<double>(fan_in + fan_out));
    KeyBuilder key;
    key.add(seed).add("init").add(static_cast<std::uint64_t>(l));
    RngStream rng(key.value());
    double* data = p.W(l);
    const std::int64_t cnt = std::int64_t(fan_in) * fan_out;
    for (std::int64_t i = 0; i < cnt; ++i) data[i] = (2.0 * rng.uniform01() - 1.0) * bound;
  }
  return p;
}

template <class R, class S>
Params<R> cast_params(const Params<S>& p) {
  Params<R> q;
  q.dims = p.dims;
  q.w.assign(p.w.begin(), p.w.end());
  q.mom.assign(p.mom.begin(), p.mom.end());
  return q;
}

// ---------------------------------------------------------------- dense kernels
// C[M][N] (row-major) = A * B with general strides: A(m,k) = A[m*sam + k*sak],
// B(k,n) = B[k*sbk + n*sbn]. Parallel over M; B is packed into 16-column panels.
template <class R>
void gemm_general(int M, int N, int K, const R* A, std::int64_t sam, std::int64_t sak, const R* B, std::int64_t sbk,
                  std::int64_t sbn, R* C, int threads) {
#if defined(ORACLE_AVX2)
  if constexpr (std::is_same_v<R, double>) {
    // Register-blocked 4 x 16 micro-kernel (explicit FMA, as Eigen's GEBP does), full tiles fully
    // unrolled so the 16 accumulators stay in ymm registers; edges fall back to scalar FMA.
    const int Nv = N & ~15;
    const int Mv = M & ~3;
    std::vector<double> Bp(std::size_t(K) * Nv);
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
    for (int n0 = 0; n0 < Nv; n0 += 16)
      for (int k = 0; k < K; ++k) {
        double* dst = &Bp[std::size_t(n0) * K + std::size_t(k) * 16];
        const double* src = B + std::int64_t(k) * sbk + std::int64_t(n0) * sbn;
        if (sbn == 1) std::memcpy(dst, src, 16 * sizeof(double));
        else
          for (int j = 0; j < 16; ++j) dst[j] = src[j * sbn];
      }
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
    for (int m0 = 0; m0 < M; m0 += 4) {
      if (m0 < Mv) {
        const double* a0 = A + std::int64_t(m0) * sam;
        const double* a1 = a0 + sam;
        const double* a2 = a1 + sam;
        const double* a3 = a2 + sam;
        for (int n0 = 0; n0 < Nv; n0 += 16) {
          __m256d c00 = _mm256_setzero_pd(), c01 = c00, c02 = c00, c03 = c00;
          __m256d c10 = c00, c11 = c00, c12 = c00, c13 = c00;
          __m256d c20 = c00, c21 = c00, c22 = c00, c23 = c00;
          __m256d c30 = c00, c31 = c00, c32 = c00, c33 = c00;
          const double* b = Bp.data() + std::size_t(n0) * K;
          for (int k = 0; k < K; ++k, b += 16) {
            const std::int64_t ko = std::int64_t(k) * sak;
            const __m256d b0 = _mm256_loadu_pd(b), b1 = _mm256_loadu_pd(b + 4), b2 = _mm256_loadu_pd(b + 8),
                          b3 = _mm256_loadu_pd(b + 12);
            __m256d a = _mm256_broadcast_sd(a0 + ko);
            c00 = _mm256_fmadd_pd(a, b0, c00); c01 = _mm256_fmadd_pd(a, b1, c01);
            c02 = _mm256_fmadd_pd(a, b2, c02); c03 = _mm256_fmadd_pd(a, b3, c03);
            a = _mm256_broadcast_sd(a1 + ko);
            c10 = _mm256_fmadd_pd(a, b0, c10); c11 = _mm256_fmadd_pd(a, b1, c11);
            c12 = _mm256_fmadd_pd(a, b2, c12); c13 = _mm256_fmadd_pd(a, b3, c13);
            a = _mm256_broadcast_sd(a2 + ko);
            c20 = _mm256_fmadd_pd(a, b0, c20); c21 = _mm256_fmadd_pd(a, b1, c21);
            c22 = _mm256_fmadd_pd(a, b2, c22); c23 = _mm256_fmadd_pd(a, b3, c23);
            a = _mm256_broadcast_sd(a3 + ko);
            c30 = _mm256_fmadd_pd(a, b0, c30); c31 = _mm256_fmadd_pd(a, b1, c31);
            c32 = _mm256_fmadd_pd(a, b2, c32); c33 = _mm256_fmadd_pd(a, b3, c33);
          }
          double* c = C + std::int64_t(m0) * N + n0;
          _mm256_storeu_pd(c, c00); _mm256_storeu_pd(c + 4, c01); _mm256_storeu_pd(c + 8, c02); _mm256_storeu_pd(c + 12, c03);
          c += N;
          _mm256_storeu_pd(c, c10); _mm256_storeu_pd(c + 4, c11); _mm256_storeu_pd(c + 8, c12); _mm256_storeu_pd(c + 12, c13);
          c += N;
          _mm256_storeu_pd(c, c20); _mm256_storeu_pd(c + 4, c21); _mm256_storeu_pd(c + 8, c22); _mm256_storeu_pd(c + 12, c23);
          c += N;
          _mm256_storeu_pd(c, c30); _mm256_storeu_pd(c + 4, c31); _mm256_storeu_pd(c + 8, c32); _mm256_storeu_pd(c + 12, c33);
        }
      }
      const int r0 = m0 < Mv ? 4 : 0;
      const int mr = std::min(4, M - m0);
      for (int r = 0; r < mr; ++r) {
        double* c = C + std::int64_t(m0 + r) * N;
        const int nlo = r < r0 ? Nv : 0;  // full 4-row tiles already covered [0, Nv)
        for (int n = nlo; n < N; ++n) {
          double acc = 0.0;
          for (int k = 0; k < K; ++k)
            acc = std::fma(A[std::int64_t(m0 + r) * sam + std::int64_t(k) * sak], B[std::int64_t(k) * sbk + std::int64_t(n) * sbn], acc);
          c[n] = acc;
        }
      }
    }
    return;
  }
#endif
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
  for (int m = 0; m < M; ++m) {
    R* c = C + std::int64_t(m) * N;
    for (int n = 0; n < N; ++n) c[n] = R(0);
    for (int k = 0; k < K; ++k) {
      const R a = A[std::int64_t(m) * sam + std::int64_t(k) * sak];
      for (int n = 0; n < N; ++n) c[n] = std::fma(a, B[std::int64_t(k) * sbk + std::int64_t(n) * sbn], c[n]);
    }
  }
}

// C[M][N] = A[M][K] * B[K][N], all row-major.
template <class R>
void gemm_nn(int M, int N, int K, const R* A, const R* B, R* C, int threads) {
  gemm_general<R>(M, N, K, A, K, 1, B, N, 1, C, threads);
}

template <class R>
std::vector<R> transpose(const R* A, int rows, int cols) {
  std::vector<R> T(std::size_t(rows) * cols);
  constexpr int kB = 32;  // cache-blocked
  for (int r0 = 0; r0 < rows; r0 += kB)
    for (int c0 = 0; c0 < cols; c0 += kB)
      for (int r = r0; r < std::min(rows, r0 + kB); ++r)
        for (int c = c0; c < std::min(cols, c0 + kB); ++c) T[std::size_t(c) * rows + r] = A[std::size_t(r) * cols + c];
  return T;
}

template <class R>
void segment_sum(const R* h, int width, const std::int64_t* offsets, std::int64_t programs, R* out);

// ---------------------------------------------------------------- forward (model.cpp:54-62)
template <class R>
struct Forward {
  std::vector<std::vector<R>> z, h;  // z[l], h[l] for hidden level l+1 (l = 0..L-2), n x width
  std::vector<R> s;                   // n
};

template <class R>
Forward<R> run_forward(const Params<R>& p, const R* x, int n, int threads = 1) {
  const int L = p.levels();
  Forward<R> f;
  const R* in = x;
  for (int l = 0; l + 1 < L; ++l) {
    const int di = p.dims[l], dout = p.dims[l + 1];
    std::vector<R> z(std::size_t(n) * dout);
    gemm_nn<R>(n, dout, di, in, p.W(l), z.data(), threads);  // X * W^T (flat block is W^T)
    const R* b = p.B(l);
    for (int r = 0; r < n; ++r)
      for (int o = 0; o < dout; ++o) z[std::size_t(r) * dout + o] += b[o];  // .rowwise() + b^T
    std::vector<R> h(z.size());
    for (std::size_t i = 0; i < z.size(); ++i) h[i] = std::max(z[i], R(0));  // cwiseMax(0)
    f.z.push_back(std::move(z));
    f.h.push_back(std::move(h));
    in = f.h.back().data();
  }
  const int dl = p.dims[L - 1];
  const R* wh = p.W(L - 1);
  const R bh = p.B(L - 1)[0];
  f.s.assign(n, R(0));
  for (int r = 0; r < n; ++r) {
    R acc = R(0);
    const R* hr = in + std::size_t(r) * dl;
    for (int i = 0; i < dl; ++i) acc = std::fma(hr[i], wh[i], acc);
    f.s[r] = acc + bh;
  }
  return f;
}

template <class R>
R stable_sigmoid(R x) {  // model.cpp:64-68
  if (x >= R(0)) return R(1) / (R(1) + std::exp(-x));
  const R e = std::exp(x);
  return e / (R(1) + e);
}

// model.cpp:71-106, restated loop for loop.
template <class R>
std::int64_t ranking_terms(const R* scores, const R* labels, int n, R* loss_out, R* gs_out) {
  std::int64_t pairs = 0;
  R loss = R(0);
  std::vector<R> gs(n, R(0));
  for (int i = 0; i < n; ++i) {
    for (int j = i + 1; j < n; ++j) {
      int hi, lo;
      if (labels[i] > labels[j]) { hi = i; lo = j; }
      else if (labels[j] > labels[i]) { hi = j; lo = i; }
      else continue;
      const R d = scores[hi] - scores[lo];
      const R e = std::exp(-std::abs(d));
      ++pairs;
      if (loss_out != nullptr) loss += d >= R(0) ? std::log1p(e) : -d + std::log1p(e);
      if (gs_out != nullptr) {
        const R sig_neg = d >= R(0) ? e / (R(1) + e) : R(1) / (R(1) + e);
        gs[hi] -= sig_neg;
        gs[lo] += sig_neg;
      }
    }
  }
  if (pairs > 0) {
    loss /= static_cast<R>(pairs);
    for (auto& v : gs) v /= static_cast<R>(pairs);
  }
  if (loss_out != nullptr) *loss_out = loss;
  if (gs_out != nullptr) std::copy(gs.begin(), gs.end(), gs_out);
  return pairs;
}

// lottery.cpp:207-218
template <class R>
R discriminator_cross_entropy(const R* zs, int m, const R* zt, int n) {
  const auto softplus = [](R v) { return std::max(v, R(0)) + std::log1p(std::exp(-std::abs(v))); };
  R ls = R(0);
  for (int i = 0; i < m; ++i) ls += softplus(-zs[i]);
  R lt = R(0);
  for (int j = 0; j < n; ++j) lt += softplus(zt[j]);
  return R(0.5) * (ls / static_cast<R>(m) + lt / static_cast<R>(n));
}

template <class R>
struct Adversary {  // lottery.hpp:36-42
  std::vector<R> weight;  // penultimate width
  R bias = R(0);
  std::vector<R> replay;  // m x D row-major
  int m = 0;
  R step_size = R(0.1);
};

// model.cpp:110-120 generalised to depth: levels L-2 .. 0.
template <class R>
void backprop_from_penultimate(const Params<R>& p, const Forward<R>& f, const R* x, int n,
                               std::vector<R> dh, std::vector<R>& g, int threads) {
  const int L = p.levels();
  for (int l = L - 2; l >= 0; --l) {
    const int di = p.dims[l], dout = p.dims[l + 1];
    const std::vector<R>& z = f.z[l];
    std::vector<R> dz(std::size_t(n) * dout);
    for (std::size_t i = 0; i < dz.size(); ++i) dz[i] = dh[i] * (z[i] > R(0) ? R(1) : R(0));
    const R* in = l == 0 ? x : f.h[l - 1].data();
    // gW (flat [in][out]) += in^T * dz ; gb += colsum(dz)
    std::vector<R> gw(std::size_t(di) * dout);
    gemm_general<R>(di, dout, n, in, 1, di, dz.data(), dout, 1, gw.data(), threads);  // in^T * dz
    R* G = g.data() + level_offset(p.dims, l);
    for (std::size_t i = 0; i < gw.size(); ++i) G[i] += gw[i];
    std::vector<R> gb(dout, R(0));
    for (int r = 0; r < n; ++r)
      for (int o = 0; o < dout; ++o) gb[o] += dz[std::size_t(r) * dout + o];
    R* GB = G + std::size_t(di) * dout;
    for (int o = 0; o < dout; ++o) GB[o] += gb[o];
    if (l > 0) {
      // dh_prev = dz * W  (W is out x in; flat block is [in][out] = W^T)
      std::vector<R> nd(std::size_t(n) * di);
      gemm_general<R>(n, di, dout, dz.data(), dout, 1, p.W(l), 1, dout, nd.data(), threads);  // dz * W
      dh = std::move(nd);
    }
  }
}

template <class R>
void check_adversary(const Params<R>& p, const Adversary<R>& adv) {  // model.cpp:130-137
  const int L = p.levels();
  if (int(adv.weight.size()) != p.dims[L - 1]) fail(Err::DimMismatch, "discriminator width != penultimate width");
  if (adv.m == 0) fail(Err::AdversaryDisabled, "adversary has an empty replay buffer");
  if (int(adv.replay.size()) != adv.m * p.dims[0]) fail(Err::DimMismatch, "replay feature width != model input width");
}

template <class R>
std::vector<R> logits(const std::vector<R>& h, int rows, int width, const Adversary<R>& adv) {
  std::vector<R> z(rows);
  for (int r = 0; r < rows; ++r) {
    R acc = R(0);
    for (int j = 0; j < width; ++j) acc = std::fma(h[std::size_t(r) * width + j], adv.weight[j], acc);
    z[r] = acc + adv.bias;
  }
  return z;
}

// model.cpp:192-244
template <class R>
std::vector<R> gradients(const Params<R>& p, const R* x, const R* y, int n, const Adversary<R>* adv,
                         R beta, R* loss_out, int threads = 1) {
  const int L = p.levels();
  const int dl = p.dims[L - 1];
  std::vector<R> g(p.w.size(), R(0));
  const Forward<R> f = run_forward(p, x, n, threads);
  R rank_loss = R(0);
  std::vector<R> gs(n);
  ranking_terms(f.s.data(), y, n, loss_out != nullptr ? &rank_loss : nullptr, gs.data());
  const std::vector<R>& hl = L >= 2 ? f.h.back() : f.h.back();
  // g.gw[L-1] = gs^T * h ; g.gb = sum(gs)
  R* GW = g.data() + level_offset(p.dims, L - 1);
  for (int j = 0; j < dl; ++j) {
    R acc = R(0);
    for (int r = 0; r < n; ++r) acc = std::fma(gs[r], hl[std::size_t(r) * dl + j], acc);
    GW[j] = acc;
  }
  R gsum = R(0);
  for (int r = 0; r < n; ++r) gsum += gs[r];
  GW[dl] = gsum;
  const R* wh = p.W(L - 1);
  std::vector<R> dh(std::size_t(n) * dl);
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < dl; ++j) dh[std::size_t(r) * dl + j] = gs[r] * wh[j];
  R total_loss = rank_loss;
  if (adv != nullptr && beta != R(0) && n > 0) {
    check_adversary(p, *adv);
    const int m = adv->m;
    const Forward<R> fs = run_forward(p, adv->replay.data(), m, threads);
    const std::vector<R> zs = logits(fs.h.back(), m, dl, *adv);
    const std::vector<R> zt = logits(hl, n, dl, *adv);
    std::vector<R> dzs(m), dzt(n);
    for (int i = 0; i < m; ++i) dzs[i] = R(0.5) * beta * stable_sigmoid(-zs[i]) / static_cast<R>(m);
    for (int j = 0; j < n; ++j) dzt[j] = R(-0.5) * beta * stable_sigmoid(zt[j]) / static_cast<R>(n);
    for (int r = 0; r < n; ++r)
      for (int j = 0; j < dl; ++j) dh[std::size_t(r) * dl + j] += dzt[r] * adv->weight[j];
    std::vector<R> dhs(std::size_t(m) * dl);
    for (int r = 0; r < m; ++r)
      for (int j = 0; j < dl; ++j) dhs[std::size_t(r) * dl + j] = dzs[r] * adv->weight[j];
    backprop_from_penultimate(p, fs, adv->replay.data(), m, std::move(dhs), g, threads);
    if (loss_out != nullptr) total_loss += beta * -discriminator_cross_entropy(zs.data(), m, zt.data(), n);
  }
  backprop_from_penultimate(p, f, x, n, std::move(dh), g, threads);
  if (loss_out != nullptr) *loss_out = total_loss;
  return g;
}

// gradients() (model.cpp:201-244, no adversary) with the score gradient gs supplied by the caller:
// g.gw[L-1] = gs^T h, g.gb[L-1] = sum(gs), then backprop_from_penultimate. With gs = ranking_terms'
// this is gradients(); with the rows of one data-parallel rank and gs from the pair terms of those rows
// against the whole (all-gathered) batch, normalised by the global pair count, it is that rank's
// share of the global batch gradient (SURVEY.md §8(e) exact mode): the shares sum to gradients().
template <class R>
std::vector<R> gradients_from_score_grads(const Params<R>& p, const R* x, int n, const R* gs, int threads = 1) {
  const int L = p.levels();
  const int dl = p.dims[L - 1];
  std::vector<R> g(p.w.size(), R(0));
  const Forward<R> f = run_forward(p, x, n, threads);
  const std::vector<R>& hl = f.h.back();
  R* GW = g.data() + level_offset(p.dims, L - 1);
  for (int j = 0; j < dl; ++j) {
    R acc = R(0);
    for (int r = 0; r < n; ++r) acc = std::fma(gs[r], hl[std::size_t(r) * dl + j], acc);
    GW[j] = acc;
  }
  R gsum = R(0);
  for (int r = 0; r < n; ++r) gsum += gs[r];
  GW[dl] = gsum;
  const R* wh = p.W(L - 1);
  std::vector<R> dh(std::size_t(n) * dl);
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < dl; ++j) dh[std::size_t(r) * dl + j] = gs[r] * wh[j];
  backprop_from_penultimate(p, f, x, n, std::move(dh), g, threads);
  return g;
}

// North-star extension (parity pinned only by this restatement; S == 1 reduces to gradients()):
// statement rows -> shared encoder -> per-program segment sum of the last hidden layer -> head.
template <class R>
std::vector<R> gradients_pooled(const Params<R>& p, const R* x, int nstmt, const std::int64_t* off, int programs,
                                const R* y, R* loss_out, int threads = 1) {
  const int L = p.levels();
  const int dl = p.dims[L - 1];
  std::vector<R> g(p.w.size(), R(0));
  const Forward<R> f = run_forward(p, x, nstmt, threads);
  const std::vector<R>& hl = f.h.back();
  std::vector<R> pooled(std::size_t(programs) * dl, R(0));
  segment_sum(hl.data(), dl, off, programs, pooled.data());
  const R* wh = p.W(L - 1);
  const R bh = p.B(L - 1)[0];
  std::vector<R> s(programs);
  for (int q = 0; q < programs; ++q) {
    R acc = R(0);
    for (int j = 0; j < dl; ++j) acc = std::fma(pooled[std::size_t(q) * dl + j], wh[j], acc);
    s[q] = acc + bh;
  }
  R loss = R(0);
  std::vector<R> gs(programs);
  ranking_terms(s.data(), y, programs, loss_out ? &loss : nullptr, gs.data());
  R* GW = g.data() + level_offset(p.dims, L - 1);
  for (int j = 0; j < dl; ++j) {
    R acc = R(0);
    for (int q = 0; q < programs; ++q) acc = std::fma(gs[q], pooled[std::size_t(q) * dl + j], acc);
    GW[j] = acc;
  }
  R gsum = R(0);
  for (int q = 0; q < programs; ++q) gsum += gs[q];
  GW[dl] = gsum;
  std::vector<R> dh(std::size_t(nstmt) * dl);
  for (int q = 0; q < programs; ++q)
    for (std::int64_t i = off[q]; i < off[q + 1]; ++i)
      for (int j = 0; j < dl; ++j) dh[std::size_t(i) * dl + j] = gs[q] * wh[j];
  backprop_from_penultimate(p, f, x, nstmt, std::move(dh), g, threads);
  if (loss_out) *loss_out = loss;
  return g;
}

// model.cpp:246-261
template <class R>
R objective(const Params<R>& p, const R* x, const R* y, int n, const Adversary<R>* adv, R beta) {
  const Forward<R> f = run_forward(p, x, n);
  R loss = R(0);
  ranking_terms(f.s.data(), y, n, &loss, static_cast<R*>(nullptr));
  if (adv != nullptr && beta != R(0) && n > 0) {
    check_adversary(p, *adv);
    const int dl = p.dims[p.levels() - 1];
    const Forward<R> fs = run_forward(p, adv->replay.data(), adv->m);
    const std::vector<R> zs = logits(fs.h.back(), adv->m, dl, *adv);
    const std::vector<R> zt = logits(f.h.back(), n, dl, *adv);
    loss += beta * -discriminator_cross_entropy(zs.data(), adv->m, zt.data(), n);
  }
  return loss;
}

// model.cpp:263-296 — one code path for masked and unmasked scalars.
template <class R>
void apply_update(Params<R>& p, const R* g, double lr_d, double mu_d, const std::uint8_t* keep,
                  bool use_momentum) {
  const R lr = static_cast<R>(lr_d);
  const R mu = static_cast<R>(mu_d);
  const std::int64_t P = std::int64_t(p.w.size());
  R* w = p.w.data();
  R* v = p.mom.data();
  for (std::int64_t i = 0; i < P; ++i) {
    if (keep != nullptr && !keep[i]) continue;
    if (use_momentum) {
      v[i] = mu * v[i] + g[i];
      const R delta = lr * v[i];
      w[i] -= delta;
    } else {
      const R delta = lr * g[i];
      w[i] -= delta;
    }
  }
}

// model.cpp:298-312 — integer counts; returns concordant/pairs.
template <class R>
void accuracy_counts(const R* scores, const R* labels, int n, std::int64_t* pairs, std::int64_t* concordant) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (labels[i] <= labels[j]) continue;
      ++*pairs;
      if (scores[i] > scores[j]) ++*concordant;
    }
}

// ---------------------------------------------------------------- lottery (lottery.cpp:35-120)
template <class R>
std::vector<R> xi_scores(const R* w, const R* g, std::int64_t P, bool normalize) {
  std::vector<R> xi(P);
  for (std::int64_t i = 0; i < P; ++i) xi[i] = std::abs(w[i] * g[i]);
  if (normalize) {
    R top = xi.empty() ? R(0) : *std::max_element(xi.begin(), xi.end());
    if (top > R(0))
      for (auto& v : xi) v /= top;
  }
  return xi;
}

enum class Mode : int { Threshold = 1, Ratio = 2 };  // "MOSK" mode byte (lottery.cpp:195,223-224)

// lottery.cpp:59-90
template <class R>
std::vector<std::uint8_t> partition(const R* xi, std::int64_t n, bool normalized, Mode mode, double value) {
  if (n == 0) fail(Err::ShapeMismatch, "empty score array");
  std::vector<std::uint8_t> mask(n, 0);
  if (mode == Mode::Threshold) {
    if (!normalized) fail(Err::UnnormalizedThreshold, "threshold partition needs normalized scores");
    const R thr = static_cast<R>(value);
    for (std::int64_t i = 0; i < n; ++i) mask[i] = xi[i] > thr;
    return mask;
  }
  if (!(value > 0.0) || value > 1.0) fail(Err::InvalidRatio, "ratio must lie in (0,1]");
  const auto keep = static_cast<std::int64_t>(std::ceil(value * static_cast<double>(n)));
  if (keep >= n) {
    std::fill(mask.begin(), mask.end(), 1);
    return mask;
  }
  std::vector<std::int64_t> order(n);
  std::iota(order.begin(), order.end(), std::int64_t{0});
  std::nth_element(order.begin(), order.begin() + keep, order.end(), [&](std::int64_t a, std::int64_t b) {
    if (xi[a] != xi[b]) return xi[a] > xi[b];
    return a < b;
  });
  for (std::int64_t i = 0; i < keep; ++i) mask[order[i]] = 1;
  return mask;
}

inline std::int64_t ratio_keep(double value, std::int64_t n) {
  return static_cast<std::int64_t>(std::ceil(value * static_cast<double>(n)));
}

// lottery.cpp:99-120
template <class R>
void variant_decay(R* w, std::int64_t P, const std::uint8_t* keep, double alpha, double lambda) {
  const double rate = alpha * lambda;
  if (!(rate >= 0.0) || rate >= 1.0) fail(Err::UnstableDecay, "decay rate alpha*lambda must lie in [0,1)");
  if (rate == 0.0) return;
  const R factor = static_cast<R>(1.0 - rate);
  for (std::int64_t i = 0; i < P; ++i)
    if (!keep[i]) w[i] *= factor;
}

// lottery.cpp:135-164
template <class R>
R adversarial_term(Adversary<R>& adv, const R* hs, int m, const R* ht, int n, int width) {
  if (adv.m == 0) fail(Err::AdversaryDisabled, "adversary has an empty replay buffer");
  if (m == 0 || n == 0) fail(Err::AdversaryDisabled, "empty activation batch");
  if (width != int(adv.weight.size())) fail(Err::DimMismatch, "activation width != discriminator width");
  std::vector<R> hsv(hs, hs + std::size_t(m) * width), htv(ht, ht + std::size_t(n) * width);
  const std::vector<R> zs = logits(hsv, m, width, adv);
  const std::vector<R> zt = logits(htv, n, width, adv);
  const R loss = discriminator_cross_entropy(zs.data(), m, zt.data(), n);
  std::vector<R> dzs(m), dzt(n);
  for (int i = 0; i < m; ++i) dzs[i] = R(-0.5) * stable_sigmoid(-zs[i]) / static_cast<R>(m);
  for (int j = 0; j < n; ++j) dzt[j] = R(0.5) * stable_sigmoid(zt[j]) / static_cast<R>(n);
  std::vector<R> du(width, R(0));
  for (int j = 0; j < width; ++j) {
    R a = R(0), b = R(0);
    for (int i = 0; i < m; ++i) a = std::fma(hs[std::size_t(i) * width + j], dzs[i], a);
    for (int i = 0; i < n; ++i) b = std::fma(ht[std::size_t(i) * width + j], dzt[i], b);
    du[j] = a + b;
  }
  R sdzs = R(0), sdzt = R(0);
  for (int i = 0; i < m; ++i) sdzs += dzs[i];
  for (int j = 0; j < n; ++j) sdzt += dzt[j];
  const R dc = sdzs + sdzt;
  for (int j = 0; j < width; ++j) adv.weight[j] -= adv.step_size * du[j];
  adv.bias -= adv.step_size * dc;
  return loss;
}

// ---------------------------------------------------------------- search (search.cpp:32-37,82-95)
// Candidate-pool order: score desc, then pool index asc (the pool index is the
// lexicographic config order when the pool is an enumeration, space.cpp:168-191).
template <class R>
std::vector<std::int64_t> topk(const R* scores, std::int64_t n, std::int64_t k) {
  std::vector<std::int64_t> idx(n);
  std::iota(idx.begin(), idx.end(), std::int64_t{0});
  k = std::min(k, n);
  const auto cmp = [&](std::int64_t a, std::int64_t b) {
    if (scores[a] != scores[b]) return scores[a] > scores[b];
    return a < b;
  };
  std::partial_sort(idx.begin(), idx.begin() + k, idx.end(), cmp);
  idx.resize(k);
  return idx;
}

// ---------------------------------------------------------------- extensions (north star; parity unpinned by reference)
// Segment-sum pooling over CSR offsets: pooled[p] = sum_{i in [off[p],off[p+1])} h[i].
template <class R>
void segment_sum(const R* h, int width, const std::int64_t* offsets, std::int64_t programs, R* out) {
  for (std::int64_t p = 0; p < programs; ++p) {
    for (int j = 0; j < width; ++j) {
      R acc = R(0);
      for (std::int64_t i = offsets[p]; i < offsets[p + 1]; ++i) acc += h[i * width + j];
      out[p * width + j] = acc;
    }
  }
}

// Biased MMD^2 with a Gaussian kernel k(a,b) = exp(-|a-b|^2 / (2 sigma^2)).
template <class R>
R mmd2(const R* xs, int m, const R* xt, int n, int width, R sigma) {
  const R inv = R(1) / (R(2) * sigma * sigma);
  auto kern = [&](const R* a, const R* b) {
    R d = R(0);
    for (int j = 0; j < width; ++j) { const R t = a[j] - b[j]; d += t * t; }
    return std::exp(-d * inv);
  };
  R ss = 0, tt = 0, st = 0;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) ss += kern(xs + std::size_t(i) * width, xs + std::size_t(j) * width);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) tt += kern(xt + std::size_t(i) * width, xt + std::size_t(j) * width);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) st += kern(xs + std::size_t(i) * width, xt + std::size_t(j) * width);
  return ss / (R(m) * R(m)) + tt / (R(n) * R(n)) - R(2) * st / (R(m) * R(n));
}

// d MMD^2 / d row for the biased estimator above: with alpha = 1/m (source), -1/n (target),
// MMD^2 = sum_a alpha_a r_a, r_a = sum_b alpha_b k_ab and d/dx_a = -4c alpha_a (x_a r_a - sum_b alpha_b k_ab x_b),
// c = 1/(2 sigma^2) (k = exp(-c |a-b|^2), dk/da = -2c (a - b) k). Returns MMD^2.
template <class R>
R mmd2_grad(const R* xs, int m, const R* xt, int n, int width, R sigma, R* gs, R* gt) {
  const R c = R(1) / (R(2) * sigma * sigma);
  const int rows = m + n;
  auto row = [&](int a) { return a < m ? xs + std::size_t(a) * width : xt + std::size_t(a - m) * width; };
  auto alpha = [&](int a) { return a < m ? R(1) / R(m) : R(-1) / R(n); };
  R value = R(0);
  std::vector<R> o(width);
  for (int a = 0; a < rows; ++a) {
    const R* xa = row(a);
    std::fill(o.begin(), o.end(), R(0));
    R r = R(0);
    for (int b = 0; b < rows; ++b) {
      const R* xb = row(b);
      R d = R(0);
      for (int j = 0; j < width; ++j) { const R t = xa[j] - xb[j]; d += t * t; }
      const R wk = alpha(b) * std::exp(-c * d);
      r += wk;
      for (int j = 0; j < width; ++j) o[j] += wk * xb[j];
    }
    value += alpha(a) * r;
    R* g = a < m ? gs + std::size_t(a) * width : gt + std::size_t(a - m) * width;
    for (int j = 0; j < width; ++j) g[j] = R(-4) * c * alpha(a) * (xa[j] * r - o[j]);
  }
  return value;
}

// gradients() (model.cpp:192-244) with beta * MMD^2(H_source, H_batch) of the last hidden layer as the
// domain term (north-star (4); the reference's discriminator slot, model.cpp:215-238): the source rows
// (ms x D) are forwarded, the MMD gradient enters dH of the batch rows (next to gs * w_head) and of the
// source rows; source rows backprop first, then the batch (model.cpp:235,240).
template <class R>
std::vector<R> gradients_mmd(const Params<R>& p, const R* x, const R* y, int n, const R* src, int ms, R beta, R sigma,
                             R* loss_out, int threads = 1) {
  if (beta == R(0) || n == 0) return gradients(p, x, y, n, static_cast<const Adversary<R>*>(nullptr), R(0), loss_out,
                                               threads);
  const int L = p.levels();
  const int dl = p.dims[L - 1];
  std::vector<R> g(p.w.size(), R(0));
  const Forward<R> f = run_forward(p, x, n, threads);
  const Forward<R> fs = run_forward(p, src, ms, threads);
  R rank_loss = R(0);
  std::vector<R> gs(n);
  ranking_terms(f.s.data(), y, n, &rank_loss, gs.data());
  const std::vector<R>& hl = f.h.back();
  R* GW = g.data() + level_offset(p.dims, L - 1);
  for (int j = 0; j < dl; ++j) {
    R acc = R(0);
    for (int r = 0; r < n; ++r) acc = std::fma(gs[r], hl[std::size_t(r) * dl + j], acc);
    GW[j] = acc;
  }
  R gsum = R(0);
  for (int r = 0; r < n; ++r) gsum += gs[r];
  GW[dl] = gsum;
  std::vector<R> gms(std::size_t(ms) * dl), gmt(std::size_t(n) * dl);
  const R mmd = mmd2_grad(fs.h.back().data(), ms, hl.data(), n, dl, sigma, gms.data(), gmt.data());
  const R* wh = p.W(L - 1);
  std::vector<R> dh(std::size_t(n) * dl);
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < dl; ++j) dh[std::size_t(r) * dl + j] = gs[r] * wh[j] + beta * gmt[std::size_t(r) * dl + j];
  std::vector<R> dhs(std::size_t(ms) * dl);
  for (std::size_t i = 0; i < dhs.size(); ++i) dhs[i] = beta * gms[i];
  backprop_from_penultimate(p, fs, src, ms, std::move(dhs), g, threads);
  backprop_from_penultimate(p, f, x, n, std::move(dh), g, threads);
  if (loss_out != nullptr) *loss_out = rank_loss + beta * mmd;
  return g;
}

// Masked Adam (bias-corrected), same skip rule as apply_update.
template <class R>
void adam_update(R* w, R* m1, R* m2, const R* g, std::int64_t P, const std::uint8_t* keep, double lr,
                 double b1, double b2, double eps, int t) {
  const R c1 = static_cast<R>(1.0 - std::pow(b1, t));
  const R c2 = static_cast<R>(1.0 - std::pow(b2, t));
  const R B1 = static_cast<R>(b1), B2 = static_cast<R>(b2), LR = static_cast<R>(lr), EPS = static_cast<R>(eps);
  for (std::int64_t i = 0; i < P; ++i) {
    if (keep != nullptr && !keep[i]) continue;
    m1[i] = B1 * m1[i] + (R(1) - B1) * g[i];
    m2[i] = B2 * m2[i] + (R(1) - B2) * (g[i] * g[i]);
    const R mh = m1[i] / c1;
    const R vh = m2[i] / c2;
    w[i] -= LR * mh / (std::sqrt(vh) + EPS);
  }
}

// ---------------------------------------------------------------- synthetic TenSet-shaped data
// Bit-identical to the device generator (csrc/synth.cu): row i of seed s draws
// from stream KeyBuilder(s,"feat",i), column j is draw j+1; labels are
// 0.1 + uniform01 of stream KeyBuilder(s,"label",i); statement counts per
// program 1 + below(8) of stream KeyBuilder(s,"stmts",p).
inline std::uint64_t feat_key(std::uint64_t seed, std::uint64_t row) {
  return KeyBuilder().add(seed).add("feat").add(row).value();
}
inline std::uint64_t label_key(std::uint64_t seed, std::uint64_t row) {
  return KeyBuilder().add(seed).add("label").add(row).value();
}
inline double synth_feature(std::uint64_t seed, std::uint64_t row, int col) {
  return u01_of(splitmix_at(feat_key(seed, row), std::uint64_t(col) + 1));
}
inline double synth_label(std::uint64_t seed, std::uint64_t row) {
  return 0.1 + u01_of(splitmix_at(label_key(seed, row), 1));
}
inline int synth_stmts(std::uint64_t seed, std::uint64_t prog, int max_stmts) {
  RngStream r(KeyBuilder().add(seed).add("stmts").add(prog).value());
  return 1 + int(r.below(std::uint64_t(max_stmts)));
}

// ---------------------------------------------------------------- knob space (space.cpp)
// Task descriptors (space.hpp:24-31) and the knob-space helpers the scorer's inputs come from.
struct TaskDesc {
  double work_gflops, bytes_per_unit, ideal_log2_tiles, ideal_log2_unroll;
};
// roles[i]: which template knob knob i is (knob_view matches by name, space.cpp:123-138):
// 0 tile_x, 1 tile_y, 2 unroll, 3 vectorize, 4 parallel, -1 none of them.
// encode_features (space.cpp:140-159): entries 0..9 live, 10..15 zero.
inline void encode_features(const TaskDesc& t, const std::int64_t* values, const int* roles, int nk, double* f) {
  std::int64_t kv[5] = {1, 1, 0, 1, 1};  // knob_view fallbacks (space.cpp:132-136)
  bool seen[5] = {false, false, false, false, false};  // find_knob takes the first knob of a name (space.cpp:19-24)
  for (int i = 0; i < nk; ++i)
    if (roles[i] >= 0 && roles[i] < 5 && !seen[roles[i]]) {
      kv[roles[i]] = values[i];
      seen[roles[i]] = true;
    }
  const double tx = double(kv[0]), ty = double(kv[1]), un = double(kv[2]);
  const double footprint = t.bytes_per_unit * tx * ty * std::max<double>(1.0, un);
  for (int j = 0; j < 16; ++j) f[j] = 0.0;
  f[0] = std::log2(tx) / 6.0;
  f[1] = std::log2(ty) / 6.0;
  f[2] = std::log2(1.0 + un) / 10.0;
  f[3] = std::log2(double(kv[3])) / 4.0;
  f[4] = std::log2(double(kv[4])) / 8.0;
  f[5] = std::log2(tx * ty) / 12.0;
  f[6] = std::log2(footprint) / 24.0;
  f[7] = std::clamp(std::log10(t.work_gflops) / 3.0, 0.0, 1.0);
  f[8] = t.ideal_log2_tiles / 16.0;
  f[9] = t.ideal_log2_unroll / 10.0;
}
// enumerate_configs (space.cpp:168-191): lexicographic, last knob fastest -> config `index`
inline void decode_config(std::uint64_t index, const std::int64_t* domains, const int* sizes, int nk,
                          std::int64_t* values) {
  int off[16];
  int o = 0;
  for (int i = 0; i < nk; ++i) { off[i] = o; o += sizes[i]; }
  for (int i = nk - 1; i >= 0; --i) {
    values[i] = domains[off[i] + int(index % std::uint64_t(sizes[i]))];
    index /= std::uint64_t(sizes[i]);
  }
}
// config_hash (space.cpp:193-197): FNV-1a over each value's 8 little-endian bytes
inline std::uint64_t config_hash(const std::int64_t* values, int nk) {
  KeyBuilder k;
  for (int i = 0; i < nk; ++i) k.add(std::uint64_t(values[i]));
  return k.h;
}

// ---------------------------------------------------------------- simulated hardware (oracle.cpp:33-105)
struct DeviceDesc {
  double peak_gflops, parallel_units, vector_lanes, cache_bytes, measure_overhead_ms, noise_std;
  int repeats;
};
inline void knob_values(const std::int64_t* values, const int* roles, int nk, std::int64_t kv[5]) {
  kv[0] = 1; kv[1] = 1; kv[2] = 0; kv[3] = 1; kv[4] = 1;
  bool seen[5] = {false, false, false, false, false};
  for (int i = 0; i < nk; ++i)
    if (roles[i] >= 0 && roles[i] < 5 && !seen[roles[i]]) { kv[roles[i]] = values[i]; seen[roles[i]] = true; }
}
// shared_factor (oracle.cpp:33-41)
inline double shared_factor(const TaskDesc& t, const std::int64_t kv[5]) {
  const double log_tiles = std::log2(static_cast<double>(kv[0] * kv[1]));
  const double tile_term = std::exp(-std::pow(log_tiles - t.ideal_log2_tiles, 2.0) / 8.0);
  const double log_unroll = std::log2(1.0 + static_cast<double>(kv[2]));
  const double unroll_term = 0.8 + 0.2 * std::exp(-std::pow(log_unroll - t.ideal_log2_unroll, 2.0) / 4.0);
  return tile_term * unroll_term;
}
// device_factor (oracle.cpp:43-56)
inline double device_factor(const DeviceDesc& d, const TaskDesc& t, const std::int64_t kv[5]) {
  const double p = static_cast<double>(kv[4]);
  const double vec = static_cast<double>(kv[3]);
  const double u = d.parallel_units, l = d.vector_lanes;
  const double parallel_term = std::min(p / u, u / p);
  const double vector_term = std::sqrt(std::min(vec / l, l / vec));
  const double footprint = t.bytes_per_unit * static_cast<double>(kv[0]) * static_cast<double>(kv[1]) *
                           std::max<double>(1.0, static_cast<double>(kv[2]));
  const double cache_term = footprint <= d.cache_bytes ? 1.0 : d.cache_bytes / footprint;
  return parallel_term * vector_term * cache_term;
}
// clean_latency_ms (oracle.cpp:58-63)
inline double clean_latency_ms(const DeviceDesc& d, const TaskDesc& t, const std::int64_t kv[5]) {
  const double throughput = d.peak_gflops * shared_factor(t, kv) * device_factor(d, t, kv);
  return t.work_gflops / throughput * 1000.0;
}
// measure (oracle.cpp:65-88): noise keyed on (seed, device id, task id, config hash)
inline void measure(const DeviceDesc& d, const TaskDesc& t, const std::int64_t* values, const int* roles, int nk,
                    std::uint64_t seed, const char* device_id, const char* task_id, double* throughput,
                    double* latency, double* wall_cost) {
  std::int64_t kv[5];
  knob_values(values, roles, nk, kv);
  KeyBuilder key;
  key.add(seed);
  key.add(std::string_view(device_id));
  key.add(std::string_view(task_id));
  key.add(config_hash(values, nk));
  RngStream rng(key.value());
  const double eps = rng.gaussian() * d.noise_std;
  const double noise = std::max(0.05, 1.0 + eps);
  *throughput = d.peak_gflops * shared_factor(t, kv) * device_factor(d, t, kv) * noise;
  *latency = t.work_gflops / *throughput * 1000.0;
  *wall_cost = d.measure_overhead_ms + static_cast<double>(d.repeats) * *latency;
}

// ---------------------------------------------------------------- files (model.cpp:344-412, lottery.cpp:182-240)
inline void put_u32(std::string& o, std::uint32_t v) { for (int i = 0; i < 4; ++i) o.push_back(char((v >> (8 * i)) & 0xff)); }
inline void put_u64(std::string& o, std::uint64_t v) { for (int i = 0; i < 8; ++i) o.push_back(char((v >> (8 * i)) & 0xff)); }
inline void put_f64(std::string& o, double d) { put_u64(o, std::bit_cast<std::uint64_t>(d)); }

inline std::string serialize(const Params<double>& p) {
  check_dims(p.dims, true);
  if (p.dims[1] != 512 || p.dims[2] != 512) fail(Err::BadDims, "only the {D,512,512,1} shape has a file form");
  std::string out;
  out.append("MOSM", 4);
  put_u32(out, 1);
  put_u32(out, std::uint32_t(p.dims[0]));
  for (double v : p.w) put_f64(out, v);
  for (double v : p.mom) put_f64(out, v);
  return out;
}

inline std::string write_mask_bytes(const std::uint8_t* mask, std::uint64_t n, std::uint32_t phase, Mode mode, double value) {
  std::string buf("MOSK", 4);
  put_u64(buf, n);
  put_u32(buf, phase);
  buf.push_back(mode == Mode::Threshold ? '\x01' : '\x02');
  put_f64(buf, value);
  std::string bits((n + 7) / 8, '\0');
  for (std::uint64_t i = 0; i < n; ++i)
    if (mask[i]) bits[i / 8] = char(bits[i / 8] | (1 << (i % 8)));
  return buf + bits;
}

}  // namespace oracle
