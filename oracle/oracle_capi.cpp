// oracle_capi.cpp — C entry points over moses_oracle.hpp for the Python tests
// and the CPU-baseline leg of bench.py. TEST INFRASTRUCTURE ONLY: nothing in
// paper_2201_05752_b200/ links or loads this library.
//
// Status convention: 0 = ok, otherwise 1 + moseslab::ErrorCode ordinal
// (errors.hpp:10-36), message retrievable with orc_last_error().
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "moses_oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + int(e.code);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1000;
  }
}

std::vector<int> to_dims(const int* dims, int nd) { return std::vector<int>(dims, dims + nd); }

template <class R>
Params<R> make_params(const int* dims, int nd, const R* w, const R* mom) {
  Params<R> p;
  p.dims = to_dims(dims, nd);
  const std::int64_t P = param_count(p.dims);
  p.w.assign(w, w + P);
  if (mom) p.mom.assign(mom, mom + P);
  else p.mom.assign(P, R(0));
  return p;
}

template <class R>
Adversary<R> make_adv(const R* aw, R ab, const R* replay, int m, int D, int width) {
  Adversary<R> a;
  a.weight.assign(aw, aw + width);
  a.bias = ab;
  a.m = m;
  a.replay.assign(replay, replay + std::size_t(m) * D);
  return a;
}
}  // namespace

#define ORC extern "C" __attribute__((visibility("default")))

ORC const char* orc_last_error() { return g_err.c_str(); }

// ---- rng / hashing KATs
ORC std::uint64_t orc_splitmix_draw(std::uint64_t seed, int k) {
  RngStream r(seed);
  std::uint64_t v = 0;
  for (int i = 0; i < k; ++i) v = r.next_u64();
  return v;
}
ORC std::uint64_t orc_splitmix_at(std::uint64_t key, std::uint64_t k) { return splitmix_at(key, k); }
ORC double orc_uniform01_first(std::uint64_t seed) { return RngStream(seed).uniform01(); }
ORC double orc_gaussian_first(std::uint64_t seed) { return RngStream(seed).gaussian(); }
ORC std::uint64_t orc_fnv_u64s(const std::uint64_t* v, int n) {
  KeyBuilder k;
  for (int i = 0; i < n; ++i) k.add(v[i]);
  return k.value();
}
ORC std::uint64_t orc_fnv_str(const char* s) { return KeyBuilder().add(std::string_view(s)).value(); }
ORC std::uint64_t orc_fnv_u64_str(std::uint64_t v, const char* s) {
  return KeyBuilder().add(v).add(std::string_view(s)).value();
}

// ---- model
ORC long long orc_param_count(const int* dims, int nd) { return param_count(to_dims(dims, nd)); }

ORC int orc_init_random(const int* dims, int nd, std::uint64_t seed, int strict, double* out_w) {
  return guarded([&] {
    Params<double> p = init_random(to_dims(dims, nd), seed, strict != 0);
    std::memcpy(out_w, p.w.data(), p.w.size() * sizeof(double));
  });
}

#define ORC_FWD(SUF, R)                                                                            \
  ORC int orc_forward_##SUF(const int* dims, int nd, const R* w, const R* x, int n, R* scores,    \
                            R* penult, int threads) {                                              \
    return guarded([&] {                                                                           \
      Params<R> p = make_params<R>(dims, nd, w, nullptr);                                          \
      Forward<R> f = run_forward(p, x, n, threads);                                                \
      if (scores) std::memcpy(scores, f.s.data(), sizeof(R) * n);                                  \
      if (penult) std::memcpy(penult, f.h.back().data(), sizeof(R) * f.h.back().size());           \
    });                                                                                            \
  }
ORC_FWD(f64, double)
ORC_FWD(f32, float)

#define ORC_RANK(SUF, R)                                                                            \
  ORC long long orc_ranking_terms_##SUF(const R* s, const R* y, int n, R* loss, R* gs) {          \
    return ranking_terms(s, y, n, loss, gs);                                                        \
  }
ORC_RANK(f64, double)
ORC_RANK(f32, float)

#define ORC_GRAD(SUF, R)                                                                            \
  ORC int orc_gradients_##SUF(const int* dims, int nd, const R* w, const R* x, const R* y, int n, \
                              const R* adv_w, R adv_b, const R* replay, int m, R beta, R* g_out,   \
                              R* loss_out, int threads) {                                           \
    return guarded([&] {                                                                            \
      Params<R> p = make_params<R>(dims, nd, w, nullptr);                                           \
      const int width = p.dims[p.levels() - 1];                                                     \
      Adversary<R> a;                                                                               \
      const Adversary<R>* ap = nullptr;                                                             \
      if (adv_w) {                                                                                  \
        a = make_adv<R>(adv_w, adv_b, replay, m, p.dims[0], width);                                 \
        ap = &a;                                                                                    \
      }                                                                                             \
      std::vector<R> g = gradients(p, x, y, n, ap, beta, loss_out, threads);                        \
      std::memcpy(g_out, g.data(), sizeof(R) * g.size());                                           \
    });                                                                                             \
  }                                                                                                 \
  ORC int orc_objective_##SUF(const int* dims, int nd, const R* w, const R* x, const R* y, int n, \
                              const R* adv_w, R adv_b, const R* replay, int m, R beta, R* out) {   \
    return guarded([&] {                                                                            \
      Params<R> p = make_params<R>(dims, nd, w, nullptr);                                           \
      const int width = p.dims[p.levels() - 1];                                                     \
      Adversary<R> a;                                                                               \
      const Adversary<R>* ap = nullptr;                                                             \
      if (adv_w) {                                                                                  \
        a = make_adv<R>(adv_w, adv_b, replay, m, p.dims[0], width);                                 \
        ap = &a;                                                                                    \
      }                                                                                             \
      *out = objective(p, x, y, n, ap, beta);                                                       \
    });                                                                                             \
  }
ORC_GRAD(f64, double)
ORC_GRAD(f32, float)

ORC int orc_mmd2_grad_f64(const double* xs, int m, const double* xt, int n, int width, double sigma, double* value,
                         double* gs, double* gt) {
  return guarded([&] { *value = mmd2_grad(xs, m, xt, n, width, sigma, gs, gt); });
}

ORC int orc_gradients_mmd_f64(const int* dims, int nd, const double* w, const double* x, const double* y, int n,
                             const double* src, int ms, double beta, double sigma, double* g_out, double* loss_out,
                             int threads) {
  return guarded([&] {
    Params<double> p = make_params<double>(dims, nd, w, nullptr);
    std::vector<double> g = gradients_mmd(p, x, y, n, src, ms, beta, sigma, loss_out, threads);
    std::memcpy(g_out, g.data(), sizeof(double) * g.size());
  });
}

ORC int orc_gradients_from_score_grads_f64(const int* dims, int nd, const double* w, const double* x, int n,
                                          const double* gs, double* g_out, int threads) {
  return guarded([&] {
    Params<double> p = make_params<double>(dims, nd, w, nullptr);
    std::vector<double> g = gradients_from_score_grads(p, x, n, gs, threads);
    std::memcpy(g_out, g.data(), sizeof(double) * g.size());
  });
}

ORC int orc_gradients_pooled_f64(const int* dims, int nd, const double* w, const double* x, int nstmt,
                                 const long long* off, int programs, const double* y, double* g_out, double* loss_out,
                                 int threads) {
  return guarded([&] {
    Params<double> p = make_params<double>(dims, nd, w, nullptr);
    std::vector<double> g = gradients_pooled(p, x, nstmt, reinterpret_cast<const std::int64_t*>(off), programs, y,
                                             loss_out, threads);
    std::memcpy(g_out, g.data(), sizeof(double) * g.size());
  });
}

#define ORC_UPD(SUF, R)                                                                             \
  ORC void orc_apply_update_##SUF(R* w, R* mom, const R* g, long long P, double lr, double mu,    \
                                  const std::uint8_t* keep, int use_momentum) {                    \
    Params<R> p;                                                                                    \
    p.w.assign(w, w + P);                                                                           \
    p.mom.assign(mom, mom + P);                                                                     \
    apply_update(p, g, lr, mu, keep, use_momentum != 0);                                            \
    std::memcpy(w, p.w.data(), sizeof(R) * P);                                                      \
    std::memcpy(mom, p.mom.data(), sizeof(R) * P);                                                  \
  }                                                                                                 \
  ORC void orc_xi_##SUF(const R* w, const R* g, long long P, int normalize, R* xi_out) {          \
    std::vector<R> xi = xi_scores(w, g, P, normalize != 0);                                         \
    std::memcpy(xi_out, xi.data(), sizeof(R) * P);                                                  \
  }                                                                                                 \
  ORC int orc_partition_##SUF(const R* xi, long long n, int normalized, int mode, double value,   \
                              std::uint8_t* mask_out) {                                             \
    return guarded([&] {                                                                            \
      std::vector<std::uint8_t> m = partition(xi, n, normalized != 0, Mode(mode), value);          \
      std::memcpy(mask_out, m.data(), m.size());                                                    \
    });                                                                                             \
  }                                                                                                 \
  ORC int orc_variant_decay_##SUF(R* w, long long P, const std::uint8_t* keep, double alpha,      \
                                  double lambda) {                                                  \
    return guarded([&] { variant_decay(w, P, keep, alpha, lambda); });                              \
  }                                                                                                 \
  ORC void orc_accuracy_counts_##SUF(const R* s, const R* y, int n, long long* pairs,             \
                                     long long* conc) {                                             \
    std::int64_t p = 0, c = 0;                                                                      \
    accuracy_counts(s, y, n, &p, &c);                                                               \
    *pairs += p;                                                                                    \
    *conc += c;                                                                                     \
  }                                                                                                 \
  ORC R orc_disc_ce_##SUF(const R* zs, int m, const R* zt, int n) {                                \
    return discriminator_cross_entropy(zs, m, zt, n);                                               \
  }                                                                                                 \
  ORC int orc_adversarial_term_##SUF(R* aw, R* ab, const R* hs, int m, const R* ht, int n,        \
                                     int width, R step, R* loss_out) {                              \
    return guarded([&] {                                                                            \
      Adversary<R> a;                                                                               \
      a.weight.assign(aw, aw + width);                                                              \
      a.bias = *ab;                                                                                 \
      a.m = 1; /* replay presence is the caller's concern */                                        \
      a.step_size = step;                                                                           \
      *loss_out = adversarial_term(a, hs, m, ht, n, width);                                         \
      std::memcpy(aw, a.weight.data(), sizeof(R) * width);                                          \
      *ab = a.bias;                                                                                 \
    });                                                                                             \
  }                                                                                                 \
  ORC void orc_topk_##SUF(const R* s, long long n, long long k, long long* idx_out) {             \
    std::vector<std::int64_t> t = topk(s, n, k);                                                    \
    for (std::size_t i = 0; i < t.size(); ++i) idx_out[i] = t[i];                                   \
  }                                                                                                 \
  ORC void orc_segment_sum_##SUF(const R* h, int width, const long long* off, long long programs, \
                                 R* out) {                                                          \
    segment_sum(h, width, reinterpret_cast<const std::int64_t*>(off), programs, out);               \
  }                                                                                                 \
  ORC R orc_mmd2_##SUF(const R* xs, int m, const R* xt, int n, int width, R sigma) {               \
    return mmd2(xs, m, xt, n, width, sigma);                                                        \
  }                                                                                                 \
  ORC void orc_adam_##SUF(R* w, R* m1, R* m2, const R* g, long long P, const std::uint8_t* keep,  \
                          double lr, double b1, double b2, double eps, int t) {                     \
    adam_update(w, m1, m2, g, P, keep, lr, b1, b2, eps, t);                                         \
  }
ORC_UPD(f64, double)
ORC_UPD(f32, float)

ORC long long orc_ratio_keep(double value, long long n) { return ratio_keep(value, n); }

// ---- synthetic data (bit-identical to the device generator)
ORC void orc_synth_features(std::uint64_t seed, long long row0, long long rows, int D, double* out) {
  for (long long r = 0; r < rows; ++r) {
    const std::uint64_t key = feat_key(seed, std::uint64_t(row0 + r));
    for (int j = 0; j < D; ++j) out[r * D + j] = u01_of(splitmix_at(key, std::uint64_t(j) + 1));
  }
}
ORC void orc_synth_labels(std::uint64_t seed, long long row0, long long rows, double* out) {
  for (long long r = 0; r < rows; ++r) out[r] = synth_label(seed, std::uint64_t(row0 + r));
}
ORC void orc_synth_offsets(std::uint64_t seed, long long programs, int max_stmts, long long* off) {
  off[0] = 0;
  for (long long p = 0; p < programs; ++p) off[p + 1] = off[p] + synth_stmts(seed, std::uint64_t(p), max_stmts);
}

// ---- files
ORC long long orc_serialize(const int* dims, int nd, const double* w, const double* mom, char* out, long long cap) {
  std::string s;
  const int rc = guarded([&] { s = serialize(make_params<double>(dims, nd, w, mom)); });
  if (rc != 0) return -rc;
  if (out && cap >= (long long)s.size()) std::memcpy(out, s.data(), s.size());
  return (long long)s.size();
}
ORC long long orc_write_mask_bytes(const std::uint8_t* mask, long long n, unsigned phase, int mode, double value,
                                   char* out, long long cap) {
  const std::string s = write_mask_bytes(mask, std::uint64_t(n), phase, Mode(mode), value);
  if (out && cap >= (long long)s.size()) std::memcpy(out, s.data(), s.size());
  return (long long)s.size();
}

// ---- CPU baseline: one pretraining step (gradients + momentum update) in fp64,
// exactly the reference's pretrain loop body (tuner.cpp:144-147).
ORC int orc_train_step_f64(const int* dims, int nd, double* w, double* mom, const double* x, const double* y, int n,
                           double lr, double mu, double* loss_out, int threads) {
  return guarded([&] {
    Params<double> p = make_params<double>(dims, nd, w, mom);
    std::vector<double> g = gradients<double>(p, x, y, n, nullptr, 0.0, loss_out, threads);
    apply_update(p, g.data(), lr, mu, nullptr, true);
    std::memcpy(w, p.w.data(), sizeof(double) * p.w.size());
    std::memcpy(mom, p.mom.data(), sizeof(double) * p.mom.size());
  });
}

// ---- knob space (space.cpp:140-197): configs [first, first+n) of the lexicographic enumeration
ORC int orc_encode_configs(const double* task4, const std::int64_t* domains, const int* sizes, const int* roles, int nk,
                           std::uint64_t first, std::int64_t n, double* feats, std::uint64_t* hashes,
                           std::int64_t* values_out) {
  return guarded([&] {
    if (nk <= 0 || nk > 16) throw std::runtime_error("knob count out of range");
    const TaskDesc t{task4[0], task4[1], task4[2], task4[3]};
    std::int64_t v[16];
    for (std::int64_t i = 0; i < n; ++i) {
      decode_config(first + std::uint64_t(i), domains, sizes, nk, v);
      if (feats) encode_features(t, v, roles, nk, feats + i * 16);
      if (hashes) hashes[i] = config_hash(v, nk);
      if (values_out)
        for (int k = 0; k < nk; ++k) values_out[i * nk + k] = v[k];
    }
  });
}

// ---- simulated hardware (oracle.cpp:33-105) over configs [first, first+n) of the enumeration
ORC int orc_measure_configs(const double* dev6, int repeats, const char* device_id, const char* task_id,
                            const double* task4, const std::int64_t* domains, const int* sizes, const int* roles,
                            int nk, std::uint64_t seed, std::uint64_t first, std::int64_t n, double* clean_ms,
                            double* throughput, double* latency, double* wall_cost) {
  return guarded([&] {
    const DeviceDesc d{dev6[0], dev6[1], dev6[2], dev6[3], dev6[4], dev6[5], repeats};
    const TaskDesc t{task4[0], task4[1], task4[2], task4[3]};
    std::int64_t v[16], kv[5];
    for (std::int64_t i = 0; i < n; ++i) {
      decode_config(first + std::uint64_t(i), domains, sizes, nk, v);
      knob_values(v, roles, nk, kv);
      if (clean_ms) clean_ms[i] = clean_latency_ms(d, t, kv);
      if (throughput) measure(d, t, v, roles, nk, seed, device_id, task_id, throughput + i, latency + i, wall_cost + i);
    }
  });
}

// true_best (oracle.cpp:90-105): exhaustive noise-free minimum, strict < keeps the lexicographically first
ORC int orc_true_best(const double* dev6, const double* task4, const std::int64_t* domains, const int* sizes,
                      const int* roles, int nk, std::int64_t* best_values, double* best_latency) {
  return guarded([&] {
    const DeviceDesc d{dev6[0], dev6[1], dev6[2], dev6[3], dev6[4], dev6[5], 1};
    const TaskDesc t{task4[0], task4[1], task4[2], task4[3]};
    std::uint64_t space = 1;
    for (int k = 0; k < nk; ++k) space *= std::uint64_t(sizes[k]);
    std::int64_t v[16], kv[5];
    double best = std::numeric_limits<double>::infinity();
    for (std::uint64_t i = 0; i < space; ++i) {
      decode_config(i, domains, sizes, nk, v);
      knob_values(v, roles, nk, kv);
      const double lat = clean_latency_ms(d, t, kv);
      if (lat < best) {
        best = lat;
        for (int k = 0; k < nk; ++k) best_values[k] = v[k];
      }
    }
    *best_latency = best;
  });
}
