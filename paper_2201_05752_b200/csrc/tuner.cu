// tuner.cu — the tuner's online loop (tuner.cpp:158-286) and its (strategy, seed, task) job grid
// (tuner.cpp:307-374) over this library's calls.
//
// Per measured batch: evolve on the device model (moses_evolve: keyed GA walk on the host, every
// generation encoded from enumeration indices and scored by the cost model on the GPU) -> select_batch
// (first unseen hashes) -> measure (the simulated hardware, oracle.cpp:65-88, on the device over the
// batch's enumeration indices) -> the controller's coefficient of variation (controller.cpp:34-56, host
// scalars) -> the strategy's update on the batch's encoded rows (Moses: gradients with the replay
// adversary -> discriminator step -> lottery step, in one moses_moses_step; vanilla / random-init:
// gradients -> apply_update without momentum). Then the prediction-only tail. The job grid runs
// independent jobs on their own handles (any GPU of the process) from a worker pool, the reference's
// compare pool shape: jobs claimed in order, the first failing job's status returned.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "kernels.cuh"

namespace moses {
void set_last_error(const std::string& msg);
int model_device(const moses_model* m);
std::vector<int> model_dims(const moses_model* m);

namespace {

// KeyBuilder (rng.hpp:16-42): FNV-1a over the little-endian bytes of u64 parts, strings with their NUL
struct Key {
  unsigned long long h = 0xcbf29ce484222325ull;
  Key& add(unsigned long long v) {
    for (int b = 0; b < 8; ++b) byte((unsigned char)(v >> (8 * b)));
    return *this;
  }
  Key& add(const char* s) {
    for (; *s; ++s) byte((unsigned char)*s);
    byte(0);
    return *this;
  }
  void byte(unsigned char c) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
};

void ck(int rc) {
  if (rc != MOSES_OK) throw Status(rc, moses_last_error());
}

// controller.cpp:10-32
struct Plan {
  int prediction_trials = 0;
  std::vector<int> batch_sizes;
};
Plan plan_split(int total, double p, int q) {
  if (q < 2) fail(MOSES_ERR_INVALID_CONFIG, "need at least 2 batches");
  if (total < q) fail(MOSES_ERR_INVALID_CONFIG, "total trials below the batch count");
  if (!(p > 0.0) || p > 1.0) fail(MOSES_ERR_INVALID_CONFIG, "train fraction must lie in (0,1]");
  const int measured = int(std::floor(p * double(total) + 1e-9));
  if (measured < q)
    fail(MOSES_ERR_INFEASIBLE_SPLIT,
         std::to_string(measured) + " measured trials cannot fill " + std::to_string(q) + " batches");
  Plan plan;
  plan.prediction_trials = total - measured;
  const int base = measured / q, rem = measured % q;
  for (int b = 0; b < q; ++b) plan.batch_sizes.push_back(base + (b < rem ? 1 : 0));
  return plan;
}
// controller.cpp:34-45 (callers guarantee >= 2 means and a non-zero mean)
double batch_cv(const std::vector<double>& means) {
  double mean = 0.0;
  for (double v : means) mean += v;
  mean /= double(means.size());
  double var = 0.0;
  for (double v : means) var += (v - mean) * (v - mean);
  var /= double(means.size());
  return std::sqrt(var) / mean;
}
// tuner.cpp:31-37
double guarded_cv(const std::vector<double>& means) {
  if (means.size() < 2) return std::numeric_limits<double>::quiet_NaN();
  double mean = 0.0;
  for (double v : means) mean += v;
  if (mean == 0.0) return std::numeric_limits<double>::quiet_NaN();
  return batch_cv(means);
}
// controller.cpp:47-56
struct Controller {
  double cv_threshold = 0.05;
  std::vector<double> batch_means;
  bool terminated = false;
  void push(double m) {
    batch_means.push_back(m);
    if (terminated || batch_means.size() < 3) return;
    double mean = 0.0;
    for (double v : batch_means) mean += v;
    if (mean == 0.0) return;
    if (std::abs(batch_cv(batch_means)) < cv_threshold) terminated = true;
  }
};

struct Space {  // enumeration order of space.cpp:168-191 (last knob fastest)
  const moses_task_spec* t;
  std::vector<int> off;
  explicit Space(const moses_task_spec* task) : t(task) {
    int o = 0;
    for (int k = 0; k < t->n_knobs; ++k) {
      off.push_back(o);
      o += t->domain_sizes[k];
    }
  }
  unsigned long long index_of(const long long* v) const {
    unsigned long long id = 0;
    for (int k = 0; k < t->n_knobs; ++k) {
      const long long* d = reinterpret_cast<const long long*>(t->domains) + off[size_t(k)];
      const int pos = int(std::lower_bound(d, d + t->domain_sizes[k], v[k]) - d);
      if (pos >= t->domain_sizes[k] || d[pos] != v[k]) fail(MOSES_ERR_INVALID_CONFIG, "value outside its knob domain");
      id = id * (unsigned long long)t->domain_sizes[k] + (unsigned long long)pos;
    }
    return id;
  }
};

unsigned long long config_hash(const long long* v, int nk) {  // space.cpp:193-197
  Key k;
  for (int i = 0; i < nk; ++i) k.add((unsigned long long)v[i]);
  return k.h;
}

struct Rec {
  std::vector<long long> values;
  double thr, lat, wall;
};

void run_task(moses_model* m, int strategy, const moses_device_spec* dev, const moses_task_spec* task,
              const moses_tune_budget* b, unsigned long long seed, const double* src, long long n_src,
              moses_task_result* out) {
  if (!m || !dev || !task || !b || !out) fail(MOSES_ERR_INVALID_ARG, "null argument");
  if (strategy < MOSES_STRATEGY_RAW || strategy > MOSES_STRATEGY_MOSES) fail(MOSES_ERR_INVALID_CONFIG, "unknown strategy");
  if (task->n_knobs < 1 || task->n_knobs > 8) fail(MOSES_ERR_INVALID_TASK, "knob count must lie in [1, 8]");
  const int nk = task->n_knobs;
  const std::vector<int> dims = model_dims(m);
  const int D = dims[0], W = dims[dims.size() - 2];
  const Space sp(task);
  cudaStream_t st = nullptr;
  ck(moses_model_stream(m, reinterpret_cast<void**>(&st)));
  const long long* domains = reinterpret_cast<const long long*>(task->domains);
  // device scratch for one batch: enumeration indices, measurements, encoded rows
  const long long cap_rows = std::max<long long>(1, b->trials_per_task);
  unsigned long long* didx = nullptr;
  double *dthr = nullptr, *dlat = nullptr, *dwall = nullptr, *dfeat = nullptr;
  MOSES_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&didx), sizeof(unsigned long long) * cap_rows, st));
  MOSES_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dthr), sizeof(double) * cap_rows * 3, st));
  MOSES_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dfeat), sizeof(double) * cap_rows * D, st));
  dlat = dthr + cap_rows;
  dwall = dlat + cap_rows;
  moses_adversary_t adv = nullptr;
  auto release = [&] {
    cudaStreamSynchronize(st);
    cudaFreeAsync(didx, st);
    cudaFreeAsync(dthr, st);
    cudaFreeAsync(dfeat, st);
    cudaStreamSynchronize(st);
    if (adv) moses_adversary_destroy(adv);
  };
  // measure (oracle.cpp:65-88) of n configurations, on the device
  auto measure = [&](const std::vector<const long long*>& cfgs, std::vector<Rec>& recs) {
    const long long n = (long long)cfgs.size();
    if (n > cap_rows) fail(MOSES_ERR_CAPACITY, "batch above trials_per_task");
    std::vector<unsigned long long> ids(static_cast<size_t>(n), 0ull);
    for (long long i = 0; i < n; ++i) ids[size_t(i)] = sp.index_of(cfgs[size_t(i)]);
    MOSES_CUDA(cudaMemcpyAsync(didx, ids.data(), sizeof(unsigned long long) * n, cudaMemcpyHostToDevice, st));
    measure_configs_idx(dev->params, dev->repeats, dev->id, task->id, task->task4, domains, task->domain_sizes,
                        task->roles, nk, seed, didx, n, dthr, dlat, dwall, st);
    std::vector<double> h(static_cast<size_t>(3 * cap_rows));
    MOSES_CUDA(cudaMemcpyAsync(h.data(), dthr, sizeof(double) * 3 * cap_rows, cudaMemcpyDeviceToHost, st));
    MOSES_CUDA(cudaStreamSynchronize(st));
    for (long long i = 0; i < n; ++i)
      recs.push_back({std::vector<long long>(cfgs[size_t(i)], cfgs[size_t(i)] + nk), h[size_t(i)],
                      h[size_t(cap_rows + i)], h[size_t(2 * cap_rows + i)]});
  };
  // encode_batch (space.cpp:161-166) of configurations, rows of width D on the host
  auto encode = [&](const std::vector<Rec>& recs, size_t first, std::vector<double>& x) {
    const long long n = (long long)(recs.size() - first);
    std::vector<unsigned long long> ids(static_cast<size_t>(n));
    for (long long i = 0; i < n; ++i) ids[size_t(i)] = sp.index_of(recs[first + size_t(i)].values.data());
    MOSES_CUDA(cudaMemcpyAsync(didx, ids.data(), sizeof(unsigned long long) * n, cudaMemcpyHostToDevice, st));
    encode_configs_idx(task->task4, domains, task->domain_sizes, task->roles, nk, didx, n, MOSES_DTYPE_F64, dfeat, D, D,
                       st);
    x.assign(size_t(n * D), 0.0);
    MOSES_CUDA(cudaMemcpyAsync(x.data(), dfeat, sizeof(double) * n * D, cudaMemcpyDeviceToHost, st));
    MOSES_CUDA(cudaStreamSynchronize(st));
  };
  // evolve(params, space, sp) (search.cpp:73-80) with the batch's keyed seed
  const long long pop_cap = std::max<long long>(b->population, (long long)b->survivors * (1 + b->mutation_count));
  std::vector<long long> pvals(static_cast<size_t>(pop_cap * nk));
  std::vector<double> pscores(static_cast<size_t>(pop_cap));
  auto evolve = [&](unsigned long long s) -> long long {
    int64_t n = 0;
    ck(moses_evolve(m, nullptr, task->task4, task->domains, task->domain_sizes, task->roles, nk, b->population,
                    b->generations, b->mutation_count, b->survivors, b->epsilon_random, s,
                    reinterpret_cast<int64_t*>(pvals.data()), pscores.data(), pop_cap, &n));
    return n;
  };
  // select_batch (search.cpp:82-95): the first `want` candidates whose hash is neither measured nor taken
  auto select = [&](long long n, const std::unordered_set<unsigned long long>& measured, int want) {
    std::vector<long long> pos;
    std::unordered_set<unsigned long long> taken;
    for (long long i = 0; i < n && (int)pos.size() < want; ++i) {
      const unsigned long long h = config_hash(&pvals[size_t(i * nk)], nk);
      if (measured.count(h) || !taken.insert(h).second) continue;
      pos.push_back(i);
    }
    return pos;
  };

  std::vector<Rec> recs;
  double wall_total = 0.0;
  int unspent = 0, termination_batch = -1, measured_trials = 0, prediction_trials = 0;
  std::vector<double> cvs, predicted;
  Controller ctrl;
  ctrl.cv_threshold = b->cv_threshold;
  std::vector<long long> best_cfg;
  double best_lat = std::numeric_limits<double>::infinity();
  try {
    if (strategy == MOSES_STRATEGY_RAW) {  // tuner.cpp:166-178: the median default configuration, once
      std::vector<long long> cfg(static_cast<size_t>(nk));
      for (int k = 0; k < nk; ++k) cfg[size_t(k)] = domains[sp.off[size_t(k)] + (task->domain_sizes[k] - 1) / 2];
      measure({cfg.data()}, recs);
      best_cfg = cfg;
      best_lat = recs[0].lat;
      wall_total = recs[0].wall;
      measured_trials = 1;
      unspent = b->trials_per_task - 1;
    } else {
      const Plan plan = plan_split(b->trials_per_task, b->train_fraction, b->num_batches);
      const bool use_adv = strategy == MOSES_STRATEGY_MOSES && b->adversary;
      if (use_adv) {  // tuner.cpp:187-201
        if (src == nullptr || n_src <= 0)
          fail(MOSES_ERR_ADVERSARY_DISABLED, "adversarial term needs source records; pass them or turn the adversary off");
        const unsigned long long rseed = Key().add(seed).add("replay").add(task->id).h;
        std::vector<long long> rows(static_cast<size_t>(std::max(b->replay_size, 1)));
        int64_t k = 0;
        ck(moses_replay_rows(n_src, b->replay_size, rseed, reinterpret_cast<int64_t*>(rows.data()), &k));
        std::vector<double> replay(static_cast<size_t>(k * D));
        for (int64_t r = 0; r < k; ++r)
          std::copy(src + rows[size_t(r)] * D, src + (rows[size_t(r)] + 1) * D, replay.begin() + r * D);
        ck(moses_adversary_create(replay.data(), k, D, W, 0.1, &adv));  // make_adversary: u = 0, c = 0, eta 0.1
      }
      std::unordered_set<unsigned long long> measured;
      for (int bi = 0; bi < b->num_batches; ++bi) {  // tuner.cpp:209-267
        const int want = plan.batch_sizes[size_t(bi)];
        if (ctrl.terminated) {
          unspent += want;
          continue;
        }
        const long long n = evolve(Key().add(seed).add("evolve").add(task->id).add((unsigned long long)bi).h);
        const std::vector<long long> pos = select(n, measured, want);
        unspent += want - int(pos.size());
        if (pos.empty()) continue;
        const size_t first = recs.size();
        std::vector<const long long*> cfgs;
        double score_sum = 0.0;
        for (long long p : pos) cfgs.push_back(&pvals[size_t(p * nk)]);
        measure(cfgs, recs);
        for (size_t i = 0; i < pos.size(); ++i) {
          const Rec& r = recs[first + i];
          wall_total += r.wall;
          if (r.lat < best_lat) {
            best_lat = r.lat;
            best_cfg = r.values;
          }
          measured.insert(config_hash(r.values.data(), nk));
          score_sum += pscores[size_t(pos[i])];
        }
        measured_trials += int(pos.size());
        ctrl.push(score_sum / double(pos.size()));
        cvs.push_back(guarded_cv(ctrl.batch_means));
        if (ctrl.terminated && termination_batch < 0) termination_batch = int(ctrl.batch_means.size());
        if (strategy == MOSES_STRATEGY_PRETRAIN_ONLY || pos.size() < 2) continue;
        // batch_from_measurements (tuner.cpp:39-55): encoded rows, measured throughputs as labels
        std::vector<double> x, y;
        encode(recs, first, x);
        for (size_t i = first; i < recs.size(); ++i) y.push_back(recs[i].thr);
        const long long nb = (long long)y.size();
        if (strategy == MOSES_STRATEGY_MOSES) {  // tuner.cpp:248-262
          const double beta = use_adv ? b->adversary_beta : 0.0;
          if (use_adv && beta != 0.0) {
            ck(moses_moses_step(m, adv, x.data(), y.data(), nb, D, beta, b->lottery_mode, b->lottery_value, bi,
                                b->learning_rate, b->weight_decay, nullptr, nullptr, nullptr));
          } else {
            ck(moses_gradients(m, x.data(), y.data(), nb, D, nullptr, 0.0, nullptr));
            int64_t pop = 0;
            ck(moses_lottery_step(m, b->lottery_mode, b->lottery_value, bi, b->learning_rate, b->weight_decay, nullptr,
                                  0, &pop));
          }
        } else {  // tuner.cpp:263-266: apply_update(params, grads, hyper, nullptr, false)
          ck(moses_gradients(m, x.data(), y.data(), nb, D, nullptr, 0.0, nullptr));
          ck(moses_apply_update(m, b->learning_rate, 0.0, nullptr, 0, 0));
        }
      }
      // prediction-only tail (tuner.cpp:271-279)
      const long long n = evolve(Key().add(seed).add("predict").add(task->id).h);
      const std::vector<long long> tail = select(n, measured, plan.prediction_trials);
      unspent += plan.prediction_trials - int(tail.size());
      for (long long p : tail) predicted.push_back(pscores[size_t(p)]);
      prediction_trials = int(tail.size());
    }
    ck(moses_model_synchronize(m));
  } catch (...) {
    release();
    throw;
  }
  release();
  if (recs.empty()) fail(MOSES_ERR_INVALID_CONFIG, std::string("no configuration was measured for task ") + task->id);
  if ((long long)recs.size() > out->capacity || (long long)predicted.size() > out->capacity)
    fail(MOSES_ERR_CAPACITY, "result capacity below trials_per_task");
  for (size_t i = 0; i < recs.size(); ++i) {
    if (out->values) std::copy(recs[i].values.begin(), recs[i].values.end(), out->values + i * size_t(nk));
    if (out->throughput) out->throughput[i] = recs[i].thr;
    if (out->latency) out->latency[i] = recs[i].lat;
    if (out->wall_cost) out->wall_cost[i] = recs[i].wall;
  }
  out->n_records = (int64_t)recs.size();
  if (out->best_values) std::copy(best_cfg.begin(), best_cfg.end(), out->best_values);
  out->best_latency_ms = best_lat;
  out->wall_cost_ms = wall_total;
  const size_t nm = ctrl.batch_means.size();
  if (nm > size_t(std::max(b->num_batches, 0))) fail(MOSES_ERR_CAPACITY, "batch means above num_batches");
  for (size_t i = 0; i < nm; ++i) {
    if (out->batch_means) out->batch_means[i] = ctrl.batch_means[i];
    if (out->cvs) out->cvs[i] = cvs[i];
  }
  out->n_batch_means = int32_t(nm);
  out->termination_batch = termination_batch;
  out->measured_trials = measured_trials;
  out->prediction_trials = prediction_trials;
  out->unspent_trials = unspent;
  for (size_t i = 0; i < predicted.size(); ++i)
    if (out->predicted_scores) out->predicted_scores[i] = predicted[i];
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return MOSES_OK;
  } catch (const Status& s) {
    set_last_error(s.what());
    return s.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return MOSES_ERR_INVALID_ARG;
  }
}

}  // namespace
}  // namespace moses

using namespace moses;

MOSES_API int moses_tune_task(moses_model_t m, int32_t strategy, const moses_device_spec* device,
                              const moses_task_spec* task, const moses_tune_budget* budget, uint64_t seed,
                              const double* source_features, int64_t n_source, moses_task_result* out) {
  return guard([&] { run_task(m, strategy, device, task, budget, seed, source_features, n_source, out); });
}

MOSES_API int moses_tune_jobs(int32_t n_jobs, const moses_model_t* models, const int32_t* strategies,
                              const uint64_t* seeds, const int32_t* task_of, const moses_task_spec* tasks,
                              int32_t n_tasks, const moses_device_spec* device, const moses_tune_budget* budget,
                              const double* source_features, int64_t n_source, int32_t threads,
                              moses_task_result* results) {
  return guard([&] {
    if (n_jobs < 0 || (n_jobs > 0 && (!models || !strategies || !seeds || !task_of || !tasks || !results)))
      fail(MOSES_ERR_INVALID_ARG, "null job arrays");
    {  // one job per handle: a handle's stream and workspaces serve one host thread at a time
      std::unordered_set<const void*> seen;
      for (int j = 0; j < n_jobs; ++j) {
        if (!models[j]) fail(MOSES_ERR_INVALID_ARG, "null model handle");
        if (!seen.insert(models[j]).second) fail(MOSES_ERR_INVALID_ARG, "a handle is listed for two jobs");
        if (task_of[j] < 0 || task_of[j] >= n_tasks) fail(MOSES_ERR_INVALID_ARG, "task index out of range");
      }
    }
    const int width = std::max(1, std::min(threads > 0 ? threads : n_jobs, std::min(n_jobs, 64)));
    std::atomic<int> next{0};
    std::mutex mu;
    int first_rc = MOSES_OK;
    int first_job = n_jobs;
    std::string first_msg;
    auto worker = [&] {
      for (;;) {
        const int j = next.fetch_add(1);
        if (j >= n_jobs) return;
        int rc = cudaSetDevice(model_device(models[j])) == cudaSuccess ? MOSES_OK : MOSES_ERR_CUDA;
        if (rc == MOSES_OK)
          rc = moses_tune_task(models[j], strategies[j], device, &tasks[task_of[j]], budget, seeds[j], source_features,
                               n_source, &results[j]);
        if (rc != MOSES_OK) {
          std::lock_guard<std::mutex> lk(mu);
          if (j < first_job) {  // the first failing job in job order (tuner.cpp:341-374 keeps the first thrown)
            first_job = j;
            first_rc = rc;
            first_msg = moses_last_error();
          }
        }
      }
    };
    int dev0 = 0;
    cudaGetDevice(&dev0);
    if (width == 1) {
      worker();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < width; ++t) pool.emplace_back(worker);
      for (auto& t : pool) t.join();
    }
    cudaSetDevice(dev0);
    if (first_rc != MOSES_OK) throw Status(first_rc, "job " + std::to_string(first_job) + ": " + first_msg);
  });
}
