// moses_gpu.hpp — header-only C++ host layer over the C ABI (moses_gpu.h).
//
// Mirrors the reference's namespace moseslab hot-path API
// (/root/reference/proj/include/moseslab/{model,lottery,search}.hpp): same function
// names, argument meaning and error behaviour (throws moseslab_gpu::Error carrying the
// reference's ErrorCode). Eigen is not a dependency: matrices are row-major
// std::vector<double> views; CostModelParams keeps the reference's flat parameter order
// (lottery.hpp:13-14), so a caller holding Eigen data maps it without reordering
// weights (only feature matrices are transposed, column-major -> row-major).
//
// Link: -L<pkg> -lmoses_gpu   (paper_2201_05752_b200/libmoses_gpu.so)
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <algorithm>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "moses_gpu.h"

namespace moseslab_gpu {

// moseslab::ErrorCode (errors.hpp:10-36)
enum class ErrorCode {
  InvalidTask, InvalidConfig, SpaceTooLarge, ImmutableSpace, BadDims, DimMismatch, ShapeMismatch,
  VersionMismatch, CorruptStream, EmptyDataset, InvalidRatio, UnnormalizedThreshold, AdversaryDisabled,
  UnstableDecay, InfeasibleSplit, ZeroMean, InsufficientBatches, BudgetInfeasible, MissingReferenceStrategy,
  MismatchedRuns, EmptyRows, ParseError, MissingField, IoError, UsageError,
  // library-side (not in the reference)
  Cuda = 100, NoDevice, Capacity, InvalidArgument
};

class Error : public std::runtime_error {
 public:
  Error(int status, const std::string& msg)
      : std::runtime_error(msg), code_(status < 100 ? ErrorCode(status - 1) : ErrorCode(status)) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

inline void check(int status) {
  if (status != MOSES_OK) throw Error(status, moses_last_error());
}

struct Matrix {  // row-major n x d
  int64_t rows = 0;
  int32_t cols = 0;
  std::vector<double> data;
  Matrix() = default;
  Matrix(int64_t r, int32_t c) : rows(r), cols(c), data(size_t(r) * c, 0.0) {}
  double& operator()(int64_t r, int32_t c) { return data[size_t(r) * cols + c]; }
  double operator()(int64_t r, int32_t c) const { return data[size_t(r) * cols + c]; }
};

struct CostModelParams {  // model.hpp:19-25, flat reference order
  std::vector<int32_t> dims;
  std::vector<double> params;
  std::vector<double> momentum;
};

struct TrainHyper {  // model.hpp:27-35
  double learning_rate = 0.001;
  double weight_decay = 0.01;
  int max_epochs = 30;
  int batch_size = 512;
  double momentum = 0.9;
  double adversary_beta = 0.01;
  uint64_t seed = 0;
};

struct RankingBatch {  // model.hpp:39-43
  Matrix features;
  std::vector<double> labels;
  std::string task_id;
};

enum class PartitionMode { Threshold = MOSES_MODE_THRESHOLD, Ratio = MOSES_MODE_RATIO };

struct XiScores {  // lottery.hpp:15-18
  std::vector<double> xi;
  bool normalized = false;
};

struct ParamMask {  // lottery.hpp:25-32
  std::vector<uint8_t> transferable;
  int phase = 0;
  PartitionMode mode = PartitionMode::Ratio;
  double value = 0.0;
  int64_t popcount() const {
    int64_t c = 0;
    for (uint8_t b : transferable) c += b != 0;
    return c;
  }
};

inline int64_t param_count(const std::vector<int32_t>& dims) {
  const int64_t n = moses_param_count(dims.data(), int32_t(dims.size()));
  if (n < 0) check(int(-n));
  return n;
}

inline CostModelParams init_random(const std::vector<int32_t>& dims, uint64_t seed, bool strict = true) {
  CostModelParams p;
  p.dims = dims;
  const int64_t P = param_count(dims);  // validates dims (BadDims)
  p.params.assign(size_t(P), 0.0);
  p.momentum.assign(size_t(P), 0.0);
  check(moses_init_random(dims.data(), int32_t(dims.size()), seed, strict ? 1 : 0, p.params.data()));
  return p;
}

// Device-resident model: one CUDA stream and workspaces per handle.
class DeviceModel {
 public:
  explicit DeviceModel(const CostModelParams& p, int precision = MOSES_PREC_TF32, int64_t max_rows = 4096)
      : dims_(p.dims), P_(param_count(p.dims)) {
    moses_model_t h = nullptr;
    check(moses_model_create(dims_.data(), int32_t(dims_.size()), precision, max_rows, &h));
    h_.reset(h);
    upload(p);
  }
  void upload(const CostModelParams& p) {
    check(moses_model_upload(h_.get(), p.params.data(), p.momentum.empty() ? nullptr : p.momentum.data(), P_));
  }
  CostModelParams download() const {
    CostModelParams p{dims_, std::vector<double>(size_t(P_)), std::vector<double>(size_t(P_))};
    check(moses_model_download(h_.get(), p.params.data(), p.momentum.data(), P_));
    return p;
  }
  std::vector<double> gradients() const {
    std::vector<double> g(static_cast<size_t>(P_));
    check(moses_gradients_download(h_.get(), g.data(), P_));
    return g;
  }
  moses_model_t handle() const { return h_.get(); }
  const std::vector<int32_t>& dims() const { return dims_; }
  int64_t size() const { return P_; }

 private:
  struct Del {
    void operator()(moses_model_t h) const { moses_model_destroy(h); }
  };
  std::vector<int32_t> dims_;
  int64_t P_;
  std::unique_ptr<moses_model, Del> h_;
};

class AdversaryState {  // lottery.hpp:36-42
 public:
  AdversaryState(const Matrix& replay, int penultimate_dim, double step_size = 0.1) : width_(penultimate_dim) {
    moses_adversary_t h = nullptr;
    check(moses_adversary_create(replay.data.data(), replay.rows, replay.cols, penultimate_dim, step_size, &h));
    h_.reset(h);
  }
  std::vector<double> weight() const {
    std::vector<double> w(static_cast<size_t>(width_));
    double b = 0;
    check(moses_adversary_get(h_.get(), w.data(), width_, &b));
    return w;
  }
  double bias() const {
    std::vector<double> w(static_cast<size_t>(width_));
    double b = 0;
    check(moses_adversary_get(h_.get(), w.data(), width_, &b));
    return b;
  }
  moses_adversary_t handle() const { return h_.get(); }

 private:
  struct Del {
    void operator()(moses_adversary_t h) const { moses_adversary_destroy(h); }
  };
  int width_;
  std::unique_ptr<moses_adversary, Del> h_;
};

// ---- model.hpp
inline std::vector<double> predict(DeviceModel& m, const Matrix& x) {  // model.cpp:169-175
  std::vector<double> s(static_cast<size_t>(x.rows));
  check(moses_predict(m.handle(), x.data.data(), x.rows, x.cols, s.data()));
  return s;
}
inline Matrix penultimate_activations(DeviceModel& m, const Matrix& x) {  // model.cpp:177-183
  Matrix h(x.rows, m.dims()[m.dims().size() - 2]);
  check(moses_penultimate(m.handle(), x.data.data(), x.rows, x.cols, h.data.data()));
  return h;
}
inline double pairwise_ranking_loss(const std::vector<double>& s, const std::vector<double>& y) {
  if (s.size() != y.size()) throw Error(1 + int(ErrorCode::DimMismatch), "scores/labels length mismatch");
  double loss = 0;
  int64_t pairs = 0;
  check(moses_ranking_loss(s.data(), y.data(), int64_t(s.size()), &loss, &pairs));
  return loss;
}
inline std::vector<double> gradients(DeviceModel& m, const RankingBatch& b, const AdversaryState* adv = nullptr,
                                     double beta = 0.0, double* loss_out = nullptr) {  // model.cpp:192-244
  if (int64_t(b.labels.size()) != b.features.rows)
    throw Error(1 + int(ErrorCode::DimMismatch), "batch rows != label count");
  check(moses_gradients(m.handle(), b.features.data.data(), b.labels.data(), b.features.rows, b.features.cols,
                        adv ? adv->handle() : nullptr, beta, loss_out));
  return m.gradients();
}
inline double objective(DeviceModel& m, const RankingBatch& b, const AdversaryState* adv = nullptr, double beta = 0.0) {
  double out = 0;
  check(moses_objective(m.handle(), b.features.data.data(), b.labels.data(), b.features.rows, b.features.cols,
                        adv ? adv->handle() : nullptr, beta, &out));
  return out;
}
// Uses the handle's device gradients (from the last gradients() call, or upload them first).
inline void apply_update(DeviceModel& m, const TrainHyper& h, const ParamMask* mask = nullptr,
                         bool use_momentum = false) {  // model.cpp:263-296
  check(moses_apply_update(m.handle(), h.learning_rate, h.momentum, mask ? mask->transferable.data() : nullptr,
                           mask ? int64_t(mask->transferable.size()) : 0, use_momentum ? 1 : 0));
}
inline double ranking_accuracy(DeviceModel& m, const std::vector<RankingBatch>& batches) {  // model.cpp:298-312
  if (batches.empty()) return 0.0;
  std::vector<double> x, y;
  std::vector<int64_t> off{0};
  const int32_t D = batches[0].features.cols;
  for (const auto& b : batches) {
    x.insert(x.end(), b.features.data.begin(), b.features.data.end());
    y.insert(y.end(), b.labels.begin(), b.labels.end());
    off.push_back(off.back() + b.features.rows);
  }
  double acc = 0;
  int64_t pairs = 0, conc = 0;
  check(moses_ranking_accuracy(m.handle(), x.data(), y.data(), off.data(), int32_t(batches.size()), D, &acc, &pairs,
                               &conc));
  return acc;
}

// ---- lottery.hpp
inline XiScores xi_scores(DeviceModel& m, bool normalize) {  // lottery.cpp:35-57
  XiScores out{std::vector<double>(size_t(m.size())), normalize};
  check(moses_xi_scores(m.handle(), normalize ? 1 : 0, out.xi.data(), m.size()));
  return out;
}
inline ParamMask partition(DeviceModel& m, const XiScores& xi, PartitionMode mode, double value, int phase) {
  check(moses_xi_upload(m.handle(), xi.xi.data(), int64_t(xi.xi.size()), xi.normalized ? 1 : 0));
  ParamMask mask{std::vector<uint8_t>(xi.xi.size()), phase, mode, value};
  int64_t pop = 0;
  check(moses_partition(m.handle(), int(mode), value, phase, mask.transferable.data(), int64_t(xi.xi.size()), &pop));
  return mask;
}
inline void transferable_step(DeviceModel& m, const ParamMask& mask, double alpha) {  // lottery.cpp:92-97
  check(moses_mask_upload(m.handle(), mask.transferable.data(), int64_t(mask.transferable.size())));
  check(moses_transferable_step(m.handle(), alpha));
}
inline void variant_decay(DeviceModel& m, const ParamMask& mask, double alpha, double lambda) {  // lottery.cpp:99-120
  check(moses_mask_upload(m.handle(), mask.transferable.data(), int64_t(mask.transferable.size())));
  check(moses_variant_decay(m.handle(), alpha, lambda));
}
// tuner.cpp:258-262 fused on device: xi -> partition -> transferable_step -> variant_decay
inline ParamMask lottery_step(DeviceModel& m, PartitionMode mode, double value, int phase, double alpha,
                              double lambda) {
  ParamMask mask{std::vector<uint8_t>(size_t(m.size())), phase, mode, value};
  int64_t pop = 0;
  check(moses_lottery_step(m.handle(), int(mode), value, phase, alpha, lambda, mask.transferable.data(), m.size(),
                           &pop));
  return mask;
}
inline double discriminator_cross_entropy(const std::vector<double>& zs, const std::vector<double>& zt) {
  double out = 0;
  check(moses_discriminator_cross_entropy(zs.data(), int64_t(zs.size()), zt.data(), int64_t(zt.size()), &out));
  return out;
}
struct AdversarialResult {
  double discriminator_loss = 0.0;
  double confusion_contribution = 0.0;
};
inline AdversarialResult adversarial_term(AdversaryState& a, const Matrix& hs, const Matrix& ht, double beta) {
  AdversarialResult r;
  check(moses_adversarial_term(a.handle(), hs.data.data(), hs.rows, ht.data.data(), ht.rows,
                               hs.rows ? hs.cols : ht.cols, beta, &r.discriminator_loss, &r.confusion_contribution));
  return r;
}

// ---- search.hpp: candidate order (score desc, pool index asc) and select_batch
inline std::vector<int64_t> topk(const std::vector<double>& scores, int64_t k) {
  if (k > int64_t(scores.size())) k = int64_t(scores.size());
  std::vector<int64_t> idx(static_cast<size_t>(k));
  check(moses_topk(scores.data(), int64_t(scores.size()), k, idx.data()));
  return idx;
}
inline std::vector<int64_t> select_batch(const std::vector<uint64_t>& ordered_hashes,
                                         const std::unordered_set<uint64_t>& already_measured, int64_t batch_size) {
  std::vector<uint64_t> meas(already_measured.begin(), already_measured.end());
  std::vector<int64_t> out(static_cast<size_t>(batch_size > 0 ? batch_size : 1));
  const int64_t n = moses_select_batch(ordered_hashes.data(), int64_t(ordered_hashes.size()), meas.data(),
                                       int64_t(meas.size()), batch_size, out.data());
  if (n < 0) check(int(-n));
  out.resize(size_t(n));
  return out;
}

// ---- space.hpp / oracle.hpp on the device: candidate generation and the simulated hardware
struct KnobSpec {  // space.hpp:16-20 (the kind only matters to validate_task)
  std::string name;
  std::vector<int64_t> domain;
};
struct TaskSpec {  // space.hpp:24-31
  std::string id;
  double work_gflops = 0.0, bytes_per_unit = 0.0, ideal_log2_tiles = 0.0, ideal_log2_unroll = 0.0;
  std::vector<KnobSpec> knobs;
};
struct DeviceSpec {  // oracle.hpp:12-21
  std::string id;
  double peak_gflops = 0.0, parallel_units = 1.0, vector_lanes = 1.0, cache_bytes = 0.0;
  double measure_overhead_ms = 0.0, noise_std = 0.0;
  int repeats = 1;
};
struct Configuration {
  std::vector<int64_t> values;
};
struct BestConfig {
  Configuration config;
  double latency_ms = 0.0;
};
inline std::vector<KnobSpec> default_knob_template() {  // space.cpp:28-36
  return {{"tile_x", {1, 2, 4, 8, 16, 32, 64}}, {"tile_y", {1, 2, 4, 8, 16, 32, 64}}, {"unroll", {0, 16, 64, 512}},
          {"vectorize", {1, 2, 4, 8, 16}}, {"parallel", {1, 2, 4, 8, 16, 32, 64, 128, 256}}};
}
namespace detail {
struct SpaceArrays {
  double task4[4];
  std::vector<int64_t> domains;
  std::vector<int32_t> sizes, roles;
  explicit SpaceArrays(const TaskSpec& t)
      : task4{t.work_gflops, t.bytes_per_unit, t.ideal_log2_tiles, t.ideal_log2_unroll} {
    const char* names[5] = {"tile_x", "tile_y", "unroll", "vectorize", "parallel"};
    for (const auto& k : t.knobs) {
      domains.insert(domains.end(), k.domain.begin(), k.domain.end());
      sizes.push_back(int32_t(k.domain.size()));
      int r = -1;
      for (int i = 0; i < 5; ++i)
        if (k.name == names[i]) r = i;
      roles.push_back(r);
    }
  }
};
inline std::vector<double> device6(const DeviceSpec& d) {
  return {d.peak_gflops, d.parallel_units, d.vector_lanes, d.cache_bytes, d.measure_overhead_ms, d.noise_std};
}
}  // namespace detail

// true_best (oracle.cpp:90-105): exhaustive noise-free optimum, lexicographically first on ties
inline BestConfig true_best(const DeviceSpec& device, const TaskSpec& task) {
  const detail::SpaceArrays a(task);
  BestConfig b;
  b.config.values.resize(task.knobs.size());
  const auto d6 = detail::device6(device);
  check(moses_true_best(d6.data(), a.task4, a.domains.data(), a.sizes.data(), a.roles.data(),
                        int32_t(task.knobs.size()), b.config.values.data(), &b.latency_ms));
  return b;
}

// enumerate_configs + encode_batch + config_hash (space.cpp:140-197) for configs [first, first+n) of the
// enumeration, computed on the device; host copies (row-major n x 16 features, hashes; either may be null).
inline void encode_configs(const TaskSpec& task, uint64_t first, int64_t n, Matrix* features,
                           std::vector<uint64_t>* hashes) {
  const detail::SpaceArrays a(task);
  if (features) *features = Matrix(n, 16);
  if (hashes) hashes->assign(size_t(n), 0);
  check(moses_encode_configs(a.task4, a.domains.data(), a.sizes.data(), a.roles.data(), int32_t(task.knobs.size()),
                             first, n, features ? features->data.data() : nullptr,
                             hashes ? hashes->data() : nullptr));
}

// ---- data.hpp: record store, ranking-batch plans (row ids), epoch seed
struct MeasurementRecord {  // oracle.hpp MeasurementRecord
  std::string task_id;
  std::vector<int64_t> values;
  double throughput_gflops = 0.0, latency_ms = 0.0, wall_cost_ms = 0.0;
  std::string device_id;
  uint64_t seq = 0;
};
struct RecordStore {  // data.hpp:17-19
  std::vector<MeasurementRecord> records;
};
namespace detail {
struct RecordsHandle {
  moses_records_t h = nullptr;
  ~RecordsHandle() { moses_records_destroy(h); }
};
}  // namespace detail
inline RecordStore read_records(const std::string& path) {  // data.cpp:113-126
  detail::RecordsHandle r;
  check(moses_records_read(path.c_str(), &r.h));
  int64_t n = 0, nv = 0;
  int32_t nt = 0, nd = 0;
  check(moses_records_shape(r.h, &n, &nv, &nt, &nd));
  std::vector<int32_t> task(static_cast<size_t>(n)), dev(static_cast<size_t>(n));
  std::vector<int64_t> off(static_cast<size_t>(n) + 1), vals(static_cast<size_t>(nv));
  std::vector<double> thr(static_cast<size_t>(n)), lat(static_cast<size_t>(n)), wall(static_cast<size_t>(n));
  std::vector<uint64_t> seq(static_cast<size_t>(n));
  check(moses_records_export(r.h, task.data(), dev.data(), off.data(), vals.data(), thr.data(), lat.data(), wall.data(),
                             seq.data()));
  RecordStore st;
  st.records.resize(size_t(n));
  for (int64_t i = 0; i < n; ++i) {
    MeasurementRecord& m = st.records[size_t(i)];
    m.task_id = moses_records_task_id(r.h, task[size_t(i)]);
    m.device_id = moses_records_device_id(r.h, dev[size_t(i)]);
    m.values.assign(vals.begin() + off[size_t(i)], vals.begin() + off[size_t(i) + 1]);
    m.throughput_gflops = thr[size_t(i)];
    m.latency_ms = lat[size_t(i)];
    m.wall_cost_ms = wall[size_t(i)];
    m.seq = seq[size_t(i)];
  }
  return st;
}
inline void write_records(const RecordStore& store, const std::string& path) {  // data.cpp:106-111
  detail::RecordsHandle r;
  check(moses_records_create(&r.h));
  for (const auto& m : store.records)
    check(moses_records_append(r.h, m.task_id.c_str(), m.device_id.c_str(), 1, int32_t(m.values.size()),
                               m.values.data(), &m.throughput_gflops, &m.latency_ms, &m.wall_cost_ms, &m.seq));
  check(moses_records_write(r.h, path.c_str()));
}
inline std::vector<std::string> store_task_ids(const RecordStore& store) {  // data.cpp:26-32
  std::vector<std::string> ids;
  for (const auto& r : store.records)
    if (std::find(ids.begin(), ids.end(), r.task_id) == ids.end()) ids.push_back(r.task_id);
  return ids;
}
struct RowBatch {  // RankingBatch as store row ids (features stay wherever the rows live)
  std::string task_id;
  std::vector<int64_t> rows;
};
struct BatchPlan {  // data.hpp:39-42
  std::vector<RowBatch> batches;
  int64_t dropped_singletons = 0;
};
inline BatchPlan make_ranking_batches(const RecordStore& store, int batch_size, uint64_t seed) {  // data.cpp:128-164
  const std::vector<std::string> ids = store_task_ids(store);
  std::vector<const char*> cids;
  for (const auto& t : ids) cids.push_back(t.c_str());
  std::vector<int32_t> rt;
  for (const auto& r : store.records)
    rt.push_back(int32_t(std::find(ids.begin(), ids.end(), r.task_id) - ids.begin()));
  const int64_t n = int64_t(rt.size());
  std::vector<int64_t> rows(size_t(n > 0 ? n : 1)), off(size_t(n / 2 + 2));
  std::vector<int32_t> task(size_t(n / 2 + 1));
  int64_t nb = 0;
  BatchPlan plan;
  check(moses_ranking_plan(rt.data(), n, cids.data(), int32_t(cids.size()), batch_size, seed, rows.data(), off.data(),
                           task.data(), &nb, &plan.dropped_singletons));
  for (int64_t b = 0; b < nb; ++b)
    plan.batches.push_back({ids[size_t(task[size_t(b)])],
                            std::vector<int64_t>(rows.begin() + off[size_t(b)], rows.begin() + off[size_t(b) + 1])});
  return plan;
}
inline uint64_t epoch_seed(uint64_t seed, uint64_t epoch) { return moses_epoch_seed(seed, epoch); }  // tuner.cpp:136-139

// ---- tuner.hpp: pretrain (tuner.cpp:130-156) on the device
struct PretrainLog {  // tuner.hpp PretrainLog
  int64_t dropped_singletons = 0;
  std::vector<double> epoch_mean_loss;
};
// Model {16,512,512,1} from init_random(dims, hyper.seed), hyper.max_epochs epochs of keyed ranking
// batches; every task shares tasks[0]'s knob template (the default task set). precision: operand
// precision of the device model (MOSES_PREC_FP32 for fp32-level parity with the fp64 reference).
inline CostModelParams pretrain(const RecordStore& store, const std::vector<TaskSpec>& tasks, const TrainHyper& hyper,
                                PretrainLog* log = nullptr, int precision = MOSES_PREC_BF16) {
  if (store.records.empty()) check(MOSES_ERR_EMPTY_DATASET);
  if (tasks.empty()) check(MOSES_ERR_INVALID_TASK);
  const detail::SpaceArrays sp(tasks[0]);
  std::vector<const char*> ids;
  std::vector<double> t4;
  for (const auto& t : tasks) {
    ids.push_back(t.id.c_str());
    t4.insert(t4.end(), {t.work_gflops, t.bytes_per_unit, t.ideal_log2_tiles, t.ideal_log2_unroll});
  }
  const size_t nk = tasks[0].knobs.size();
  std::vector<int32_t> rt;
  std::vector<int64_t> vals;
  std::vector<double> thr;
  for (const auto& r : store.records) {
    int32_t t = -1;
    for (size_t k = 0; k < tasks.size(); ++k)
      if (tasks[k].id == r.task_id) t = int32_t(k);
    if (t < 0 || r.values.size() != nk) check(t < 0 ? MOSES_ERR_INVALID_TASK : MOSES_ERR_INVALID_CONFIG);
    rt.push_back(t);
    vals.insert(vals.end(), r.values.begin(), r.values.end());
    thr.push_back(r.throughput_gflops);
  }
  DeviceModel m(init_random({16, 512, 512, 1}, hyper.seed), precision, std::max(hyper.batch_size, 2));
  std::vector<double> losses(size_t(std::max(hyper.max_epochs, 0)));
  int64_t dropped = 0;
  check(moses_pretrain(m.handle(), int32_t(tasks.size()), ids.data(), t4.data(), sp.domains.data(), sp.sizes.data(),
                       sp.roles.data(), int32_t(nk), rt.data(), vals.data(), thr.data(), int64_t(rt.size()),
                       hyper.batch_size, hyper.seed, hyper.max_epochs, hyper.learning_rate, hyper.momentum,
                       losses.data(), &dropped));
  if (log) {
    log->dropped_singletons = dropped;
    log->epoch_mean_loss = losses;
  }
  return m.download();
}

// ---- search.hpp: evolve with the model scorer on the device (search.cpp:41-80)
struct SearchParams {  // search.hpp:13-20
  int population = 128;
  int generations = 4;
  int mutation_count = 4;
  int survivors = 32;
  double epsilon_random = 0.05;
  uint64_t seed = 0;
};
struct ScoredCandidate {  // search.hpp:22-25
  Configuration config;
  double score = 0.0;
};
inline std::vector<ScoredCandidate> evolve(DeviceModel& model, const TaskSpec& task, const SearchParams& p) {
  const detail::SpaceArrays a(task);
  const size_t nk = task.knobs.size();
  const int64_t cap = std::max<int64_t>(p.population, int64_t(p.survivors) * (1 + p.mutation_count));
  std::vector<int64_t> vals(size_t(std::max<int64_t>(cap, 1)) * nk);
  std::vector<double> sc(size_t(std::max<int64_t>(cap, 1)));
  int64_t n = 0;
  check(moses_evolve(model.handle(), nullptr, a.task4, a.domains.data(), a.sizes.data(), a.roles.data(), int32_t(nk),
                     p.population, p.generations, p.mutation_count, p.survivors, p.epsilon_random, p.seed,
                     vals.data(), sc.data(), cap, &n));
  std::vector<ScoredCandidate> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    out[size_t(i)].config.values.assign(vals.begin() + i * int64_t(nk), vals.begin() + (i + 1) * int64_t(nk));
    out[size_t(i)].score = sc[size_t(i)];
  }
  return out;
}

// ---- tuner.hpp: the per-task online loop and the job grid on the device (tuner.cpp:158-286, 307-374)
enum class StrategyKind { Raw = MOSES_STRATEGY_RAW, RandomInit = MOSES_STRATEGY_RANDOM_INIT,
                          PretrainOnly = MOSES_STRATEGY_PRETRAIN_ONLY, VanillaFinetune = MOSES_STRATEGY_VANILLA,
                          Moses = MOSES_STRATEGY_MOSES };
struct LotterySettings {  // tuner.hpp LotterySettings
  PartitionMode mode = PartitionMode::Ratio;
  double value = 0.5;
};
struct TuneBudget {  // tuner.hpp TuneBudget
  int trials_per_task = 64;
  double train_fraction = 0.9;
  int num_batches = 5;
  double cv_threshold = 0.05;
  SearchParams search;
  TrainHyper hyper;
  LotterySettings lottery;
  bool adversary = true;
  int replay_size = 256;
};
struct ControllerTrace {  // tuner.hpp ControllerTrace
  std::vector<double> batch_means, cvs;
  int termination_batch = -1, measured_trials = 0, prediction_trials = 0, unspent_trials = 0;
  std::vector<double> predicted_scores;
};
struct TaskResult {  // tuner.hpp TaskResult
  std::string task_id;
  Configuration best_config;
  double best_latency_ms = 0.0, wall_cost_ms = 0.0;
  std::vector<MeasurementRecord> records;
  ControllerTrace trace;
};
namespace detail {
struct TuneArgs {
  moses_device_spec dev{};
  moses_tune_budget bud{};
  TuneArgs(const DeviceSpec& d, const TuneBudget& b) {
    dev.id = d.id.c_str();
    const auto d6 = device6(d);
    std::copy(d6.begin(), d6.end(), dev.params);
    dev.repeats = d.repeats;
    bud = {b.trials_per_task, b.train_fraction, b.num_batches, b.cv_threshold, b.search.population,
           b.search.generations, b.search.mutation_count, b.search.survivors, b.search.epsilon_random,
           b.hyper.learning_rate, b.hyper.weight_decay, b.hyper.adversary_beta,
           b.lottery.mode == PartitionMode::Threshold ? MOSES_MODE_THRESHOLD : MOSES_MODE_RATIO, b.lottery.value,
           b.adversary ? 1 : 0, b.replay_size};
  }
};
struct ResultBuf {  // caller-owned arrays of moses_task_result
  std::vector<int64_t> values, best;
  std::vector<double> thr, lat, wall, means, cvs, pred;
  moses_task_result r{};
  ResultBuf(const TuneBudget& b, size_t nk)
      : values(size_t(std::max(b.trials_per_task, 1)) * nk), best(nk), thr(size_t(std::max(b.trials_per_task, 1))),
        lat(thr.size()), wall(thr.size()), means(size_t(std::max(b.num_batches, 1))), cvs(means.size()),
        pred(thr.size()) {
    r.capacity = int64_t(thr.size());
    r.values = values.data();
    r.throughput = thr.data();
    r.latency = lat.data();
    r.wall_cost = wall.data();
    r.best_values = best.data();
    r.batch_means = means.data();
    r.cvs = cvs.data();
    r.predicted_scores = pred.data();
  }
  TaskResult take(const TaskSpec& task, const DeviceSpec& dev) const {
    TaskResult t;
    t.task_id = task.id;
    const size_t nk = task.knobs.size();
    t.best_config.values = best;
    t.best_latency_ms = r.best_latency_ms;
    t.wall_cost_ms = r.wall_cost_ms;
    for (int64_t i = 0; i < r.n_records; ++i) {
      MeasurementRecord m;
      m.task_id = task.id;
      m.device_id = dev.id;
      m.values.assign(values.begin() + i * int64_t(nk), values.begin() + (i + 1) * int64_t(nk));
      m.throughput_gflops = thr[size_t(i)];
      m.latency_ms = lat[size_t(i)];
      m.wall_cost_ms = wall[size_t(i)];
      t.records.push_back(std::move(m));
    }
    t.trace.batch_means.assign(means.begin(), means.begin() + r.n_batch_means);
    t.trace.cvs.assign(cvs.begin(), cvs.begin() + r.n_batch_means);
    t.trace.termination_batch = r.termination_batch;
    t.trace.measured_trials = r.measured_trials;
    t.trace.prediction_trials = r.prediction_trials;
    t.trace.unspent_trials = r.unspent_trials;
    t.trace.predicted_scores.assign(pred.begin(), pred.begin() + r.prediction_trials);
    return t;
  }
};
}  // namespace detail
// tune_task on the parameters held by `model` (updated in place: the reference copies initial_model per
// job, tuner.cpp:349 — give each job its own DeviceModel). source_features: the source store's encoded
// rows (the adversary's replay pool), or nullptr.
inline TaskResult tune_task(StrategyKind strategy, DeviceModel& model, const DeviceSpec& device, const TaskSpec& task,
                            const TuneBudget& budget, uint64_t seed, const Matrix* source_features = nullptr) {
  const detail::SpaceArrays a(task);
  const detail::TuneArgs ta(device, budget);
  moses_task_spec ts{task.id.c_str(), {a.task4[0], a.task4[1], a.task4[2], a.task4[3]}, a.domains.data(),
                     a.sizes.data(), a.roles.data(), int32_t(task.knobs.size())};
  detail::ResultBuf buf(budget, task.knobs.size());
  check(moses_tune_task(model.handle(), int32_t(strategy), &ta.dev, &ts, &ta.bud, seed,
                        source_features ? source_features->data.data() : nullptr,
                        source_features ? int64_t(source_features->rows) : 0, &buf.r));
  return buf.take(task, device);
}

}  // namespace moseslab_gpu
