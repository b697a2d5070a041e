// C++ drop-in check: reference test bodies (test_model.cpp, test_lottery.cpp, test_search.cpp)
// re-pointed at the B200 library through include/moses_gpu.hpp. Built by build(), run by
// tests/test_cpp_api.py on a GPU box. Prints one line per case, exits non-zero on failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "moses_gpu.hpp"

using namespace moseslab_gpu;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);      \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

template <class F>
static void expect_error(ErrorCode code, F&& f) {  // test_util.hpp:13-23
  try {
    f();
    std::printf("FAIL expected error %d, nothing thrown\n", int(code));
    ++failures;
  } catch (const Error& e) {
    if (e.code() != code) {
      std::printf("FAIL expected error %d got %d (%s)\n", int(code), int(e.code()), e.what());
      ++failures;
    }
  }
}

static uint64_t splitmix(uint64_t& s) {
  s += 0x9e3779b97f4a7c15ull;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double u01(uint64_t& s) { return double(splitmix(s) >> 11) * 0x1.0p-53; }

int main() {
  // test_model.cpp:77-81
  CHECK(param_count({16, 512, 512, 1}) == 271873);
  // test_model.cpp:100-104
  expect_error(ErrorCode::BadDims, [] { init_random({16, 512, 1}, 0); });
  expect_error(ErrorCode::BadDims, [] { init_random({16, 512, 512, 2}, 0); });
  // test_model.cpp:387-398 (golden predictions; TF32 tolerance)
  {
    DeviceModel m(init_random({16, 512, 512, 1}, 12345), MOSES_PREC_TF32, 128);
    Matrix x(3, 16);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 16; ++c) x(r, c) = (r + 1) * 0.1 + c * 0.01;
    const auto s = predict(m, x);
    const double want[3] = {0.068432722090836534, 0.10419522897402726, 0.14194361818494705};
    for (int i = 0; i < 3; ++i) CHECK(std::abs(s[i] - want[i]) < 2e-3 * 0.142);
  }
  // test_model.cpp:136-139
  {
    DeviceModel m(init_random({4, 8, 8, 1}, 3), MOSES_PREC_TF32, 16);
    expect_error(ErrorCode::DimMismatch, [&] { predict(m, Matrix(2, 5)); });
  }
  // test_model.cpp:155-165
  CHECK(std::abs(pairwise_ranking_loss({2.0, 1.0}, {3.0, 1.0}) - std::log(1.0 + std::exp(-1.0))) < 1e-6);
  CHECK(std::abs(pairwise_ranking_loss({1.0, 1.0}, {3.0, 1.0}) - std::log(2.0)) < 1e-6);
  CHECK(pairwise_ranking_loss({1.0, 1.0}, {1.0, 1.0}) == 0.0);
  // test_model.cpp:205-211 pair-free batch -> zero gradient
  {
    DeviceModel m(init_random({4, 8, 8, 1}, 7), MOSES_PREC_TF32, 16);
    RankingBatch b{Matrix(4, 4), {1.0, 1.0, 1.0, 1.0}, "t"};
    uint64_t s = 20;
    for (auto& v : b.features.data) v = u01(s);
    for (double g : gradients(m, b)) CHECK(g == 0.0);
  }
  // test_model.cpp:267-292 update arithmetic (fp32 device arithmetic)
  {
    CostModelParams p = init_random({4, 8, 8, 1}, 40);
    p.params[0] = 1.0;
    DeviceModel m(p, MOSES_PREC_TF32, 16);
    std::vector<double> g(p.params.size(), 0.0);
    g[0] = 2.0;
    check(moses_gradients_upload(m.handle(), g.data(), int64_t(g.size())));
    TrainHyper h;
    apply_update(m, h, nullptr, false);
    CHECK(std::abs(m.download().params[0] - 0.998) < 1e-7);
  }
  // test_lottery.cpp:138-150 canonical ratio popcounts
  {
    DeviceModel m(init_random({16, 512, 512, 1}, 0), MOSES_PREC_TF32, 16);
    XiScores xi{std::vector<double>(271873), false};
    uint64_t s = 8;
    for (auto& v : xi.xi) v = double(float(u01(s)));
    CHECK(partition(m, xi, PartitionMode::Ratio, 0.01, 0).popcount() == 2719);
    CHECK(partition(m, xi, PartitionMode::Ratio, 0.3, 0).popcount() == 81562);
    CHECK(partition(m, xi, PartitionMode::Ratio, 0.5, 0).popcount() == 135937);
    CHECK(partition(m, xi, PartitionMode::Ratio, 0.7, 0).popcount() == 190312);
    CHECK(partition(m, xi, PartitionMode::Ratio, 1.0, 0).popcount() == 271873);
    expect_error(ErrorCode::InvalidRatio, [&] { partition(m, xi, PartitionMode::Ratio, 1.5, 0); });
    expect_error(ErrorCode::UnnormalizedThreshold, [&] { partition(m, xi, PartitionMode::Threshold, 0.5, 0); });
  }
  // test_lottery.cpp:152-166 ties -> ascending index
  {
    DeviceModel m(init_random({4, 8, 8, 1}, 0), MOSES_PREC_TF32, 16);
    XiScores xi{std::vector<double>(size_t(m.size()), 0.0), false};
    const double v[6] = {0.5, 0.9, 0.5, 0.1, 0.9, 0.5};
    for (int i = 0; i < 6; ++i) xi.xi[i] = v[i];
    const ParamMask mk = partition(m, xi, PartitionMode::Ratio, 3.0 / double(m.size()), 0);
    CHECK(mk.popcount() == 3 && mk.transferable[0] && mk.transferable[1] && mk.transferable[4]);
  }
  // test_lottery.cpp:256-263
  {
    DeviceModel m(init_random({4, 8, 8, 1}, 15), MOSES_PREC_TF32, 16);
    ParamMask mk{std::vector<uint8_t>(size_t(m.size()), 0)};
    expect_error(ErrorCode::UnstableDecay, [&] { variant_decay(m, mk, 1.0, 1.0); });
  }
  // test_lottery.cpp:265-274
  CHECK(std::abs(discriminator_cross_entropy({0, 0, 0}, {0, 0}) - std::log(2.0)) < 1e-15);
  // test_search.cpp:161-172 select_batch dedup
  {
    const auto pos = select_batch({11, 22, 11, 33}, {22}, 10);
    CHECK(pos.size() == 2 && pos[0] == 0 && pos[1] == 3);
  }
  // search.cpp:32-37 order
  {
    const auto idx = topk({0.5, 0.9, 0.5, 0.1, 0.9, 0.5}, 4);
    CHECK(idx.size() == 4 && idx[0] == 1 && idx[1] == 4 && idx[2] == 0 && idx[3] == 2);
  }
  // test_oracle.cpp:313-335: frozen optimum of conv3x3_64 on the shipped server device (true_best_default.json)
  {
    TaskSpec t{"conv3x3_64", 2.0, 8.0, 9.0, 6.0, default_knob_template()};
    DeviceSpec d{"server", 8000.0, 16.0, 8.0, 2000000.0, 2.0, 0.05, 3};
    const BestConfig b = true_best(d, t);
    CHECK((b.config.values == std::vector<int64_t>{8, 64, 64, 8, 16}));
    CHECK(std::abs(b.latency_ms - 0.2500062537535723) < 1e-14 * 0.25);
  }
  // test_space.cpp:142-157, 206-208: feature reference vector and config hash of {16,32,16,8,32}
  {
    TaskSpec t{"conv3x3_64", 2.0, 8.0, 9.0, 5.0, default_knob_template()};
    const uint64_t idx = ((((4ull * 7 + 5) * 4 + 1) * 5 + 3) * 9 + 5);  // mixed radix of (16,32,16,8,32)
    Matrix f;
    std::vector<uint64_t> h;
    encode_configs(t, idx, 1, &f, &h);
    CHECK(std::abs(f(0, 0) - 0.66666666666666663) < 1e-14 && std::abs(f(0, 2) - 0.40874628412503389) < 1e-14);
    CHECK(std::abs(f(0, 7) - 0.10034333188799373) < 1e-14 && f(0, 12) == 0.0);
    CHECK(h[0] == 0xc27c832e9cdb768dull);
  }
  // test_data.cpp:115-143,162-192: record files round trip byte-identically; plans partition per task
  {
    RecordStore st;
    for (int i = 0; i < 46; ++i)
      st.records.push_back({i < 23 ? "a" : "b", {8, 64, 0, 1, 256}, 123.45678901234567 + i, 0.0078125, 1.5, "dev",
                            uint64_t(i)});
    write_records(st, "/tmp/moses_api_records.jsonl");
    const RecordStore back = read_records("/tmp/moses_api_records.jsonl");
    CHECK(back.records.size() == 46 && back.records[30].throughput_gflops == st.records[30].throughput_gflops &&
          back.records[45].task_id == "b" && back.records[7].values == st.records[7].values);
    const BatchPlan plan = make_ranking_batches(back, 8, 99);
    int rows_a = 0, rows_b = 0;
    for (const auto& b : plan.batches) {
      CHECK(b.rows.size() >= 2 && b.rows.size() <= 8);
      for (int64_t r : b.rows) CHECK(back.records[size_t(r)].task_id == b.task_id);
      (b.task_id == "a" ? rows_a : rows_b) += int(b.rows.size());
    }
    CHECK(plan.batches.size() == 6 && plan.dropped_singletons == 0 && rows_a == 23 && rows_b == 23);
    expect_error(ErrorCode::InvalidConfig, [&] { make_ranking_batches(back, 1, 0); });
    CHECK(epoch_seed(5, 1) != epoch_seed(5, 2));
    std::remove("/tmp/moses_api_records.jsonl");
  }
  // test_tuner.cpp:320-340 shape: pretrain logs epoch losses and counts dropped singletons; the
  // loss falls over the epochs on a learnable store
  {
    TaskSpec ta{"a", 1.0, 4.0, 6.0, 3.0, default_knob_template()};
    TaskSpec tb{"b", 1.0, 4.0, 9.0, 3.0, default_knob_template()};
    RecordStore st;
    for (int i = 0; i < 131; ++i) {
      const int64_t tx = int64_t(1) << (i % 7), ty = int64_t(1) << ((i / 7) % 7);
      st.records.push_back({i % 2 ? "a" : "b", {tx, ty, 16, 4, 16}, double(tx * ty) + 0.5 * (i % 5), 1.0, 1.0, "d",
                            uint64_t(i)});
    }
    TrainHyper h;
    h.max_epochs = 6;
    h.batch_size = 16;
    h.learning_rate = 0.01;
    PretrainLog log;
    const CostModelParams p = pretrain(st, {ta, tb}, h, &log);
    CHECK(p.params.size() == size_t(param_count({16, 512, 512, 1})) && log.epoch_mean_loss.size() == 6);
    CHECK(log.dropped_singletons == 1);  // "a" has 65 rows: 4 x 16 + 1
    CHECK(log.epoch_mean_loss.back() < log.epoch_mean_loss.front());
    RecordStore bad = st;
    bad.records[3].values[2] = 17;  // not an unroll value
    expect_error(ErrorCode::InvalidConfig, [&] { pretrain(bad, {ta, tb}, h); });
    expect_error(ErrorCode::EmptyDataset, [&] { pretrain(RecordStore{}, {ta, tb}, h); });
  }
  // test_search.cpp:82-120: evolve's result is sorted by score then config, of the refilled size
  {
    TaskSpec t{"conv3x3_64", 2.0, 8.0, 9.0, 5.0, default_knob_template()};
    DeviceModel m(init_random({16, 512, 512, 1}, 3), MOSES_PREC_BF16, 1024);
    SearchParams sp;
    sp.seed = 4;
    const auto pop = evolve(m, t, sp);
    CHECK(pop.size() == 160);
    bool sorted = true;
    for (size_t i = 1; i < pop.size(); ++i)
      sorted = sorted && (pop[i - 1].score > pop[i].score ||
                          (pop[i - 1].score == pop[i].score && pop[i - 1].config.values <= pop[i].config.values));
    CHECK(sorted);
    SearchParams bad = sp;
    bad.survivors = 500;
    expect_error(ErrorCode::InvalidConfig, [&] { evolve(m, t, bad); });
  }
  // test_tuner.cpp:139-203: tune_task's budget is conserved (measured + predicted + unspent = trials), the
  // best latency is the minimum of the measured ones, and the plan rejects infeasible splits
  {
    TaskSpec t{"conv3x3_64", 2.0, 8.0, 9.0, 5.0, default_knob_template()};
    DeviceSpec d{"toy", 1000.0, 16.0, 8.0, 1e6, 1.0, 0.05, 3};
    TuneBudget b;
    b.trials_per_task = 20;
    b.num_batches = 4;
    b.search.population = 32;
    b.search.generations = 1;
    b.search.survivors = 8;
    b.search.mutation_count = 3;
    b.adversary = false;
    for (StrategyKind s : {StrategyKind::Raw, StrategyKind::PretrainOnly, StrategyKind::VanillaFinetune,
                           StrategyKind::Moses}) {
      DeviceModel m(init_random({16, 64, 64, 1}, 7), MOSES_PREC_TF32, 512);
      const TaskResult r = tune_task(s, m, d, t, b, 3);
      CHECK(r.trace.measured_trials + r.trace.prediction_trials + r.trace.unspent_trials == b.trials_per_task);
      double best = 1e300;
      for (const auto& rec : r.records) best = std::min(best, rec.latency_ms);
      CHECK(!r.records.empty() && best == r.best_latency_ms);
    }
    TuneBudget bad = b;
    bad.trials_per_task = 8;
    bad.train_fraction = 0.4;
    DeviceModel m(init_random({16, 64, 64, 1}, 7), MOSES_PREC_TF32, 512);
    expect_error(ErrorCode::InfeasibleSplit, [&] { tune_task(StrategyKind::VanillaFinetune, m, d, t, bad, 3); });
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
