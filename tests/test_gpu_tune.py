"""The tuner's online loop and job grid (tuner.cpp:158-286, 307-374) through the C ABI
(moses_tune_task / moses_tune_jobs) against the oracle's restatement of tune_task (oracle/oracle.py
tune_task, controller.cpp + tuner.cpp control flow) driven by the same device operations: evolve on the
device model, measure() on the device, the strategy's update through the per-call C ABI. Bars: every
measured configuration, measurement, controller trace, predicted score and the final parameters
bit-identical; the reference's own run-level properties (test_tuner.cpp): budget conservation,
Moses(rho = 1, no adversary) == vanilla fine-tuning, worker-pool width invariance."""
import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DEVICE = {"id": "toy", "peak_gflops": 1000.0, "parallel_units": 16.0, "vector_lanes": 8.0,
          "cache_bytes": 1e6, "measure_overhead_ms": 1.0, "noise_std": 0.05, "repeats": 3}
TASKS = [("conv_a", (1.0, 4.0, 6.0, 3.0)), ("conv_b", (2.0, 8.0, 9.0, 6.0))]
DIMS = [16, 64, 64, 1]


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0, moseslab.lib().moses_last_error()
    return moseslab


def budget(ml, **kw):
    b = ml.TuneBudget(trials_per_task=24, train_fraction=0.9, num_batches=4, cv_threshold=0.05, population=32,
                      generations=2, mutation_count=3, survivors=8, replay_size=64)
    for k, v in kw.items():
        setattr(b, k, v)
    return b


def source_rows(n=200):
    return np.random.default_rng(3).random((n, 16))


class DeviceOps:
    """The injected operations of oracle.tune_task, each one call of this library's C ABI."""

    def __init__(self, ml, dm, task_id, task, knobs, b, seed, src, width):
        import torch

        self.ml, self.dm, self.tid, self.task, self.knobs, self.b, self.seed, self.src, self.width = \
            ml, dm, task_id, task, knobs, b, seed, src, width
        self.adv = None
        self.buf = torch.zeros(64, dtype=torch.float64, device="cuda")

    def idx(self, vals):
        i = 0
        for (_, dom), v in zip(self.knobs, vals):
            i = i * len(dom) + dom.index(int(v))
        return i

    def evolve(self, s):
        b = self.b
        vals, scores = self.ml.evolve(self.dm, self.task, self.knobs, b.population, b.generations, b.mutation_count,
                                      b.survivors, b.epsilon_random, s)
        return list(zip(vals.tolist(), scores.tolist()))

    def measure(self, cfgs):
        import torch

        out = []
        for v in cfgs:
            t = torch.zeros(3, dtype=torch.float64, device="cuda")
            p = t.data_ptr()
            self.ml.measure_configs_device(DEVICE, self.tid, self.task, self.knobs, self.seed, self.idx(v), 1,
                                           thr_ptr=C.c_void_p(p), lat_ptr=C.c_void_p(p + 8), wall_ptr=C.c_void_p(p + 16))
            torch.cuda.synchronize()
            out.append(tuple(t.cpu().numpy().tolist()))
        return out

    def encode(self, cfgs):
        import torch

        rows = []
        for v in cfgs:
            self.ml.encode_configs_device(self.task, self.knobs, self.idx(v), 1, self.ml.DTYPE_F64,
                                          C.c_void_p(self.buf.data_ptr()), 16, 16)
            torch.cuda.synchronize()
            rows.append(self.buf[:16].cpu().numpy().copy())
        return np.array(rows)

    def make_adversary(self, rseed):
        rows = self.ml.replay_rows(len(self.src), self.b.replay_size, rseed)
        self.adv = self.ml.make_adversary(self.src[rows], self.width)

    def moses_update(self, rows, labels, b, with_adv):
        x, y = self.encode(rows), np.asarray(labels, dtype=np.float64)
        L = self.ml.lib()
        if with_adv:
            self.ml._ck(L.moses_moses_step(self.dm.h, self.adv.h, self.ml._p(np.ascontiguousarray(x)),
                                           self.ml._p(np.ascontiguousarray(y)), len(y), 16, self.b.adversary_beta,
                                           self.b.lottery_mode, self.b.lottery_value, b, self.b.learning_rate,
                                           self.b.weight_decay, None, None, None))
        else:
            self.ml.gradients(self.dm, self.ml.RankingBatch(x, y))
            self.ml.lottery_step(self.dm, self.b.lottery_mode, self.b.lottery_value, b, self.b.learning_rate,
                                 self.b.weight_decay)

    def vanilla_update(self, rows, labels):
        x, y = self.encode(rows), np.asarray(labels, dtype=np.float64)
        self.ml.gradients(self.dm, self.ml.RankingBatch(x, y))
        self.ml.apply_update(self.dm, self.ml.TrainHyper(learning_rate=self.b.learning_rate, momentum=0.0), None, False)


def same(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return a.shape == b.shape and np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(a[~np.isnan(a)],
                                                                                                 b[~np.isnan(b)])


def check_against_restatement(ml, orc, res, ref, b):
    recs = ref["records"]
    assert res.values.tolist() == [list(map(int, r[0])) for r in recs]
    assert res.throughput.tolist() == [r[1] for r in recs]
    assert res.latency.tolist() == [r[2] for r in recs]
    assert res.wall_cost.tolist() == [r[3] for r in recs]
    assert res.best_values.tolist() == list(map(int, ref["best_values"]))
    assert res.best_latency_ms == ref["best_latency"]
    assert res.wall_cost_ms == ref["wall"]
    assert same(res.batch_means, ref["batch_means"])
    assert same(res.cvs, ref["cvs"]), (res.cvs.tolist(), ref["cvs"], res.batch_means.tolist())
    assert res.termination_batch == ref["termination_batch"]
    assert (res.measured_trials, res.prediction_trials, res.unspent_trials) == \
        (ref["measured"], ref["prediction"], ref["unspent"])
    assert res.predicted_scores.tolist() == ref["predicted"]
    # budget conservation (test_tuner.cpp:185-203)
    assert res.measured_trials + res.prediction_trials + res.unspent_trials == b.trials_per_task


@pytest.mark.parametrize("strategy,adv,prec", [(0, True, "TF32"), (1, True, "TF32"), (2, True, "TF32"),
                                                (3, True, "TF32"), (4, True, "TF32"), (4, False, "TF32"),
                                                (4, True, "BF16X3_WIDE"), (3, True, "BF16")])
def test_tune_task_matches_restatement(ml, orc, strategy, adv, prec):
    dims = [16, 512, 512, 1] if prec == "BF16X3_WIDE" else DIMS
    P = ml.PREC_BF16X3 if prec == "BF16X3_WIDE" else getattr(ml, "PREC_" + prec)
    knobs = orc.default_knob_template()
    tid, task = TASKS[0]
    b = budget(ml, adversary=adv)
    p = ml.init_random(dims, 9)
    a, r = ml.DeviceModel(p, P, 512), ml.DeviceModel(p, P, 512)
    src = source_rows()
    seed = 5
    res = ml.tune_task(a, strategy, DEVICE, tid, task, knobs, b, seed, src)
    ops = DeviceOps(ml, r, tid, task, knobs, b, seed, src, dims[-2])
    ref = orc.tune_task(strategy, ops, tid, knobs, b, seed)
    check_against_restatement(ml, orc, res, ref, b)
    assert np.array_equal(a.download().params, r.download().params)
    if strategy in (0, 2):  # no update: the model is untouched
        assert np.array_equal(a.download().params, np.asarray(p.params, np.float32).astype(np.float64))


def test_moses_ratio_one_without_adversary_equals_vanilla(ml, orc):
    """acceptance.cpp:250-263 / test_tuner.cpp:243-255 at run level: Moses with rho = 1 keeps every scalar
    (the masked step is the unmasked one, no scalar decays) and no adversary == vanilla fine-tuning."""
    knobs = orc.default_knob_template()
    tid, task = TASKS[1]
    p = ml.init_random(DIMS, 13)
    a, v = ml.DeviceModel(p, ml.PREC_TF32, 512), ml.DeviceModel(p, ml.PREC_TF32, 512)
    rm = ml.tune_task(a, ml.STRATEGY_MOSES, DEVICE, tid, task, knobs,
                      budget(ml, adversary=False, lottery_mode=ml.RATIO, lottery_value=1.0), 21)
    rv = ml.tune_task(v, ml.STRATEGY_VANILLA, DEVICE, tid, task, knobs, budget(ml), 21)
    assert rm.values.tolist() == rv.values.tolist() and rm.best_latency_ms == rv.best_latency_ms
    assert np.array_equal(a.download().params, v.download().params)


def test_tune_jobs_grid_equals_single_runs(ml, orc):
    """The (strategy, seed, task) grid on the native worker pool (tuner.cpp:331-374) == every job run alone;
    results independent of the pool width (test_tuner.cpp:409-434)."""
    knobs = orc.default_knob_template()
    p = ml.init_random(DIMS, 17)
    src = source_rows()
    b = budget(ml)
    jobs = [(s, seed, t) for s in (ml.STRATEGY_VANILLA, ml.STRATEGY_MOSES) for seed in (1, 2) for t in (0, 1)]
    runs = {}
    for width in (1, 4):
        models = [ml.DeviceModel(p, ml.PREC_TF32, 512) for _ in jobs]
        runs[width] = (ml.tune_jobs(models, [j[0] for j in jobs], [j[1] for j in jobs], [j[2] for j in jobs], TASKS,
                                    knobs, DEVICE, b, src, threads=width), [m.download().params for m in models])
    for j, (s, seed, t) in enumerate(jobs):
        m = ml.DeviceModel(p, ml.PREC_TF32, 512)
        alone = ml.tune_task(m, s, DEVICE, TASKS[t][0], TASKS[t][1], knobs, b, seed, src)
        for width in (1, 4):
            got, params = runs[width][0][j], runs[width][1][j]
            assert got.values.tolist() == alone.values.tolist(), (j, width)
            assert got.best_latency_ms == alone.best_latency_ms and got.unspent_trials == alone.unspent_trials
            assert same(got.cvs, alone.cvs) and got.predicted_scores.tolist() == alone.predicted_scores.tolist()
            assert np.array_equal(params, m.download().params), (j, width)


def test_tune_errors(ml, orc):
    """plan_split / tune_task failure modes with the reference's codes (controller.cpp:10-32, tuner.cpp:189-192)."""
    knobs = orc.default_knob_template()
    tid, task = TASKS[0]
    dm = ml.DeviceModel(ml.init_random(DIMS, 1), ml.PREC_TF32, 512)
    cases = [(budget(ml, num_batches=1), "invalid-config"), (budget(ml, trials_per_task=3), "invalid-config"),
             (budget(ml, train_fraction=0.0), "invalid-config"),
             (budget(ml, trials_per_task=8, train_fraction=0.4, num_batches=4), "infeasible-split")]
    for b, code in cases:
        with pytest.raises(ml.MosesError) as e:
            ml.tune_task(dm, ml.STRATEGY_VANILLA, DEVICE, tid, task, knobs, b, 1)
        assert e.value.code == code, (b, e.value.code)
    with pytest.raises(ml.MosesError) as e:  # Moses with the adversary needs the source rows
        ml.tune_task(dm, ml.STRATEGY_MOSES, DEVICE, tid, task, knobs, budget(ml), 1)
    assert e.value.code == "adversary-disabled"
    with pytest.raises(ml.MosesError):  # one handle for two jobs
        ml.tune_jobs([dm, dm], [3, 3], [1, 2], [0, 0], TASKS, knobs, DEVICE, budget(ml))
    assert math.isfinite(ml.tune_task(dm, ml.STRATEGY_RAW, DEVICE, tid, task, knobs, budget(ml), 1).best_latency_ms)
