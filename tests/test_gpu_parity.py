"""Parity of the sm_100a path (through the C ABI) against the CPU oracle.

Tolerances (north star): tensor-core TF32/bf16 GEMM stages <= 1e-3 normwise
relative (max |d| / max |ref|); masks, top-k indices, popcounts, accuracy counts
bit-exact on identical inputs in identical precision (fp32 on both sides).
bf16 mode is the throughput mode: its error is measured and bounded looser.
"""
import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_TF32 = 1e-3
TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0, moseslab.lib().moses_last_error()
    return moseslab


def nrel(got, ref):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


def rows(n, d, seed):
    return np.random.default_rng(seed).random((n, d))


def labels(n, seed):
    return 0.1 + np.random.default_rng(seed).random(n)


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def grad_close(got, ref, q_tol=1e-3, frob_tol=2e-2):
    """Robust gradient agreement: 99.9% of entries within q_tol * max|ref| and a relative
    Frobenius error below frob_tol. A single ReLU-kink sign flip (|z| below the fp32
    accumulation error) moves one row's contribution to one column — a few entries — which
    this tolerates while any systematic error fails it."""
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    d = np.abs(got - ref) / max(np.max(np.abs(ref)), 1e-300)
    frob = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
    return float(np.quantile(d, 0.999)) <= q_tol and frob <= frob_tol, (float(np.quantile(d, 0.999)), frob)


# ---------------------------------------------------------------- forward
def test_golden_model_predictions(ml):
    p = ml.init_random([16, 512, 512, 1], 12345)
    x = np.array([[(r + 1) * 0.1 + c * 0.01 for c in range(16)] for r in range(3)])
    want = [0.068432722090836534, 0.10419522897402726, 0.14194361818494705]
    from precision_model import device_forward

    # the three golden scores are small sums of 512 mixed-sign terms (cancellation): TF32 operand
    # rounding alone moves them by ~1e-3 relative; the device matches its operand-precision model
    # to fp32 accumulation order.
    for prec, tol, mode in ((ml.PREC_TF32, 2e-3, "tf32"), (ml.PREC_BF16, TOL_BF16, "bf16")):
        dm = ml.DeviceModel(p, prec, 128)
        got = ml.predict(dm, x)
        assert nrel(got, want) < tol
        s_model = device_forward([16, 512, 512, 1], p.params, x, mode)[0]
        assert np.max(np.abs(got - s_model)) < 1e-5


@pytest.mark.parametrize("dims", [[4, 8, 8, 1], [16, 512, 512, 1], [164, 256, 256, 1], [164, 512, 512, 1],
                                  [164, 512, 512, 512, 512, 1], [33, 72, 40, 1]])
@pytest.mark.parametrize("n", [1, 5, 300])
def test_predict_vs_oracle(ml, orc, dims, n):
    """fp64 oracle within the TF32 tolerance (normwise over >= 5 rows); any n against the
    operand-precision model (same rounding as the device) at 1e-5."""
    from precision_model import device_forward

    p = ml.init_random(dims, 11, strict=False)
    x = rows(n, dims[0], n)
    ref, h_ref = orc.forward(dims, p.params, x)
    dm = ml.DeviceModel(p, ml.PREC_TF32, 512)
    s = ml.predict(dm, x)
    if n >= 5:
        assert nrel(s, ref) < TOL_TF32
        assert nrel(ml.penultimate_activations(dm, x), h_ref) < TOL_TF32
    for mode, handle in (("tf32", dm), ("bf16", ml.DeviceModel(p, ml.PREC_BF16, 512))):
        s_model, _, _, _, _ = device_forward(dims, p.params, x, mode)
        got = s if mode == "tf32" else ml.predict(handle, x)
        assert np.max(np.abs(got - s_model)) <= 2e-4 * max(1.0, np.max(np.abs(s_model)))
    if n >= 5:
        db = ml.DeviceModel(p, ml.PREC_BF16, 512)
        assert nrel(ml.predict(db, x), ref) < TOL_BF16


def test_predict_large_chunked(ml, orc):
    dims = [164, 512, 512, 1]
    p = ml.init_random(dims, 5)
    x = rows(5000, 164, 1)
    dm = ml.DeviceModel(p, ml.PREC_TF32, 1024)  # forces 5 chunks
    ref, _ = orc.forward(dims, p.params, x, threads=8)
    assert nrel(ml.predict(dm, x), ref) < TOL_TF32


def test_predict_rejects_wrong_width(ml):
    dm = ml.DeviceModel(ml.init_random([4, 8, 8, 1], 3), ml.PREC_TF32, 16)
    with pytest.raises(ml.MosesError) as e:
        ml.predict(dm, rows(2, 5, 0))
    assert e.value.code == "dim-mismatch"


def test_predict_purity_duplicate_rows(ml):
    dm = ml.DeviceModel(ml.init_random([4, 8, 8, 1], 2), ml.PREC_TF32, 16)
    x = rows(2, 4, 9)
    x[1] = x[0]
    s = ml.predict(dm, x)
    assert s[0] == s[1]


def test_pooled_predict_reduces_to_predict_and_matches_oracle(ml, orc):
    dims = [164, 256, 256, 1]
    p = ml.init_random(dims, 4)
    off = orc.synth_offsets(3, 200, 8)
    x = rows(int(off[-1]), 164, 2)
    dm = ml.DeviceModel(p, ml.PREC_TF32, 1024)
    got = ml.predict_pooled(dm, x, off)
    _, h = orc.forward(dims, p.params, x)
    pooled = orc.segment_sum(h, off)
    ref = pooled @ p.params[-257:-1] + p.params[-1]
    assert nrel(got, ref) < TOL_TF32
    # all segments of length 1 == predict
    one = np.arange(41, dtype=np.int64)
    assert nrel(ml.predict_pooled(dm, x[:40], one), ml.predict(dm, x[:40])) < 1e-6


# ---------------------------------------------------------------- gradients
# Raw gradients are compared with the reference algorithm evaluated on the device's operands
# (tests/precision_model.py: identical bf16 / tf32 rounding, fp64 arithmetic) — comparing raw
# gradients of a reduced-precision forward with an fp64 one is dominated by ReLU-kink sign flips
# (test_model.cpp:61-71 redraws kink-grazing trials for the same reason). The fp64 oracle bounds
# what the north star names: loss and updated weights within 1e-3.
GRAD_DIMS = [[4, 8, 8, 1], [16, 512, 512, 1], [164, 256, 256, 1], [164, 512, 512, 512, 512, 1]]


@pytest.mark.parametrize("dims", GRAD_DIMS)
@pytest.mark.parametrize("n", [2, 12, 512])
@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_gradients_vs_precision_model(ml, orc, dims, n, mode):
    from precision_model import device_gradients

    p = ml.init_random(dims, 21, strict=False)
    x, y = rows(n, dims[0], 7), labels(n, 8)
    g_ref, loss_ref = device_gradients(dims, p.params, x, y, mode)
    dm = ml.DeviceModel(p, ml.PREC_TF32 if mode == "tf32" else ml.PREC_BF16, 1024)
    g, loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
    deep = len(dims) > 4 and n >= 512  # 4 hidden layers x 512 rows: more kink candidates
    ok, why = grad_close(g, g_ref, q_tol=5e-3 if deep else 1e-3)
    assert ok, why
    _, loss64 = orc.gradients(dims, p.params, x, y)
    assert abs(loss - loss64) <= TOL_TF32 * max(1.0, abs(loss64))


@pytest.mark.parametrize("dims", [[16, 512, 512, 1], [164, 512, 512, 1]])
@pytest.mark.parametrize("n", [1500, 3000])
@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_gradients_large_batch_vs_precision_model(ml, orc, dims, n, mode):
    """Ranking batches past the 16-CTA cluster form's limits take the grid form of the fused step."""
    from precision_model import device_gradients

    p = ml.init_random(dims, 22)
    x, y = rows(n, dims[0], 9), labels(n, 10)
    g_ref, _ = device_gradients(dims, p.params, x, y, mode)
    dm = ml.DeviceModel(p, ml.PREC_TF32 if mode == "tf32" else ml.PREC_BF16, 4096)
    g, loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
    ok, why = grad_close(g, g_ref, q_tol=2e-3)
    assert ok, why
    _, loss64 = orc.gradients(dims, p.params, x, y, threads=8)
    assert abs(loss - loss64) <= TOL_TF32 * max(1.0, abs(loss64))


@pytest.mark.parametrize("dims", GRAD_DIMS)
@pytest.mark.parametrize("prec", [1, 0])
def test_train_step_updated_weights_vs_oracle(ml, orc, dims, prec):
    """tuner.cpp:146-147 (gradients + momentum update) vs the fp64 oracle: updated weights and loss."""
    p = ml.init_random(dims, 3, strict=False)
    x, y = rows(512, dims[0], 1), labels(512, 2)
    dm = ml.DeviceModel(p, prec, 512)
    w, mom = p.params.copy(), np.zeros_like(p.params)
    for it in range(3):
        loss_ref = orc.train_step_f64(dims, w, mom, x, y, 0.001, 0.9, threads=8)
        loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)[1]
        ml.apply_update(dm, ml.TrainHyper(learning_rate=0.001, momentum=0.9), None, True)
        assert abs(loss - loss_ref) <= TOL_TF32 * max(1.0, abs(loss_ref))
    got = dm.download()
    assert nrel(got.params, w) < 1e-3  # the north-star bound: updated weights within 1e-3
    # momentum = accumulated raw gradients of a reduced-precision forward vs fp64 (ReLU-kink flips,
    # bf16 dZ quantisation): bounded loosely here; the tight raw-gradient check is against the
    # operand-precision model (test_gradients_vs_precision_model).
    frob = np.linalg.norm(got.momentum - mom) / np.linalg.norm(mom)
    assert frob < (0.5 if prec == 0 else 0.2)


@pytest.mark.parametrize("beta", [0.0, 0.01, 0.5])
@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_gradients_with_adversary(ml, orc, beta, mode):
    from precision_model import device_gradients

    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 31)
    x, y = rows(12, 16, 1), labels(12, 2)
    replay = rows(256, 16, 3)
    u = np.random.default_rng(4).normal(0, 0.05, 512)
    c = 0.03
    g_ref, loss_ref = device_gradients(dims, p.params, x, y, mode, (u, c, replay), beta)
    _, loss64 = orc.gradients(dims, p.params, x, y, (u, c, replay), beta)
    adv = ml.make_adversary(replay, 512, 7)
    adv.set(u, c)
    dm = ml.DeviceModel(p, ml.PREC_TF32 if mode == "tf32" else ml.PREC_BF16, 512)
    g, loss = ml.gradients(dm, ml.RankingBatch(x, y), adv, beta, want_loss=True)
    ok, why = grad_close(g, g_ref)
    assert ok, why
    assert abs(loss - loss64) <= TOL_TF32 * max(1.0, abs(loss64))
    if beta == 0.0:  # model.cpp:213-215: adversary-free gradient bit-for-bit
        g0 = ml.gradients(dm, ml.RankingBatch(x, y))
        assert np.array_equal(g, g0)


def test_gradients_pair_free_and_empty(ml):
    dm = ml.DeviceModel(ml.init_random([4, 8, 8, 1], 7), ml.PREC_TF32, 16)
    g = ml.gradients(dm, ml.RankingBatch(rows(4, 4, 20), np.ones(4)))
    assert np.all(g == 0)
    g = ml.gradients(dm, ml.RankingBatch(np.zeros((0, 4)), np.zeros(0)))
    assert np.all(g == 0)


def test_gradients_deterministic(ml):
    dm = ml.DeviceModel(ml.init_random([164, 512, 512, 1], 1), ml.PREC_BF16, 1024)
    b = ml.RankingBatch(rows(1000, 164, 5), labels(1000, 6))
    a = ml.gradients(dm, b)
    assert np.array_equal(a, ml.gradients(dm, b))


def test_objective_matches_gradient_loss(ml, orc):
    dims = [4, 8, 8, 1]
    p = ml.init_random(dims, 30)
    x, y = rows(6, 4, 31), labels(6, 32)
    replay = rows(7, 4, 33)
    adv = ml.make_adversary(replay, 8, 1)
    adv.set(np.linspace(-0.2, 0.2, 8), 0.1)
    dm = ml.DeviceModel(p, ml.PREC_TF32, 64)
    _, loss = ml.gradients(dm, ml.RankingBatch(x, y), adv, 0.01, want_loss=True)
    assert ml.objective(dm, ml.RankingBatch(x, y), adv, 0.01) == pytest.approx(loss, rel=1e-12)
    ref = orc.objective(dims, p.params, x, y, (np.linspace(-0.2, 0.2, 8), 0.1, replay), 0.01)
    assert loss == pytest.approx(ref, rel=TOL_TF32)


# ---------------------------------------------------------------- ranking
@pytest.mark.parametrize("n", [0, 1, 2, 8, 513, 4096])
def test_ranking_loss_vs_oracle(ml, orc, n):
    rng = np.random.default_rng(n)
    s = f32(rng.uniform(-2, 2, n))
    y = f32(np.round(rng.random(n) * 20) / 20)  # ties in labels
    ref, _, _ = orc.ranking_terms(s, y)
    got = ml.pairwise_ranking_loss(s, y)
    assert got == pytest.approx(ref, rel=1e-5, abs=1e-12)


def test_ranking_loss_hand_cases(ml):
    assert ml.pairwise_ranking_loss([2.0, 1.0], [3.0, 1.0]) == pytest.approx(math.log(1 + math.exp(-1)), rel=1e-6)
    assert ml.pairwise_ranking_loss([1.0, 1.0], [3.0, 1.0]) == pytest.approx(math.log(2), rel=1e-6)
    assert ml.pairwise_ranking_loss([1.0, 1.0], [1.0, 1.0]) == 0.0


def test_ranking_accuracy_counts_exact(ml, orc):
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 44)
    dm = ml.DeviceModel(p, ml.PREC_TF32, 512)
    batches = [ml.RankingBatch(rows(n, 16, n), np.round(labels(n, n + 1), 2)) for n in (3, 12, 100, 1)]
    acc = ml.ranking_accuracy(dm, batches)
    pairs = conc = 0
    for b in batches:
        s = ml.predict(dm, b.features).astype(np.float32)
        pp, cc = orc.accuracy_counts(s, np.asarray(b.labels, np.float32))
        pairs, conc = pairs + pp, conc + cc
    assert acc == (conc / pairs if pairs else 0.0)


# ---------------------------------------------------------------- updates (bit-exact on identical fp32 inputs)
def _f32_params(p):
    return ml_params(p.dims, f32(p.params))


def ml_params(dims, w, mom=None):
    from paper_2201_05752_b200.moseslab import CostModelParams

    return CostModelParams(list(dims), w, mom)


@pytest.mark.parametrize("use_momentum", [False, True])
@pytest.mark.parametrize("masked", [False, True])
def test_apply_update_bit_exact(ml, orc, use_momentum, masked):
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 40)
    w = f32(p.params)
    mom = f32(np.random.default_rng(1).normal(0, 1e-3, len(w)))
    g = f32(np.random.default_rng(2).normal(0, 1e-2, len(w)))
    mask = np.random.default_rng(3).random(len(w)) < 0.5 if masked else None
    dm = ml.DeviceModel(ml_params(dims, w, mom), ml.PREC_BF16, 16)
    ml.apply_update(dm, ml.TrainHyper(learning_rate=0.001, momentum=0.9),
                    ml.ParamMask(mask) if masked else None, use_momentum, grads=g)
    got = dm.download()
    ref_w, ref_m = orc.apply_update(w.astype(np.float32), mom.astype(np.float32), g.astype(np.float32), 0.001, 0.9,
                                    mask, use_momentum)
    assert np.array_equal(got.params, ref_w.astype(np.float64))
    assert np.array_equal(got.momentum, ref_m.astype(np.float64))


def test_update_arithmetic_kat(ml):
    p = ml.init_random([4, 8, 8, 1], 40)
    p.params[0] = 1.0
    g = np.zeros_like(p.params); g[0] = 2.0
    dm = ml.DeviceModel(p, ml.PREC_TF32, 16)
    before = dm.download().params
    ml.apply_update(dm, ml.TrainHyper(learning_rate=0.001), None, False, grads=g)
    after = dm.download().params
    assert after[0] == pytest.approx(0.998, rel=1e-7)
    assert np.array_equal(after[1:], before[1:])


# ---------------------------------------------------------------- lottery (bit-exact)
def test_xi_scores_bit_exact(ml, orc):
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 9)
    w = f32(p.params)
    g = f32(np.random.default_rng(5).normal(0, 1e-2, len(w)))
    g[::7] = 0.0
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_TF32, 16)
    for norm in (False, True):
        xi = ml.xi_scores(dm, norm, grads=g)
        ref = orc.xi_scores(w.astype(np.float32), g.astype(np.float32), norm)
        assert np.array_equal(xi.xi, ref.astype(np.float64))


@pytest.mark.parametrize("rho,want", [(0.01, 2719), (0.3, 81562), (0.5, 135937), (0.7, 190312), (1.0, 271873)])
def test_ratio_popcounts_canonical(ml, orc, rho, want):
    n = 271873
    xi = np.array([(orc.lib().orc_splitmix_at(8, i + 1) >> 11) * 2.0 ** -53 for i in range(n)])
    xi32 = f32(xi)
    dm = ml.DeviceModel(ml.init_random([16, 512, 512, 1], 0), ml.PREC_TF32, 16)
    mask = ml.partition(dm, ml.XiScores(xi32, False), ml.RATIO, rho, 0)
    assert mask.popcount() == want
    ref = orc.partition(xi32.astype(np.float32), False, orc.RATIO, rho)
    assert np.array_equal(mask.transferable, ref)


def test_ratio_tie_break_and_heavy_zero_ties(ml, orc):
    dm = ml.DeviceModel(ml.init_random([4, 8, 8, 1], 0), ml.PREC_TF32, 16)
    P = dm.P
    xi = np.zeros(P)
    xi[:6] = [0.5, 0.9, 0.5, 0.1, 0.9, 0.5]
    for rho in (3 / P, 0.25, 0.5, 0.9):
        m = ml.partition(dm, ml.XiScores(xi, False), ml.RATIO, rho, 1)
        assert np.array_equal(m.transferable, orc.partition(xi.astype(np.float32), False, orc.RATIO, rho))
    m = ml.partition(dm, ml.XiScores(xi, False), ml.RATIO, 3 / P, 1)
    assert sorted(np.flatnonzero(m.transferable)) == [0, 1, 4]
    # half the scalars tied at zero (README.md:106-113) at canonical scale
    n = 271873
    rng = np.random.default_rng(3)
    xi = f32(np.where(rng.random(n) < 0.5, 0.0, rng.random(n)))
    xi[100:5000] = xi[99]  # a long run of equal non-zero keys too
    dm2 = ml.DeviceModel(ml.init_random([16, 512, 512, 1], 0), ml.PREC_TF32, 16)
    for rho in (0.3, 0.5, 0.51, 0.7):
        m = ml.partition(dm2, ml.XiScores(xi, False), ml.RATIO, rho, 0)
        assert np.array_equal(m.transferable, orc.partition(xi.astype(np.float32), False, orc.RATIO, rho))


def test_threshold_partition(ml, orc):
    dm = ml.DeviceModel(ml.init_random([4, 8, 8, 1], 0), ml.PREC_TF32, 16)
    xi = np.zeros(dm.P)
    xi[:5] = [0.2, 0.5, 0.50000001, 0.9, 1.0]
    m = ml.partition(dm, ml.XiScores(xi, True), ml.THRESHOLD, 0.5, 3)
    ref = orc.partition(f32(xi).astype(np.float32), True, orc.THRESHOLD, 0.5)
    assert np.array_equal(m.transferable, ref)
    with pytest.raises(ml.MosesError) as e:
        ml.partition(dm, ml.XiScores(xi, False), ml.THRESHOLD, 0.5, 0)
    assert e.value.code == "unnormalized-threshold"
    for bad in (0.0, 1.5, -0.1):
        with pytest.raises(ml.MosesError) as e:
            ml.partition(dm, ml.XiScores(xi, False), ml.RATIO, bad, 0)
        assert e.value.code == "invalid-ratio"


@pytest.mark.parametrize("mode,value", [(2, 0.01), (2, 0.5), (2, 0.7), (1, 0.5), (1, 0.05), (2, 1.0)])
def test_fused_lottery_step_bit_exact(ml, orc, mode, value):
    """tuner.cpp:258-262: xi -> partition -> transferable_step -> variant_decay, fused on device."""
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 13)
    w = f32(p.params)
    g = f32(np.random.default_rng(6).normal(0, 1e-2, len(w)))
    g[np.random.default_rng(7).random(len(w)) < 0.4] = 0.0  # zero-gradient ties
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_BF16, 16)
    dm.set_gradients(g)
    mask = ml.lottery_step(dm, mode, value, 2, 0.001, 0.01)
    got = dm.download().params
    w32, g32 = w.astype(np.float32), g.astype(np.float32)
    xi = orc.xi_scores(w32, g32, mode == 1)
    ref_mask = orc.partition(xi, mode == 1, mode, value)
    ref_w, _ = orc.apply_update(w32, np.zeros_like(w32), g32, 0.001, 0.0, ref_mask, False)
    ref_w = orc.variant_decay(ref_w, ref_mask, 0.001, 0.01)
    assert np.array_equal(mask.transferable, ref_mask)
    assert np.array_equal(got, ref_w.astype(np.float64))


def test_step_and_decay_separate_ops(ml, orc):
    dims = [4, 8, 8, 1]
    p = ml.init_random(dims, 10)
    w = f32(p.params)
    g = np.ones_like(w)
    mask = np.zeros(len(w), bool); mask[0] = True; mask[32] = True
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_TF32, 16)
    ml.transferable_step(dm, ml.ParamMask(mask), 0.01, grads=g)
    got = dm.download().params
    exp = w.astype(np.float32).copy()
    exp[0] = np.float32(exp[0]) - np.float32(0.01)
    exp[32] = np.float32(exp[32]) - np.float32(0.01)
    assert np.array_equal(got, exp.astype(np.float64))
    ml.variant_decay(dm, ml.ParamMask(mask), 0.001, 0.01)
    ref = orc.variant_decay(exp, mask, 0.001, 0.01)
    assert np.array_equal(dm.download().params, ref.astype(np.float64))
    before = dm.download().params
    ml.variant_decay(dm, None, 0.5, 0.0)
    assert before.tobytes() == dm.download().params.tobytes()
    for a, l in ((1.0, 1.0), (2.0, 0.5), (0.1, -0.5)):
        with pytest.raises(ml.MosesError) as e:
            ml.variant_decay(dm, None, a, l)
        assert e.value.code == "unstable-decay"
    with pytest.raises(ml.MosesError) as e:
        ml.transferable_step(dm, ml.ParamMask(np.ones(7, bool)), 0.01)
    assert e.value.code == "shape-mismatch"


def test_moses_rho1_equals_vanilla(ml):
    """acceptance.cpp:250-263: Moses with rho = 1 and no adversary == vanilla fine-tune, bit-exact."""
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 99)
    b = ml.RankingBatch(rows(12, 16, 1), labels(12, 2))
    a = ml.DeviceModel(p, ml.PREC_BF16, 64)
    v = ml.DeviceModel(p, ml.PREC_BF16, 64)
    for _ in range(3):
        ml.gradients(a, b)
        ml.lottery_step(a, ml.RATIO, 1.0, 0, 0.001, 0.01)
        ml.gradients(v, b)
        ml.apply_update(v, ml.TrainHyper(learning_rate=0.001), None, False)
    assert np.array_equal(a.download().params, v.download().params)


def test_adam_update_vs_oracle(ml, orc):
    dims = [16, 512, 512, 1]
    w = f32(ml.init_random(dims, 3).params)
    g = f32(np.random.default_rng(1).normal(0, 1e-2, len(w)))
    mask = np.random.default_rng(2).random(len(w)) < 0.5
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_TF32, 16)
    dm.set_gradients(g)
    ml.adam_update(dm, 1e-3, 0.9, 0.999, 1e-8, 1, ml.ParamMask(mask))
    ref, _, _ = orc.adam(w.astype(np.float32), np.zeros(len(w), np.float32), np.zeros(len(w), np.float32),
                         g.astype(np.float32), 1e-3, 0.9, 0.999, 1e-8, 1, mask)
    assert nrel(dm.download().params, ref) < 1e-6


# ---------------------------------------------------------------- adversary
def test_adversarial_term_vs_oracle(ml, orc):
    rng = np.random.default_rng(0)
    hs, ht = rng.random((64, 32)), rng.random((24, 32))
    hs[:, 0] += 2
    adv = ml.make_adversary(rows(4, 4, 1), 32, 2)
    aw, ab = np.zeros(32), 0.0
    for _ in range(20):
        res = ml.adversarial_term(adv, hs, ht, 0.01)
        aw, ab, lref = orc.adversarial_term(aw, ab, hs, ht)
        assert res.discriminator_loss == pytest.approx(lref, rel=1e-4)
        assert res.confusion_contribution == pytest.approx(-0.01 * res.discriminator_loss, rel=1e-12)
    assert nrel(adv.weight, aw) < 1e-4 and adv.bias == pytest.approx(ab, rel=1e-4, abs=1e-6)


def test_adversary_validation(ml):
    with pytest.raises(ml.MosesError) as e:
        ml.make_adversary(np.zeros((0, 4)), 4)
    assert e.value.code == "adversary-disabled"
    with pytest.raises(ml.MosesError) as e:
        ml.make_adversary(rows(3, 4, 0), 0)
    assert e.value.code == "bad-dims"
    adv = ml.make_adversary(rows(3, 4, 1), 4)
    with pytest.raises(ml.MosesError) as e:
        ml.adversarial_term(adv, rows(3, 5, 2), rows(3, 4, 3), 0.0)
    assert e.value.code == "dim-mismatch"
    with pytest.raises(ml.MosesError) as e:
        ml.adversarial_term(adv, np.zeros((0, 4)), rows(3, 4, 3), 0.0)
    assert e.value.code == "adversary-disabled"


def test_discriminator_ce(ml, orc):
    z = np.zeros(5)
    assert ml.discriminator_cross_entropy(z, z) == pytest.approx(math.log(2), rel=1e-15)
    zs, zt = np.random.default_rng(1).normal(0, 3, 17), np.random.default_rng(2).normal(0, 3, 9)
    assert ml.discriminator_cross_entropy(zs, zt) == pytest.approx(orc.disc_ce(zs, zt), rel=1e-14)


def test_fused_adversarial_step_matches_reference_sequence(ml, orc):
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 5)
    replay, xt = rows(256, 16, 1), rows(12, 16, 2)
    dm = ml.DeviceModel(p, ml.PREC_TF32, 512)
    adv = ml.make_adversary(replay, 512, 3)
    res = ml.adversarial_step(adv, dm, xt, 0.01)
    _, hs = orc.forward(dims, p.params, replay)
    _, ht = orc.forward(dims, p.params, xt)
    aw, ab, lref = orc.adversarial_term(np.zeros(512), 0.0, hs, ht)
    assert res.discriminator_loss == pytest.approx(lref, rel=1e-5)
    assert nrel(adv.weight, aw) < TOL_TF32


# ---------------------------------------------------------------- top-k / selection (bit-exact)
@pytest.mark.parametrize("n,k", [(1, 1), (7, 3), (1000, 12), (100000, 1024), (1 << 20, 4096), (5000, 5000)])
def test_topk_bit_exact(ml, orc, n, k):
    rng = np.random.default_rng(n)
    s = f32(np.round(rng.normal(0, 1, n), 3))  # many ties
    if k > 4096:
        k = 4096
    got = ml.topk(s, k)
    ref = orc.topk(s.astype(np.float32), k)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("kind,k", [("normal", 1), ("normal", 12), ("normal", 1024), ("normal", 4096),
                                    ("ascending", 1024), ("descending", 4096), ("ties", 777), ("equal", 4096),
                                    ("negative", 100)])
def test_topk_large_pool_bit_exact(ml, orc, kind, k):
    """3M-candidate pools: the one-pass sampled top-k (topk.cu) and, where the sample is not
    conclusive (all-equal scores: the candidate set overflows), the exact radix fallback."""
    n = 3_000_001
    rng = np.random.default_rng(k)
    s = rng.normal(0, 1, n)
    if kind == "ascending":
        s = np.sort(s)
    elif kind == "descending":
        s = np.sort(s)[::-1].copy()
    elif kind == "ties":
        s = np.round(s, 2)
    elif kind == "equal":
        s = np.full(n, 0.25)
    elif kind == "negative":
        s = -np.abs(s) - 1.0
    s = f32(s)
    assert np.array_equal(ml.topk(s, k), orc.topk(s.astype(np.float32), k))


@pytest.mark.parametrize("n,k", [(20_000_003, 1024), ((1 << 20) + 1, 1), (8_388_611, 4096)])
def test_topk_one_launch_pools(ml, orc, n, k):
    """Pools sized like the scoring workload (ragged tails: n mod 4 = 3 / 1 / 3) through the one-launch
    sampled top-k: the result equals the oracle order, ties in the candidate set included."""
    rng = np.random.default_rng(n)
    s = f32(np.round(rng.normal(0, 1, n), 4))
    L = ml.lib()
    L.moses_kernel_launches.restype = C.c_int64
    l0 = L.moses_kernel_launches()
    got = ml.topk(s, k)
    assert L.moses_kernel_launches() - l0 == 2  # f64 -> f32 conversion + the one top-k launch (conclusive)
    assert np.array_equal(got, orc.topk(s.astype(np.float32), k))


def test_topk_negative_and_equal_scores(ml, orc):
    s = np.array([-1.0, -0.5, -0.5, -3.0, 0.0, -0.0, 2.5, -0.5])
    assert np.array_equal(ml.topk(s, 8), orc.topk(s.astype(np.float32), 8))
    assert list(ml.topk(np.full(10, 3.0), 4)) == [0, 1, 2, 3]


# ---------------------------------------------------------------- pooling / MMD
def test_segment_sum_vs_oracle(ml, orc):
    off = orc.synth_offsets(5, 1000, 8)
    h = f32(rows(int(off[-1]), 37, 1))
    got = ml.segment_sum(h, off)
    ref = orc.segment_sum(h, off)
    assert nrel(got, ref) < 1e-6
    empty = np.array([0, 0, 3, 3], dtype=np.int64)  # empty segments
    assert nrel(ml.segment_sum(h[:3], empty), orc.segment_sum(h[:3], empty)) < 1e-6


def gram_sum(a, b, sigma):
    d = (a * a).sum(1)[:, None] + (b * b).sum(1)[None, :] - 2 * a @ b.T
    return np.exp(-np.maximum(d, 0) / (2 * sigma * sigma)).sum()


@pytest.mark.parametrize("m,n,w,shift", [(300, 120, 64, 0.3), (1000, 257, 512, 0.1), (129, 130, 37, 0.0),
                                         (2000, 500, 512, 0.0)])
def test_mmd_vs_oracle(ml, orc, m, n, w, shift):
    """MMD^2 on tcgen05 kind::tf32 Gram tiles (gemm_gram.cuh) vs fp64: within 1e-3 of the kernel-sum
    scale S(s,s)/m^2 + S(t,t)/n^2 + 2 S(s,t)/(mn) (the north-star TF32 tolerance; MMD^2 itself can
    cancel to ~0). Small cases against the C oracle, the large one against its numpy restatement."""
    rng = np.random.default_rng(m + n + w)
    xs, xt = rng.normal(0, 1, (m, w)), rng.normal(shift, 1, (n, w))
    sigma = float(np.sqrt(w))
    ss, tt, st = gram_sum(xs, xs, sigma), gram_sum(xt, xt, sigma), gram_sum(xs, xt, sigma)
    scale = ss / m**2 + tt / n**2 + 2 * st / (m * n)
    ref = orc.mmd2(xs, xt, sigma) if m * n < 400_000 else ss / m**2 + tt / n**2 - 2 * st / (m * n)
    got = ml.mmd2(xs, xt, sigma)
    assert abs(got - ref) <= 1e-3 * scale, (got, ref, scale)


def test_mmd_device_entry_matches_host_entry(ml):
    import ctypes as C

    import torch

    rng = np.random.default_rng(4)
    xs, xt = rng.normal(0, 1, (700, 512)), rng.normal(0.2, 1, (300, 512))
    ld = 520  # padded row stride
    X = torch.zeros((1000, ld), dtype=torch.float32)
    X[:700, :512] = torch.from_numpy(xs)
    X[700:, :512] = torch.from_numpy(xt)
    X = X.cuda()
    out = C.c_double()
    rc = ml.lib().moses_mmd2_device(C.c_void_p(X.data_ptr()), 700, C.c_void_p(X[700:].data_ptr()), 300, 512, ld,
                                    8.0, C.byref(out))
    assert rc == 0, ml.lib().moses_last_error()
    assert out.value == pytest.approx(ml.mmd2(xs, xt, 8.0), rel=1e-9, abs=1e-12)


# ---------------------------------------------------------------- synthetic generator bit-exactness
def test_device_synthetic_features_match_oracle(ml, orc):
    import torch

    n, D = 333, 164
    ld = 168
    buf = torch.zeros((n, ld), dtype=torch.float32, device="cuda")
    assert ml.lib().moses_synth_features_device(1, 1000, n, D, ml.DTYPE_F32, buf.data_ptr(), ld) == 0
    torch.cuda.synchronize()
    ref = orc.synth_features(1, 1000, n, D).astype(np.float32)
    got = buf.cpu().numpy()
    assert np.array_equal(got[:, :D], ref)
    assert np.all(got[:, D] == 1.0) and np.all(got[:, D + 1:] == 0.0)
    y = torch.zeros(n, dtype=torch.float32, device="cuda")
    assert ml.lib().moses_synth_labels_device(1, 1000, n, y.data_ptr()) == 0
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), orc.synth_labels(1, 1000, n).astype(np.float32))


# ---------------------------------------------------------------- CUDA-graph training step
def test_train_graph_matches_eager_steps(ml):
    """moses_train_graph_* (device gather + gradients + update, replayed) == eager steps, bit for bit."""
    import ctypes as C

    import torch

    dims = [164, 512, 512, 1]
    p = ml.init_random(dims, 2)
    L = ml.lib()
    a = ml.DeviceModel(p, ml.PREC_BF16, 512)
    b = ml.DeviceModel(p, ml.PREC_BF16, 512)
    ld = a.packed_ld
    nb, batch = 3, 256
    X = torch.empty((nb * batch, ld), dtype=torch.bfloat16, device="cuda")
    Y = torch.empty(nb * batch, dtype=torch.float32, device="cuda")
    assert L.moses_synth_features_device(1, 0, nb * batch, dims[0], ml.DTYPE_BF16, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(1, 0, nb * batch, Y.data_ptr()) == 0
    torch.cuda.synchronize()
    ml._ck(L.moses_train_graph_create(a.h, X.data_ptr(), ld, Y.data_ptr(), nb, batch, 0.001, 0.9, 1))
    ml._ck(L.moses_train_graph_launch(a.h, 5))
    for s in range(5):
        r = s % nb
        ml._ck(L.moses_train_step_device(b.h, X.data_ptr() + r * batch * ld * 2, ld, Y.data_ptr() + r * batch * 4,
                                         batch, 0.001, 0.9, None))
    pa, pb = a.download(), b.download()
    assert np.array_equal(pa.params, pb.params) and np.array_equal(pa.momentum, pb.momentum)


# ---------------------------------------------------------------- pooled (TenSet-shaped) training
@pytest.mark.parametrize("mode", ["tf32", "bf16"])
@pytest.mark.parametrize("programs,max_stmts", [(12, 4), (512, 8)])
def test_pooled_gradients(ml, orc, mode, programs, max_stmts):
    from precision_model import device_gradients_pooled

    dims = [164, 512, 512, 1]
    p = ml.init_random(dims, 8)
    off = ml.synth_offsets(3, programs, max_stmts)
    assert np.array_equal(off, orc.synth_offsets(3, programs, max_stmts))
    x = rows(int(off[-1]), 164, 4)
    y = labels(programs, 5)
    dm = ml.DeviceModel(p, ml.PREC_TF32 if mode == "tf32" else ml.PREC_BF16, 4096)
    g, loss = ml.gradients_pooled(dm, x, off, y, want_loss=True)
    g_ref, _ = device_gradients_pooled(dims, p.params, x, off, y, mode)
    ok, why = grad_close(g, g_ref)
    assert ok, why
    _, loss64 = orc.gradients_pooled(dims, p.params, x, off, y)
    assert abs(loss - loss64) <= TOL_TF32 * max(1.0, abs(loss64))


def test_pooled_with_unit_segments_equals_unpooled(ml):
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 9)
    x, y = rows(40, 16, 1), labels(40, 2)
    dm = ml.DeviceModel(p, ml.PREC_BF16, 64)
    g0 = ml.gradients(dm, ml.RankingBatch(x, y))
    g1 = ml.gradients_pooled(dm, x, np.arange(41), y)
    assert np.array_equal(g0[:-1], g1[:-1])  # everything but the head bias (summed in another order)
    assert abs(g1[-1] - g0[-1]) < 1e-6  # sum_p gs_p is 0 up to rounding noise


def test_pooled_train_graph(ml):
    """Device-resident TenSet-shaped step (gather of variable-length programs + pooled gradients + update)
    == the host pooled path, bit for bit."""
    import torch

    dims = [164, 512, 512, 1]
    p = ml.init_random(dims, 2)
    L = ml.lib()
    B, nb = 64, 3
    off = ml.synth_offsets(7, B * nb, 8)
    rows_total = int(off[-1])
    per_batch = [int(off[(b + 1) * B] - off[b * B]) for b in range(nb)]
    rows_pad = (max(per_batch) + 127) // 128 * 128
    a = ml.DeviceModel(p, ml.PREC_BF16, rows_pad)
    bm = ml.DeviceModel(p, ml.PREC_BF16, rows_pad)
    ld = a.packed_ld
    X = torch.empty((rows_total, ld), dtype=torch.bfloat16, device="cuda")
    Y = torch.empty(B * nb, dtype=torch.float32, device="cuda")
    assert L.moses_synth_features_device(1, 0, rows_total, dims[0], ml.DTYPE_BF16, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(1, 0, B * nb, Y.data_ptr()) == 0
    OFF = torch.from_numpy(off).cuda()
    torch.cuda.synchronize()
    ml._ck(L.moses_train_graph_create_pooled(a.h, X.data_ptr(), ld, Y.data_ptr(), OFF.data_ptr(), nb, B, rows_pad,
                                             0.001, 0.9, 1))
    ml._ck(L.moses_train_graph_launch(a.h, 1))  # the alternating graphs keep their parity across calls:
    ml._ck(L.moses_train_graph_launch(a.h, 7))  # A | B A B A B A B
    xs = X.float().cpu().numpy()[:, :dims[0]].astype(np.float64)  # bf16-exact values
    ys = Y.cpu().numpy().astype(np.float64)
    for s in range(8):
        b = s % nb
        lo, hi = int(off[b * B]), int(off[(b + 1) * B])
        ml.gradients_pooled(bm, xs[lo:hi], off[b * B:(b + 1) * B + 1] - lo, ys[b * B:(b + 1) * B])
        ml.apply_update(bm, ml.TrainHyper(learning_rate=0.001, momentum=0.9), None, True)
    pa, pb = a.download(), bm.download()
    assert np.array_equal(pa.params, pb.params)


@pytest.mark.parametrize("rho", [0.3, 0.5, 0.7])
def test_fused_lottery_step_large_bit_exact(ml, orc, rho):
    """8.4M scalars (multi-round histogram passes), 40% zero-gradient ties, ratio mode: mask and
    updated weights bit-identical to xi -> nth_element partition -> step -> decay in fp32."""
    dims = [4096, 2048, 8, 1]
    P = ml.param_count(dims)
    rng = np.random.default_rng(int(rho * 10))
    w = f32(rng.normal(0, 0.05, P))
    g = f32(rng.normal(0, 1e-2, P))
    g[rng.random(P) < 0.4] = 0.0
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_BF16, 16)
    dm.set_gradients(g)
    mask = ml.lottery_step(dm, ml.RATIO, rho, 0, 0.001, 0.01)
    w32, g32 = w.astype(np.float32), g.astype(np.float32)
    ref_mask = orc.partition(orc.xi_scores(w32, g32, False), False, orc.RATIO, rho)
    assert np.array_equal(mask.transferable, ref_mask)
    ref_w, _ = orc.apply_update(w32, np.zeros_like(w32), g32, 0.001, 0.0, ref_mask, False)
    ref_w = orc.variant_decay(ref_w, ref_mask, 0.001, 0.01)
    assert np.array_equal(dm.download().params, ref_w.astype(np.float64))


@pytest.mark.parametrize("kind,rho", [("normal", 0.3), ("normal", 0.5), ("normal", 0.01), ("zeros", 0.7),
                                      ("quantized", 0.37), ("ties", 0.42)])
def test_fused_lottery_step_compaction_path_bit_exact(ml, orc, kind, rho):
    """16.8M scalars: the sampled-bracket compaction path of the ratio step (lottery.cu). 'zeros'
    puts the keep-th key inside the 40% zero-gradient ties (bracket disabled -> exact fallback);
    'quantized' draws w, g from a few values so the cut falls inside a huge tie group of a non-zero
    key (general chunked index cut); 'ties' copies the keep-th scalar's (w, g) to 200 random slots
    so a small tie group straddles the cut (sorted-candidate index cut). Mask and weights bit-exact."""
    dims = [8192, 2048, 8, 1]
    P = ml.param_count(dims)
    rng = np.random.default_rng(int(rho * 100) + len(kind))
    if kind == "quantized":
        w = f32(rng.choice([-0.05, -0.02, 0.01, 0.03, 0.07], P))
        g = f32(rng.choice([-2e-2, -5e-3, 1e-3, 4e-3, 1e-2], P))
    else:
        w = f32(rng.normal(0, 0.05, P))
        g = f32(rng.normal(0, 1e-2, P))
        g[rng.random(P) < 0.4] = 0.0
    if kind == "ties":
        xi = np.abs(w.astype(np.float32) * g.astype(np.float32))
        keep = orc.ratio_keep(rho, P)
        r = int(np.argpartition(-xi, keep - 1)[keep - 1])  # the keep-th largest
        slots = rng.choice(P, 200, replace=False)
        w[slots], g[slots] = w[r], g[r]
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_BF16, 16)
    dm.set_gradients(g)
    mask = ml.lottery_step(dm, ml.RATIO, rho, 0, 0.001, 0.01)
    w32, g32 = w.astype(np.float32), g.astype(np.float32)
    ref_mask = orc.partition(orc.xi_scores(w32, g32, False), False, orc.RATIO, rho)
    assert np.array_equal(mask.transferable, ref_mask)
    ref_w, _ = orc.apply_update(w32, np.zeros_like(w32), g32, 0.001, 0.0, ref_mask, False)
    ref_w = orc.variant_decay(ref_w, ref_mask, 0.001, 0.01)
    assert np.array_equal(dm.download().params, ref_w.astype(np.float64))


@pytest.mark.parametrize("kind", ["normal", "zeros", "quantized", "ties"])
@pytest.mark.parametrize("mode,value", [(2, 0.01), (2, 0.5), (2, 0.7), (1, 0.5)])
def test_resident_lottery_step_bit_exact(ml, orc, kind, mode, value):
    """The single-launch register-resident step (lottery.cu lot_resident_kernel, P <= ~1.2M): three
    consecutive Moses steps (barrier / histogram state reused across calls, a second model
    interleaved) — masks and weights bit-identical to xi -> partition -> step -> decay in fp32."""
    dims = [1024, 1024, 8, 1]
    P = ml.param_count(dims)
    rng = np.random.default_rng(int(value * 100) + mode + len(kind))
    if kind == "quantized":
        w = f32(rng.choice([-0.05, -0.02, 0.01, 0.03, 0.07], P))
        g = f32(rng.choice([-2e-2, -5e-3, 1e-3, 4e-3, 1e-2], P))
    else:
        w = f32(rng.normal(0, 0.05, P))
        g = f32(rng.normal(0, 1e-2, P))
        if kind in ("zeros", "ties"):
            g[rng.random(P) < 0.4] = 0.0
    if kind == "ties" and mode == 2:
        xi = np.abs(w.astype(np.float32) * g.astype(np.float32))
        keep = orc.ratio_keep(value, P)
        r = int(np.argpartition(-xi, keep - 1)[keep - 1])
        slots = rng.choice(P, 300, replace=False)
        w[slots], g[slots] = w[r], g[r]
    other = ml.DeviceModel(ml_params([64, 64, 8, 1], f32(rng.normal(0, 1, ml.param_count([64, 64, 8, 1])))),
                           ml.PREC_BF16, 16)
    other.set_gradients(f32(rng.normal(0, 1, other.P)))
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_BF16, 16)
    w32, g32 = w.astype(np.float32), g.astype(np.float32)
    for it in range(3):
        dm.set_gradients(g32.astype(np.float64))
        mask = ml.lottery_step(dm, mode, value, it, 0.001, 0.01)
        ml.lottery_step(other, 2, 0.5, it, 0.001, 0.01)
        xi = orc.xi_scores(w32, g32, mode == 1)
        ref_mask = orc.partition(xi, mode == 1, orc.RATIO if mode == 2 else orc.THRESHOLD, value)
        assert np.array_equal(mask.transferable, ref_mask), it
        w32, _ = orc.apply_update(w32, np.zeros_like(w32), g32, 0.001, 0.0, ref_mask, False)
        w32 = orc.variant_decay(w32, ref_mask, 0.001, 0.01)
        assert np.array_equal(dm.download().params, w32.astype(np.float64)), it


@pytest.mark.parametrize("theta", [0.5, 0.01, 0.999, 0.0])
def test_threshold_step_large_bit_exact(ml, orc, theta):
    """Multi-pass threshold step at 4.2M scalars (lot_max -> lot_apply with the division-free
    normalised test, lottery.cu thresh_key): mask, popcount and weights bit-identical to
    xi_scores(normalize) -> xi > theta -> step -> decay in fp32."""
    dims = [2048, 2048, 8, 1]
    P = ml.param_count(dims)
    rng = np.random.default_rng(int(theta * 1000) + 3)
    w = f32(rng.normal(0, 0.05, P))
    g = f32(rng.normal(0, 1e-2, P))
    g[rng.random(P) < 0.4] = 0.0
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_BF16, 16)
    dm.set_gradients(g)
    mask = ml.lottery_step(dm, ml.THRESHOLD, theta, 0, 0.001, 0.01)
    w32, g32 = w.astype(np.float32), g.astype(np.float32)
    ref_mask = orc.partition(orc.xi_scores(w32, g32, True), True, orc.THRESHOLD, theta)
    assert np.array_equal(mask.transferable, ref_mask)
    ref_w, _ = orc.apply_update(w32, np.zeros_like(w32), g32, 0.001, 0.0, ref_mask, False)
    ref_w = orc.variant_decay(ref_w, ref_mask, 0.001, 0.01)
    assert np.array_equal(dm.download().params, ref_w.astype(np.float64))


@pytest.mark.parametrize("kind,theta", [("normal", 0.5), ("normal", 0.9), ("outlier", 0.5), ("zeros", 0.0),
                                         ("allzero", 0.5), ("normal", 0.0)])
def test_threshold_step_single_pass_bit_exact(ml, orc, kind, theta):
    """16.8M scalars: the one-pass threshold step (lottery.cu lot_thresh_pass / lot_thresh_fix). 'normal':
    the few scalars at or above the sampled bound resolve from the candidate list; 'outlier': one huge
    xi outside every sampled stratum puts the sampled max far below the true max, the candidate list
    overflows and the fix-up scans the mask bytes; 'allzero': g == 0 (max 0, xi not normalised, nothing
    kept); theta = 0 keeps every non-zero xi. Mask, popcount and weights bit-identical to
    xi_scores(normalize) -> xi > theta -> step -> decay in fp32."""
    dims = [8192, 2048, 8, 1]
    P = ml.param_count(dims)
    rng = np.random.default_rng(int(theta * 100) + len(kind))
    w = f32(rng.normal(0, 0.05, P))
    g = f32(rng.normal(0, 1e-2, P))
    if kind == "zeros":
        g[rng.random(P) < 0.4] = 0.0
    if kind == "allzero":
        g[:] = 0.0
    if kind == "outlier":
        # the sample reads one float4 per 1024 scalars at a hashed offset; index 5 of stratum 7 is
        # never sampled when the hashed float4 of stratum 7 is elsewhere (checked below)
        i = 7 * 1024 + 5
        w[i], g[i] = 3.0, 2.0
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_BF16, 16)
    dm.set_gradients(g)
    import ctypes

    out = np.zeros(P, dtype=np.uint8)
    pop = ctypes.c_int64()
    ml._ck(ml.lib().moses_lottery_step(dm.h, ml.THRESHOLD, theta, 0, 0.001, 0.01, out.ctypes.data, P, ctypes.byref(pop)))
    w32, g32 = w.astype(np.float32), g.astype(np.float32)
    ref_mask = orc.partition(orc.xi_scores(w32, g32, True), True, orc.THRESHOLD, theta)
    assert np.array_equal(out.astype(bool), ref_mask)
    assert pop.value == int(np.sum(ref_mask))  # the device count of the kept scalars
    ref_w, _ = orc.apply_update(w32, np.zeros_like(w32), g32, 0.001, 0.0, ref_mask, False)
    ref_w = orc.variant_decay(ref_w, ref_mask, 0.001, 0.01)
    assert np.array_equal(dm.download().params, ref_w.astype(np.float64))


@pytest.mark.parametrize("pinned_losses", [True, False])
def test_async_pooled_steps_match_synchronous(ml, pinned_losses):
    """moses_train_step_pooled_async (double-buffered upload + per-slot graph) == gradients_pooled +
    apply_update(momentum) step by step: parameters bit-identical, per-step losses equal (delivered
    through the slot mailboxes into pinned or pageable host memory)."""
    import ctypes

    import torch

    dims = [164, 512, 512, 512, 1]
    p = ml.init_random(dims, 4, strict=False)
    B = 128
    batches = []
    for b in range(3):
        off = ml.synth_offsets(20 + b, B, 8)
        x = rows(int(off[-1]), dims[0], 30 + b)
        y = labels(B, 40 + b)
        batches.append((np.ascontiguousarray(x), np.ascontiguousarray(off), np.ascontiguousarray(y)))
    cap = 1024
    a = ml.DeviceModel(p, ml.PREC_BF16, cap)
    s = ml.DeviceModel(p, ml.PREC_BF16, cap)
    hyper = ml.TrainHyper(learning_rate=0.001, momentum=0.9)
    steps = [0, 1, 2, 0, 1]
    losses = torch.full((len(steps),), -1.0, dtype=torch.float64)
    if pinned_losses:
        losses = losses.pin_memory()
    keep = []
    for k, b in enumerate(steps):
        x, off, y = batches[b]
        xp, op, yp = (torch.from_numpy(v).pin_memory() for v in (x, off, y))
        keep.append((xp, op, yp))  # must outlive the queued step
        ml._ck(ml.lib().moses_train_step_pooled_async(a.h, ctypes.c_void_p(xp.data_ptr()), x.shape[0], dims[0],
                                                       ctypes.c_void_p(op.data_ptr()), B, ctypes.c_void_p(yp.data_ptr()),
                                                       0.001, 0.9, ctypes.c_void_p(losses[k:k + 1].data_ptr())))
    ml._ck(ml.lib().moses_model_synchronize(a.h))
    ref_losses = []
    for b in steps:
        x, off, y = batches[b]
        ref_losses.append(ml.gradients_pooled(s, x, off, y, want_loss=True)[1])
        ml.apply_update(s, hyper, None, True)
    assert np.array_equal(a.download().params, s.download().params)
    assert np.allclose(losses.numpy(), ref_losses, rtol=0, atol=1e-12)


@pytest.mark.parametrize("dims", [[164, 512, 512, 512, 512, 1], [2048, 2048, 8, 1]])
@pytest.mark.parametrize("mode,value", [(2, 0.5), (1, 0.5)])
def test_lottery_step_adam_bit_exact(ml, orc, dims, mode, value):
    """Fused Moses step with masked Adam (resident kernel at 873K scalars, multi-pass at 4.2M):
    two consecutive steps, mask and weights bit-identical to xi -> partition -> adam_update(mask)
    -> variant_decay(lr, lambda) in fp32."""
    P = ml.param_count(dims)
    rng = np.random.default_rng(P % 97 + mode)
    w = f32(rng.normal(0, 0.05, P))
    g = f32(rng.normal(0, 1e-2, P))
    g[rng.random(P) < 0.4] = 0.0
    dm = ml.DeviceModel(ml_params(dims, w), ml.PREC_BF16, 16)
    w32, g32 = w.astype(np.float32), g.astype(np.float32)
    m1, m2 = np.zeros(P, np.float32), np.zeros(P, np.float32)
    lr, b1, b2, eps, lam = 1e-3, 0.9, 0.999, 1e-8, 0.01
    for step in (1, 2):
        dm.set_gradients(g32.astype(np.float64))
        mask = ml.lottery_step_adam(dm, mode, value, step, lr, b1, b2, eps, step, lam)
        xi = orc.xi_scores(w32, g32, mode == 1)
        ref_mask = orc.partition(xi, mode == 1, mode, value)
        assert np.array_equal(mask.transferable, ref_mask)
        w32, m1, m2 = orc.adam(w32, m1, m2, g32, lr, b1, b2, eps, step, ref_mask)
        w32 = orc.variant_decay(w32, ref_mask, lr, lam)
        assert np.array_equal(dm.download().params, w32.astype(np.float64)), step


# ---------------------------------------------------------------- fused ranking step: grid vs cluster form
@pytest.mark.parametrize("kind,n", [("plain", 2), ("plain", 64), ("plain", 512), ("plain", 1000), ("pooled", 37),
                                    ("pooled", 512), ("pooled", 900), ("plain", 3000), ("pooled", 2000)])
@pytest.mark.parametrize("prec", ["bf16", "tf32"])
def test_rank_step_grid_matches_cluster(ml, kind, n, prec):
    """Both forms evaluate the same (split, row) pair items and per-row sums, so every backward
    coefficient — hence every weight gradient except the head bias — is bitwise equal; loss and
    head-bias gradient differ only by the order of the final double sums."""
    dims = [164, 512, 512, 1]
    p = ml.init_random(dims, 4)
    dm = ml.DeviceModel(p, ml.PREC_BF16 if prec == "bf16" else ml.PREC_TF32, 16384)
    rng = np.random.default_rng(n)
    y = np.round(rng.random(n) * 8) / 8  # ties included
    L = ml.lib()
    out = []
    L.moses_debug_set_rank_sym(0)  # grid vs cluster here; the symmetric form: tests/test_gpu_rank_sym.py
    for grid in (1, 0):
        L.moses_debug_set_rank_grid(grid)  # 0: default policy (cluster form where it fits)
        try:
            if kind == "plain":
                x = rng.random((n, 164)) if not out else xs
                xs = x
                g, loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
            else:
                off = ml.synth_offsets(7, n, 8)
                x = rng.random((int(off[-1]), 164)) if not out else xs
                xs = x
                g, loss = ml.gradients_pooled(dm, x, off, y, want_loss=True)
        finally:
            L.moses_debug_set_rank_grid(0)
        out.append((g, loss))
    L.moses_debug_set_rank_sym(1)
    (g1, l1), (g0, l0) = out
    hb = dm.P - 1  # head bias: last scalar of the reference order
    mask = np.ones(dm.P, dtype=bool)
    mask[hb] = False
    assert np.array_equal(g1[mask], g0[mask])
    assert abs(g1[hb] - g0[hb]) <= 1e-6 * max(1e-6, abs(g0[hb]))
    assert abs(l1 - l0) <= 1e-12 * max(1.0, abs(l0))


@pytest.mark.parametrize("beta", [0.01, 0.0])
@pytest.mark.parametrize("mode,value", [(2, 0.5), (1, 0.5)])
def test_moses_step_fused_equals_three_calls(ml, beta, mode, value):
    """moses_moses_step == moses_gradients(adv) + moses_adversarial_step + moses_lottery_step, bit for
    bit: parameters, discriminator weights, losses and popcount over three consecutive steps."""
    import ctypes as C

    dims = [164, 512, 512, 512, 512, 1]
    p = ml.init_random(dims, 31, strict=False)
    rng = np.random.default_rng(5)
    replay = rng.random((256, dims[0]))
    L = ml.lib()
    out = []
    for fused in (True, False):
        dm = ml.DeviceModel(p, ml.PREC_BF16, 1024)
        adv = ml.AdversaryState(replay, dims[-2])
        rec = []
        for k in range(3):
            x = np.ascontiguousarray(np.random.default_rng(100 + k).random((512, dims[0])))
            y = np.ascontiguousarray(0.1 + np.random.default_rng(200 + k).random(512))
            loss, dl, cf, pop = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
            if fused:
                ml._ck(L.moses_moses_step(dm.h, adv.h, x.ctypes.data, y.ctypes.data, 512, dims[0], beta, mode, value, 0,
                                          1e-3, 1e-2, C.byref(loss), C.byref(dl), C.byref(pop)))
            else:
                ml._ck(L.moses_gradients(dm.h, x.ctypes.data, y.ctypes.data, 512, dims[0], adv.h, beta, C.byref(loss)))
                ml._ck(L.moses_adversarial_step(adv.h, dm.h, x.ctypes.data, 512, dims[0], beta, C.byref(dl),
                                                C.byref(cf)))
                ml._ck(L.moses_lottery_step(dm.h, mode, value, 0, 1e-3, 1e-2, None, 0, C.byref(pop)))
            rec.append((loss.value, dl.value, pop.value))
        out.append((rec, dm.download().params, adv.weight, adv.bias))
        del adv
        dm.close()
    (r1, w1, u1, c1), (r0, w0, u0, c0) = out
    assert r1 == r0
    assert np.array_equal(w1, w0) and np.array_equal(u1, u0) and c1 == c0
