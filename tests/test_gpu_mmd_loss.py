"""MMD^2 as a differentiable domain loss on the device (north-star (4)) against the fp64 oracle:
row gradients of the statistic, the model gradient with beta * MMD^2 in the domain-term slot (FP32 and
split-bf16 handles), beta = 0 == gradients(), and the cfg3 fine-tune step (MMD gradient -> ratio-0.5
lottery step: mask, masked update, variant decay)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0, moseslab.lib().moses_last_error()
    return moseslab


def nrel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


@pytest.mark.parametrize("m,n,w", [(7, 5, 16), (256, 512, 512), (300, 41, 100)])
def test_mmd2_row_gradients_vs_oracle(ml, orc, m, n, w):
    rng = np.random.default_rng(m)
    xs, xt = f32(rng.random((m, w))), f32(rng.random((n, w)) + 0.05)
    sigma = float(np.sqrt(w / 6.0))
    v, gs, gt = ml.mmd2_grad(xs, xt, sigma)
    vr, gsr, gtr = orc.mmd2_grad(xs, xt, sigma)
    assert abs(v - vr) <= 1e-5 * max(abs(vr), 1e-3)
    assert nrel(np.concatenate([gs, gt]), np.concatenate([gsr, gtr])) < 1e-4


@pytest.mark.parametrize("prec,tol", [("FP32", 1e-5), ("BF16X3", 1e-3)])
def test_gradients_with_mmd_vs_oracle(ml, orc, prec, tol):
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 21)
    rng = np.random.default_rng(5)
    x, y, src = f32(rng.random((64, 16))), f32(0.1 + rng.random(64)), f32(rng.random((256, 16)) * 0.9)
    p32 = ml.CostModelParams(dims, f32(p.params))
    dm = ml.DeviceModel(p32, getattr(ml, "PREC_" + prec), 512)
    for beta in (0.5, 0.01):
        g, loss = ml.gradients_mmd(dm, ml.RankingBatch(x, y), src, beta, 4.0, want_loss=True)
        g_ref, loss_ref = orc.gradients_mmd(dims, p32.params, x, y, src, beta, 4.0)
        assert abs(loss - loss_ref) <= tol * abs(loss_ref)
        assert nrel(g, g_ref) < tol, (beta, nrel(g, g_ref))
    # beta = 0: gradients() bit for bit
    g0 = ml.gradients_mmd(dm, ml.RankingBatch(x, y), src, 0.0, 4.0)
    assert np.array_equal(g0, ml.gradients(dm, ml.RankingBatch(x, y)))


def test_cfg3_mmd_finetune_step_vs_oracle(ml, orc):
    """cfg3 step with the MMD domain loss: gradients with beta * MMD^2 (256 source rows, 512-row target
    batch) -> xi -> ratio-0.5 partition -> transferable step -> variant decay (tuner.cpp:251-262 with the
    MMD term in the domain slot). The mask is bit-exact against the oracle's partition of the device's
    xi; the updated weights within 1e-5 of the oracle sequence on the device's gradient, and the
    gradient within 1e-5 of the fp64 oracle (FP32 handle)."""
    dims = [164, 512, 512, 1]
    p = ml.init_random(dims, 12345)
    p32 = ml.CostModelParams(dims, f32(p.params))
    rng = np.random.default_rng(9)
    src, x, y = f32(rng.random((256, 164))), f32(rng.random((512, 164)) + 0.02), f32(0.1 + rng.random(512))
    dm = ml.DeviceModel(p32, ml.PREC_FP32, 1024)
    g = ml.gradients_mmd(dm, ml.RankingBatch(x, y), src, 0.01, 6.0)
    g_ref, _ = orc.gradients_mmd(dims, p32.params, x, y, src, 0.01, 6.0)
    assert nrel(g, g_ref) < 1e-5
    mask = ml.lottery_step(dm, ml.RATIO, 0.5, 0, 0.001, 0.01)
    w = p32.params
    xi = np.abs(np.float32(w) * np.float32(g)).astype(np.float64)
    want = orc.partition(xi, False, 2, 0.5)
    assert np.array_equal(np.asarray(mask.transferable, bool), want)
    w_ref = np.where(want, np.float32(w) - np.float32(0.001) * np.float32(g),
                     np.float32(w) * np.float32(1.0 - 0.001 * 0.01)).astype(np.float64)
    assert nrel(dm.download().params - w, w_ref - w) < 1e-5
