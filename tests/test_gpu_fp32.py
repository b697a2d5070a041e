"""FP32 parity mode (MOSES_PREC_FP32): 3xTF32 split-operand GEMMs on the tensor cores.

North-star tolerance for the fp32 path: <= 1e-5 normwise relative against the fp64 oracle
(oracle/moses_oracle.hpp) on the same fp32-representable inputs and weights. Every GEMM
operand is carried as hi = rna_tf32(v), lo = rna_tf32(v - hi) and multiplied as
hi*hi + hi*lo + lo*hi, which leaves ~2^-22 relative operand error (fp32-level).
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_FP32 = 1e-5


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0, moseslab.lib().moses_last_error()
    return moseslab


def nrel(got, ref):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


def frob(got, ref):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rows(n, d, seed):
    return f32(np.random.default_rng(seed).random((n, d)))


def labels(n, seed):
    return f32(0.1 + np.random.default_rng(seed).random(n))


def f32_params(ml, p):
    return ml.CostModelParams(list(p.dims), f32(p.params))


def grad_ok(g, ref, tol=TOL_FP32):
    """Normwise within tol; a ReLU-kink flip (|z| below the fp32 rounding error) may move a
    handful of entries, so the max-norm check uses the 99.9% quantile."""
    d = np.abs(np.asarray(g) - ref) / max(np.max(np.abs(ref)), 1e-300)
    return float(np.quantile(d, 0.999)) <= tol and frob(g, ref) <= tol, (float(np.quantile(d, 0.999)), frob(g, ref))


@pytest.mark.parametrize("dims", [[16, 512, 512, 1], [164, 512, 512, 512, 512, 1], [33, 72, 40, 1]])
@pytest.mark.parametrize("n", [7, 300])
def test_fp32_predict_vs_oracle(ml, orc, dims, n):
    p = f32_params(ml, ml.init_random(dims, 11, strict=False))
    x = rows(n, dims[0], n)
    ref, h_ref = orc.forward(dims, p.params, x)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 512)
    assert nrel(ml.predict(dm, x), ref) <= TOL_FP32
    assert nrel(ml.penultimate_activations(dm, x), h_ref) <= TOL_FP32


def test_fp32_is_tighter_than_tf32(ml, orc):
    dims = [164, 512, 512, 1]
    p = f32_params(ml, ml.init_random(dims, 2))
    x = rows(256, 164, 3)
    ref, _ = orc.forward(dims, p.params, x)
    e32 = nrel(ml.predict(ml.DeviceModel(p, ml.PREC_FP32, 256), x), ref)
    etf = nrel(ml.predict(ml.DeviceModel(p, ml.PREC_TF32, 256), x), ref)
    assert e32 * 20 < etf, (e32, etf)


@pytest.mark.parametrize("dims", [[16, 512, 512, 1], [164, 512, 512, 512, 512, 1], [33, 72, 40, 1]])
@pytest.mark.parametrize("n", [12, 512])
def test_fp32_gradients_vs_oracle(ml, orc, dims, n):
    p = f32_params(ml, ml.init_random(dims, 21, strict=False))
    x, y = rows(n, dims[0], 7), labels(n, 8)
    g_ref, loss_ref = orc.gradients(dims, p.params, x, y)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 1024)
    g, loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
    ok, why = grad_ok(g, g_ref)
    assert ok, why
    assert abs(loss - loss_ref) <= TOL_FP32 * max(1.0, abs(loss_ref))


@pytest.mark.parametrize("beta", [0.01, 0.5])
def test_fp32_gradients_with_adversary(ml, orc, beta):
    dims = [16, 512, 512, 1]
    p = f32_params(ml, ml.init_random(dims, 31))
    x, y = rows(12, 16, 1), labels(12, 2)
    replay = rows(256, 16, 3)
    u = f32(np.random.default_rng(4).normal(0, 0.05, 512))
    c = 0.03
    g_ref, loss_ref = orc.gradients(dims, p.params, x, y, (u, c, replay), beta)
    adv = ml.make_adversary(replay, 512, 7)
    adv.set(u, c)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 512)
    g, loss = ml.gradients(dm, ml.RankingBatch(x, y), adv, beta, want_loss=True)
    ok, why = grad_ok(g, g_ref)
    assert ok, why
    assert abs(loss - loss_ref) <= TOL_FP32 * max(1.0, abs(loss_ref))


def test_fp32_pooled_gradients_vs_oracle(ml, orc):
    dims = [164, 512, 512, 1]
    p = f32_params(ml, ml.init_random(dims, 8))
    off = ml.synth_offsets(3, 512, 8)
    x = rows(int(off[-1]), 164, 4)
    y = labels(512, 5)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 4096)
    g, loss = ml.gradients_pooled(dm, x, off, y, want_loss=True)
    g_ref, loss_ref = orc.gradients_pooled(dims, p.params, x, off, y)
    ok, why = grad_ok(g, g_ref)
    assert ok, why
    assert abs(loss - loss_ref) <= TOL_FP32 * max(1.0, abs(loss_ref))


def test_fp32_train_steps_vs_oracle(ml, orc):
    """tuner.cpp:146-147 (gradients + momentum update) x3 in the fp32 path: the hi/lo weight shadow
    is refreshed after every update, so later steps see the updated weights at fp32 accuracy."""
    dims = [164, 512, 512, 1]
    p = f32_params(ml, ml.init_random(dims, 3))
    x, y = rows(512, 164, 1), labels(512, 2)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 512)
    w, mom = p.params.copy(), np.zeros_like(p.params)
    for _ in range(3):
        loss_ref = orc.train_step_f64(dims, w, mom, x, y, 0.001, 0.9, threads=8)
        loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)[1]
        ml.apply_update(dm, ml.TrainHyper(learning_rate=0.001, momentum=0.9), None, True)
        assert abs(loss - loss_ref) <= TOL_FP32 * max(1.0, abs(loss_ref))
    got = dm.download()
    assert nrel(got.params, w) <= TOL_FP32
    assert frob(got.momentum, mom) <= 1e-4  # accumulated raw gradients (3 steps, fp32 sums)


def test_fp32_lottery_step_refreshes_operands(ml, orc):
    """After a fused lottery step the forward must see the stepped/decayed weights (hi/lo pair)."""
    dims = [16, 512, 512, 1]
    p = f32_params(ml, ml.init_random(dims, 5))
    x, y = rows(64, 16, 6), labels(64, 7)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 128)
    ml.gradients(dm, ml.RankingBatch(x, y))
    ml.lottery_step(dm, ml.RATIO, 0.3, 1, 0.05, 0.5)
    w = dm.download().params
    ref, _ = orc.forward(dims, w, x)
    assert nrel(ml.predict(dm, x), ref) <= TOL_FP32


def test_fp32_rejects_training_graphs(ml):
    lib = ml.lib()
    dims = [16, 64, 64, 1]
    dm = ml.DeviceModel(ml.init_random(dims, 1), ml.PREC_FP32, 128)
    rc = lib.moses_train_graph_create(dm.h, ctypes.c_void_p(0), ctypes.c_int64(lib.moses_packed_ld(dm.h)),
                                      None, ctypes.c_int64(1), ctypes.c_int64(16), ctypes.c_double(0.001),
                                      ctypes.c_double(0.9), ctypes.c_int32(1))
    assert rc == 103
    msg = lib.moses_last_error()
    assert "FP32" in (msg.decode() if isinstance(msg, bytes) else msg)


def test_fp32_device_rows_equal_host_rows(ml):
    """FP32 handles take device-resident fp32 rows (split into their tf32 hi/lo planes on the device)."""
    import torch

    lib = ml.lib()
    dims = [16, 64, 64, 1]
    dm = ml.DeviceModel(ml.init_random(dims, 1), ml.PREC_FP32, 128)
    ld = lib.moses_packed_ld(dm.h)
    x = f32(np.random.default_rng(0).random((100, 16)))
    Xd = torch.zeros((100, ld), dtype=torch.float32, device="cuda")
    Xd[:, :16] = torch.from_numpy(x).float().cuda()
    S = torch.empty(100, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ml._ck(lib.moses_predict_device(dm.h, ctypes.c_void_p(Xd.data_ptr()), ml.DTYPE_F32, ctypes.c_int64(ld),
                                    ctypes.c_int64(100), ctypes.c_void_p(S.data_ptr())))
    ml._ck(lib.moses_model_synchronize(dm.h))
    assert np.array_equal(S.cpu().numpy(), ml.predict(dm, x).astype(np.float32))
