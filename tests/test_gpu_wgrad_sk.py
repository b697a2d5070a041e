"""Split-bf16 weight gradients split over the batch rows in clusters (csrc/gemm_wgrad_sk.cuh) against
the one-CTA-per-tile kernel (csrc/gemm_group.cuh) and the fp64 oracle.

Within a 128-row chunk both kernels issue the same tcgen05 MMAs in the same order, so with one split
per tile (S = 1) every weight row of the gradient is bit-identical to the tile kernel; only the bias
rows of 512-wide levels (summed on the CUDA cores instead of through the ones column) and the
split-order association of S > 1 differ, at fp32 rounding level. Results are deterministic for a
fixed S (fixed DSMEM reduction order)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG2 = [164, 512, 512, 512, 512, 1]
CFG5 = [164, 512, 512, 1]


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    L = moseslab.lib()
    assert L.moses_device_check() == 0, L.moses_last_error()
    L.moses_debug_set_wgrad_sk.argtypes = [C.c_int, C.c_int]
    yield moseslab
    L.moses_debug_set_wgrad_sk(1, 0)


def nrel(got, ref):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


def bias_mask(dims):
    """True at the bias entries of every level (flat layout: W block [in][out], then b)."""
    m = []
    for i in range(len(dims) - 1):
        m += [False] * (dims[i] * dims[i + 1]) + [True] * dims[i + 1]
    return np.array(m)


def grads(ml, dims, p, x, y, sk, splits=0):
    ml.lib().moses_debug_set_wgrad_sk(sk, splits)
    try:
        dm = ml.DeviceModel(p, ml.PREC_BF16X3, max(128, x.shape[0]))
        g, loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
        dm.close()
    finally:
        ml.lib().moses_debug_set_wgrad_sk(1, 0)
    return g, loss


def batch(dims, n, seed):
    rng = np.random.default_rng(seed)
    return rng.random((n, dims[0])), 0.1 + rng.random(n)


@pytest.mark.parametrize("dims", [CFG2, CFG5, [16, 512, 512, 1], [512, 512, 512, 1], [33, 512, 1]])
@pytest.mark.parametrize("n", [7, 300, 2500, 4096])
def test_one_split_equals_tile_kernel(ml, dims, n):
    p = ml.init_random(dims, 3, strict=False)
    x, y = batch(dims, n, n)
    g_old, l_old = grads(ml, dims, p, x, y, 0)
    g_sk, l_sk = grads(ml, dims, p, x, y, 1, splits=1)
    assert l_old == l_sk
    head = len(g_old) - (dims[-2] + 1)  # head level: column_dot, not the grouped kernel
    bm = bias_mask(dims)
    w = ~bm
    w[head:] = False
    assert np.array_equal(g_old[w], g_sk[w])
    assert nrel(g_sk[bm], g_old[bm]) < 2e-6
    assert np.array_equal(g_old[head:], g_sk[head:])


@pytest.mark.parametrize("dims,n", [(CFG2, 2560), (CFG5, 4096), ([512, 512, 512, 1], 1000)])
def test_splits_agree_and_are_deterministic(ml, dims, n):
    p = ml.init_random(dims, 5, strict=False)
    x, y = batch(dims, n, 9)
    g1, _ = grads(ml, dims, p, x, y, 1, splits=1)
    for s in (2, 3, 4, 5, 8, 0):  # 0: the launcher's own choice
        ga, _ = grads(ml, dims, p, x, y, 1, splits=s)
        gb, _ = grads(ml, dims, p, x, y, 1, splits=s)
        assert np.array_equal(ga, gb), s
        assert nrel(ga, g1) < 2e-6, s


@pytest.mark.parametrize("dims,n", [(CFG2, 2300), (CFG5, 4096)])
def test_gradients_vs_oracle(ml, orc, dims, n):
    """The benched shapes against the fp64 oracle (model.cpp:192-244): the split-K kernel sits exactly as
    far from fp64 as the tile kernel (the distance is set by the forward's ReLU-kink flips on these
    unpooled uniform rows, not by the weight-gradient GEMM), normwise and on the 99.9% quantile. The
    absolute bound on the benched pooled inputs is tests/test_gpu_bf16x3.py."""
    p = ml.init_random(dims, 12345, strict=False)
    x, y = batch(dims, n, 4)
    g_ref, loss_ref = orc.gradients(dims, p.params, x, y, threads=8)
    g, loss = grads(ml, dims, p, x, y, 1)
    g_old, _ = grads(ml, dims, p, x, y, 0)
    assert abs(loss - loss_ref) <= 1e-4 * abs(loss_ref)
    assert nrel(g, g_ref) <= nrel(g_old, g_ref) + 1e-5, (nrel(g, g_ref), nrel(g_old, g_ref))
    q = lambda a: float(np.quantile(np.abs(a - g_ref), 0.999) / np.max(np.abs(g_ref)))
    assert q(g) <= q(g_old) + 1e-5, (q(g), q(g_old))


def test_fused_update_matches_tile_kernel(ml):
    """moses_train_step: gradients + momentum update fused into the wgrad epilogue (weights, momentum
    and the hi/lo operand shadow) — split-K clusters against the tile kernel. One step from zero
    momentum: v = g at fp32 reassociation level, and the fp32 weights w - lr*v within one ulp of each
    other (an update of ~1e-7 on |w| ~ 0.05 is quantised by w's ulp). Three steps: the momentum still
    within 1e-3 (ReLU-kink flips of the slightly different weights)."""
    dims = CFG5
    p = ml.init_random(dims, 8, strict=False)
    for steps, tol in ((1, 1e-5), (3, 1e-3)):
        out = {}
        for sk in (0, 1):
            ml.lib().moses_debug_set_wgrad_sk(sk, 0)
            try:
                dm = ml.DeviceModel(p, ml.PREC_BF16X3, 4096)
                for s in range(steps):
                    x, y = batch(dims, 4096, 100 + s)
                    loss = C.c_double()
                    ml._ck(ml.lib().moses_train_step(dm.h, ml._p(np.ascontiguousarray(x)),
                                                     ml._p(np.ascontiguousarray(y)), 4096, dims[0], C.c_double(0.001),
                                                     C.c_double(0.9), C.byref(loss)))
                w = np.zeros(dm.P)
                v = np.zeros(dm.P)
                ml._ck(ml.lib().moses_model_download(dm.h, ml._p(w), ml._p(v), dm.P))
                out[sk] = (w, v)
                dm.close()
            finally:
                ml.lib().moses_debug_set_wgrad_sk(1, 0)
        assert nrel(out[1][1], out[0][1]) < tol, (steps, nrel(out[1][1], out[0][1]))
        if steps == 1:
            ulp = np.spacing(np.abs(out[0][0]).astype(np.float32)).astype(np.float64)
            dw0 = out[0][0] - p.params
            assert np.all(np.abs(out[1][0] - out[0][0]) <= ulp + 1e-5 * np.max(np.abs(dw0)))


@pytest.mark.parametrize("dims,n", [(CFG2, 2560), (CFG5, 4096), ([16, 512, 512, 512, 1], 700)])
def test_early_last_level_beside_the_chain(ml, dims, n):
    """The last hidden level's weight gradient launched beside the dZ chain (its own cluster width for
    the SMs the chain leaves free) equals the single grouped launch up to split-order association."""
    L = ml.lib()
    p = ml.init_random(dims, 13, strict=False)
    x, y = batch(dims, n, 3)
    L.moses_debug_set_wgrad_early(0)
    try:
        g0, l0 = grads(ml, dims, p, x, y, 1)
    finally:
        L.moses_debug_set_wgrad_early(1)
    g1, l1 = grads(ml, dims, p, x, y, 1)
    g2, _ = grads(ml, dims, p, x, y, 1)
    assert l0 == l1 and np.array_equal(g1, g2)
    assert nrel(g1, g0) < 2e-6


@pytest.mark.parametrize("n", [300, 512, 2560])
def test_fused_update_with_early_level_equals_single_launch(ml, n):
    """moses_train_step with the last level's weight gradient beside the dZ chain: that launch computes the
    gradient only and the level's update runs after the chain has read its weights (the chain's first layer
    uses them), so weights, momentum and the split operand shadow (via the next step) are bit-identical to
    the single grouped launch at the same cluster width — over small batches too, where the early launch
    would otherwise finish inside the chain's first layer."""
    L = ml.lib()
    dims = CFG2
    p = ml.init_random(dims, 21, strict=False)
    out = {}
    for early in (1, 0):
        L.moses_debug_set_wgrad_early(early)
        L.moses_debug_set_wgrad_sk(1, 2)
        try:
            dm = ml.DeviceModel(p, ml.PREC_BF16X3, max(128, n))
            for s in range(2):
                x, y = batch(dims, n, 300 + s)
                loss = C.c_double()
                ml._ck(L.moses_train_step(dm.h, ml._p(np.ascontiguousarray(x)), ml._p(np.ascontiguousarray(y)), n,
                                          dims[0], C.c_double(0.001), C.c_double(0.9), C.byref(loss)))
            w = np.zeros(dm.P)
            v = np.zeros(dm.P)
            ml._ck(L.moses_model_download(dm.h, ml._p(w), ml._p(v), dm.P))
            out[early] = (w, v, loss.value)
            dm.close()
        finally:
            L.moses_debug_set_wgrad_early(1)
            L.moses_debug_set_wgrad_sk(1, 0)
    assert np.array_equal(out[1][0], out[0][0]) and np.array_equal(out[1][1], out[0][1])
    assert out[1][2] == out[0][2]
