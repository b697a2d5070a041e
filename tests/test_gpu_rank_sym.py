"""Symmetric form of the fused ranking step (csrc/kernels.cu rank_sym_kernel): each unordered pair of
the batch evaluated once, in 32 x 32 tiles of the pair matrix's upper triangle, for batches past the
16-CTA cluster form (cfg5: 4096 programs). Against the grid form (every pair from both rows, same
pair arithmetic): backward coefficients equal up to summation order; against the fp64 oracle
(model.cpp:71-106 via gradients) on an FP32-precision handle; deterministic."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    L = moseslab.lib()
    assert L.moses_device_check() == 0, L.moses_last_error()
    yield moseslab
    L.moses_debug_set_rank_grid(0)
    L.moses_debug_set_rank_sym(1)


def nrel(got, ref):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


def run(ml, dm, kind, x, y, off, form):
    L = ml.lib()
    L.moses_debug_set_rank_grid(1 if form == "grid" else 0)
    try:
        if kind == "plain":
            return ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
        return ml.gradients_pooled(dm, x, off, y, want_loss=True)
    finally:
        L.moses_debug_set_rank_grid(0)


@pytest.mark.parametrize("kind,n", [("plain", 1500), ("plain", 2048), ("plain", 3001), ("plain", 4096),
                                    ("plain", 6000), ("pooled", 2000), ("pooled", 4096)])
@pytest.mark.parametrize("labels", ["distinct", "ties"])
def test_symmetric_matches_grid_form(ml, kind, n, labels):
    # FP32 handles: on bf16 ones an fp32-ulp change of a row coefficient can flip the bf16 rounding
    # of that row's dZ and show up at bf16 precision in the weight gradients
    dims = [164, 512, 512, 1]
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    dm = ml.DeviceModel(ml.CostModelParams(dims, f32(ml.init_random(dims, 4).params)), ml.PREC_FP32, 40000)
    rng = np.random.default_rng(n)
    y = rng.random(n) if labels == "distinct" else np.round(rng.random(n) * 8) / 8
    off = ml.synth_offsets(7, n, 8) if kind == "pooled" else None
    x = rng.random((int(off[-1]) if off is not None else n, 164))
    g_sym, l_sym = run(ml, dm, kind, x, y, off, "sym")
    g_sym2, l_sym2 = run(ml, dm, kind, x, y, off, "sym")
    g_grid, l_grid = run(ml, dm, kind, x, y, off, "grid")
    assert np.array_equal(g_sym, g_sym2) and l_sym == l_sym2  # deterministic
    assert abs(l_sym - l_grid) <= 1e-6 * max(1.0, abs(l_grid))
    # head bias: sum of all score gradients, zero up to cancellation (each pair adds -sigma and +sigma)
    hb = dm.P - 1
    assert nrel(g_sym[:hb], g_grid[:hb]) < 1e-5
    assert abs(g_sym[hb] - g_grid[hb]) <= 1e-3 * np.max(np.abs(g_grid[:hb]))


def test_symmetric_vs_oracle_fp32(ml, orc):
    """FP32 parity mode (3xTF32, <= 1e-5 forward): loss and gradients of a 4096-program batch against
    the fp64 oracle — the ranking term of every pair enters through the symmetric form."""
    dims = [164, 512, 512, 1]
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    p = ml.init_random(dims, 21)
    p32 = ml.CostModelParams(dims, f32(p.params))
    rng = np.random.default_rng(5)
    n = 4096
    x = f32(rng.random((n, 164)) * 0.5)
    y = f32(0.1 + rng.random(n))
    g_ref, loss_ref = orc.gradients(dims, p32.params, x, y, threads=8)
    dm = ml.DeviceModel(p32, ml.PREC_FP32, n)
    g, loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
    assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref)
    assert nrel(g, g_ref) < 1e-4
    assert float(np.quantile(np.abs(g - g_ref), 0.999) / np.max(np.abs(g_ref))) < 1e-5


def test_symmetric_all_ties_and_tiny(ml):
    """Every label equal: no pairs, zero loss and zero gradient; n just past the cluster form."""
    dims = [16, 512, 512, 1]
    dm = ml.DeviceModel(ml.init_random(dims, 2), ml.PREC_BF16, 4096)
    x = np.random.default_rng(0).random((3000, 16))
    g, loss = ml.gradients(dm, ml.RankingBatch(x, np.full(3000, 0.5)), want_loss=True)
    assert loss == 0.0 and not np.any(g)
