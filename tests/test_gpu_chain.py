"""The fused hidden-layer chain kernels (mlp_chain.cuh) and the grouped weight-gradient kernel
with the fused momentum update (gemm_group.cuh) against the per-layer GEMM path.

Both compute the same bf16 operands with the same tcgen05 K order and the same fp32 epilogue
arithmetic, so forward scores, penultimate activations and gradients must agree BITWISE.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0, moseslab.lib().moses_last_error()
    moseslab.lib().moses_debug_set_chain.argtypes = [ctypes.c_int]
    moseslab.lib().moses_debug_set_group.argtypes = [ctypes.c_int]
    yield moseslab
    moseslab.lib().moses_debug_set_chain(1)
    moseslab.lib().moses_debug_set_group(1)


def run(ml, fused, fn):
    ml.lib().moses_debug_set_chain(fused)
    ml.lib().moses_debug_set_group(fused)
    try:
        return fn()
    finally:
        ml.lib().moses_debug_set_chain(1)
        ml.lib().moses_debug_set_group(1)


@pytest.mark.parametrize("dims", [[164, 512, 512, 1], [164, 512, 512, 512, 512, 1], [16, 512, 1],
                                  [512, 512, 512, 512, 1], [100, 512, 512, 512, 512, 512, 512, 512, 512, 1]])
@pytest.mark.parametrize("n", [1, 130, 2300])
def test_chain_forward_and_gradients_bitwise(ml, dims, n):
    p = ml.init_random(dims, 4, strict=False)
    rng = np.random.default_rng(n)
    x, y = rng.random((n, dims[0])), 0.1 + rng.random(n)

    def go():
        dm = ml.DeviceModel(p, ml.PREC_BF16, 4096)
        s = ml.predict(dm, x)
        h = ml.penultimate_activations(dm, x)
        g, loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
        return s, h, g, loss

    s1, h1, g1, l1 = run(ml, 1, go)
    s0, h0, g0, l0 = run(ml, 0, go)
    assert np.array_equal(s1, s0)
    assert np.array_equal(h1, h0)
    assert np.array_equal(g1, g0)
    assert l1 == l0


def test_chain_with_adversary_bitwise(ml):
    dims = [16, 512, 512, 512, 1]
    p = ml.init_random(dims, 31, strict=False)
    rng = np.random.default_rng(1)
    x, y = rng.random((40, 16)), 0.1 + rng.random(40)
    replay = rng.random((256, 16))
    u = rng.normal(0, 0.05, 512)

    def go():
        adv = ml.make_adversary(replay, 512, 7)
        adv.set(u, 0.03)
        dm = ml.DeviceModel(p, ml.PREC_BF16, 512)
        return ml.gradients(dm, ml.RankingBatch(x, y), adv, 0.5, want_loss=True)

    g1, l1 = run(ml, 1, go)
    g0, l0 = run(ml, 0, go)
    assert np.array_equal(g1, g0) and l1 == l0


def test_chain_pooled_graph_bitwise(ml):
    """The bench path: pooled CUDA-graph training steps (gather -> chain fwd -> rank -> chain dZ -> wgrad -> update)."""
    import torch

    dims = [164, 512, 512, 512, 512, 1]
    L = ml.lib()

    def go():
        programs, max_stmts, batch = 2048, 8, 256
        off = ml.synth_offsets(5, programs, max_stmts)
        rows = int(off[-1])
        rows_pad = int(max(off[i + batch] - off[i] for i in range(0, programs, batch)))
        rows_pad = (rows_pad + 127) // 128 * 128
        dm = ml.DeviceModel(ml.init_random(dims, 2, strict=False), ml.PREC_BF16, rows_pad)
        ld = dm.packed_ld
        X = torch.zeros((rows, ld), dtype=torch.bfloat16, device="cuda")
        Y = torch.empty(programs, dtype=torch.float32, device="cuda")
        assert L.moses_synth_features_device(3, 0, rows, dims[0], ml.DTYPE_BF16, X.data_ptr(), ld) == 0
        assert L.moses_synth_labels_device(3, 0, programs, Y.data_ptr()) == 0
        O = torch.from_numpy(np.asarray(off, dtype=np.int64)).cuda()
        torch.cuda.synchronize()
        ml._ck(L.moses_train_graph_create_pooled(dm.h, X.data_ptr(), ld, Y.data_ptr(), O.data_ptr(),
                                                 programs // batch, batch, rows_pad, 0.001, 0.9, 1))
        ml._ck(L.moses_train_graph_launch(dm.h, 5))
        torch.cuda.synchronize()
        return dm.download()

    w1 = run(ml, 1, go)
    w0 = run(ml, 0, go)
    assert np.array_equal(w1.params, w0.params)
    assert np.array_equal(w1.momentum, w0.momentum)


@pytest.mark.parametrize("dims", [[164, 512, 512, 512, 512, 1], [33, 72, 40, 1]])
def test_fused_train_step_device_bitwise(ml, dims):
    """moses_train_step_device: gradients + momentum update; fused into the grouped wgrad epilogue
    when enabled — identical parameters and momentum to the separate update kernel."""
    import torch

    p = ml.init_random(dims, 9, strict=False)
    n = 700
    rng = np.random.default_rng(3)
    x = rng.random((n, dims[0]))
    y = torch.from_numpy(0.1 + rng.random(n)).float().cuda()

    def go():
        dm = ml.DeviceModel(p, ml.PREC_BF16, 1024)
        ld = dm.packed_ld
        X = torch.zeros((n, ld), dtype=torch.bfloat16, device="cuda")
        X[:, :dims[0]] = torch.from_numpy(x).to(torch.bfloat16).cuda()
        X[:, dims[0]] = 1.0
        torch.cuda.synchronize()
        for _ in range(3):
            ml._ck(ml.lib().moses_train_step_device(dm.h, X.data_ptr(), ld, y.data_ptr(), n, 0.001, 0.9, None))
        return dm.download()

    a = run(ml, 1, go)
    b = run(ml, 0, go)
    assert np.array_equal(a.params, b.params) and np.array_equal(a.momentum, b.momentum)


@pytest.mark.parametrize("n", [2, 12, 511, 512, 3000])
@pytest.mark.parametrize("pooled", [False, True])
def test_rank_step_matches_two_kernel_path(ml, n, pooled):
    """rank_step (pairs + finalize in one launch, last-CTA reduction) vs rank_pairs + rank_finalize:
    identical per-row coefficients -> bitwise-equal gradients; the loss uses log1p(e) = -log(1/(1+e))
    (fast log of the reciprocal) and a different summation order: equal to ~1e-6."""
    L = ml.lib()
    L.moses_debug_set_rank_fused.argtypes = [ctypes.c_int]
    dims = [164, 512, 512, 1]
    p = ml.init_random(dims, 6, strict=False)
    rng = np.random.default_rng(n)
    y = 0.1 + np.round(rng.random(n), 2)  # ties included
    if pooled:
        off = ml.synth_offsets(2, n, 5)
        x = rng.random((int(off[-1]), 164))
    else:
        x = rng.random((n, 164))

    def go(flag):
        L.moses_debug_set_rank_fused(flag)
        L.moses_debug_set_rank_sym(0)  # bitwise against the two-kernel path: the grid / cluster forms
        try:
            dm = ml.DeviceModel(p, ml.PREC_BF16, 16384)
            if pooled:
                return ml.gradients_pooled(dm, x, off, y, want_loss=True)
            return ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
        finally:
            L.moses_debug_set_rank_fused(1)
            L.moses_debug_set_rank_sym(1)

    g1, l1 = go(1)
    g0, l0 = go(0)
    assert np.array_equal(g1, g0)
    assert abs(l1 - l0) <= 2e-6 * max(1.0, abs(l0))
