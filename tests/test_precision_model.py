"""The operand-precision model reduces to the fp64 oracle when nothing is rounded."""
import numpy as np

from precision_model import bf16_rn, device_gradients, nrel, tf32_rna


def test_model_matches_oracle_without_rounding(orc):
    for dims in ([4, 8, 8, 1], [16, 64, 32, 1], [20, 32, 32, 32, 1]):
        w = orc.init_random(dims, 5, strict=False)
        rng = np.random.default_rng(1)
        x, y = rng.random((37, dims[0])), 0.1 + rng.random(37)
        g_ref, loss_ref = orc.gradients(dims, w, x, y)
        g, loss = device_gradients(dims, w, x, y, "none")
        assert nrel(g, g_ref) < 1e-12 and abs(loss - loss_ref) < 1e-12


def test_rounding_helpers():
    assert tf32_rna(np.array([1.0 + 2 ** -11]))[0] == 1.0 + 2 ** -10  # tie away from zero
    assert tf32_rna(np.array([-(1.0 + 2 ** -11)]))[0] == -(1.0 + 2 ** -10)
    assert bf16_rn(np.array([1.0 + 2 ** -8]))[0] == 1.0  # tie to even
    assert bf16_rn(np.array([1.0 + 3 * 2 ** -8]))[0] == 1.0 + 2 ** -6


def test_model_with_adversary_matches_oracle(orc):
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 9)
    rng = np.random.default_rng(2)
    x, y = rng.random((6, 4)), 0.1 + rng.random(6)
    replay = rng.random((5, 4))
    u = rng.normal(0, 0.3, 8)
    for beta in (0.0, 0.01, 0.7):
        g_ref, l_ref = orc.gradients(dims, w, x, y, (u, 0.1, replay), beta)
        g, l = device_gradients(dims, w, x, y, "none", (u, 0.1, replay), beta)
        assert nrel(g, g_ref) < 1e-12 and abs(l - l_ref) < 1e-12


def test_pooled_model_matches_oracle(orc):
    from precision_model import device_gradients_pooled

    dims = [6, 16, 16, 1]
    w = orc.init_random(dims, 4)
    off = orc.synth_offsets(2, 9, 4)
    rng = np.random.default_rng(5)
    x, y = rng.random((int(off[-1]), 6)), 0.1 + rng.random(9)
    g_ref, l_ref = orc.gradients_pooled(dims, w, x, off, y)
    g, l = device_gradients_pooled(dims, w, x, off, y, "none")
    assert nrel(g, g_ref) < 1e-12 and abs(l - l_ref) < 1e-12
