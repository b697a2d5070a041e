"""The oracle's MMD^2 loss restatement (north-star (4); no reference code exists for it, so its parity is
pinned here): the analytic row gradients and the full model gradient with beta * MMD^2 against central
finite differences of the objective, and beta = 0 reducing to gradients() exactly."""
import numpy as np


def test_mmd2_row_gradients_finite_differences(orc):
    rng = np.random.default_rng(0)
    xs, xt = rng.random((7, 6)), rng.random((5, 6)) + 0.3
    v, gs, gt = orc.mmd2_grad(xs, xt, 0.8)
    assert abs(v - orc.mmd2(xs, xt, 0.8)) <= 1e-14
    eps = 1e-6
    for arr, g in ((xs, gs), (xt, gt)):
        for (i, j) in ((0, 0), (2, 3), (arr.shape[0] - 1, 5)):
            p, m = arr.copy(), arr.copy()
            p[i, j] += eps
            m[i, j] -= eps
            a = (orc.mmd2(p, xt, 0.8) - orc.mmd2(m, xt, 0.8)) if arr is xs else \
                (orc.mmd2(xs, p, 0.8) - orc.mmd2(xs, m, 0.8))
            assert abs(a / (2 * eps) - g[i, j]) <= 1e-7 * max(1.0, abs(g[i, j]))


def test_gradients_mmd_finite_differences(orc):
    dims = [4, 8, 8, 1]
    rng = np.random.default_rng(1)
    w = orc.init_random(dims, 3)
    x, y, src = rng.random((6, 4)), 0.1 + rng.random(6), rng.random((5, 4))
    g, _ = orc.gradients_mmd(dims, w, x, y, src, 0.5, 1.3)

    def obj(wv):
        return orc.gradients_mmd(dims, wv, x, y, src, 0.5, 1.3)[1]

    for k in rng.choice(len(w), 20, replace=False):
        wp, wm = w.copy(), w.copy()
        wp[k] += 1e-6
        wm[k] -= 1e-6
        fd = (obj(wp) - obj(wm)) / 2e-6
        assert abs(fd - g[k]) <= 1e-4 * max(abs(g[k]), 1e-6)


def test_gradients_mmd_beta0_is_gradients(orc):
    dims = [4, 8, 8, 1]
    rng = np.random.default_rng(2)
    w = orc.init_random(dims, 4)
    x, y, src = rng.random((6, 4)), 0.1 + rng.random(6), rng.random((5, 4))
    g0, l0 = orc.gradients_mmd(dims, w, x, y, src, 0.0, 1.0)
    g1, l1 = orc.gradients(dims, w, x, y)
    assert np.array_equal(g0, g1) and l0 == l1
