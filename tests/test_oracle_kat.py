"""Pin the CPU oracle against the reference's own known-answer tests.

Every case cites the reference test it restates (tests/golden/reference_kats.json
holds the values). No GPU needed.
"""
import json
import math
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
KAT = json.load(open(os.path.join(HERE, "golden", "reference_kats.json")))


def random_rows(rows, cols, seed):
    """RngStream(seed) row-major uniform01 fill (test_model.cpp:24-30)."""
    out = np.zeros((rows, cols))
    k = 0
    for r in range(rows):
        for c in range(cols):
            k += 1
            out[r, c] = (oracle_draw(seed, k) >> 11) * 2.0 ** -53
    return out


def oracle_draw(seed, k):
    import oracle

    return oracle.lib().orc_splitmix_at(seed, k)


def random_batch(rows, dim, seed):
    """test_model.cpp:32-40."""
    x = random_rows(rows, dim, seed)
    y = np.array([0.1 + (oracle_draw(seed + 1, r + 1) >> 11) * 2.0 ** -53 for r in range(rows)])
    return x, y


def test_splitmix_and_fnv(orc):
    got = [orc.splitmix_draw(0, k) for k in (1, 2, 3)]
    assert got == [int(v, 16) for v in KAT["splitmix64_seed0_first3"]["values"]]
    f = KAT["fnv"]
    assert orc.fnv_u64s([]) == int(f["empty"], 16)
    assert orc.fnv_str("a") == int(f["a"], 16)
    assert orc.fnv_u64s([42]) == int(f["u64_42"], 16)
    assert orc.lib().orc_fnv_u64_str(7, b"x") == int(f["u64_7_then_x"], 16)
    assert orc.fnv_u64s([16, 32, 16, 8, 32]) == int(KAT["config_hash_16_32_16_8_32"]["value"], 16)


def test_uniform_gaussian(orc):
    assert orc.uniform01_first(5) == pytest.approx(KAT["uniform01_seed5_first"]["value"], rel=1e-15)
    assert orc.gaussian_first(99) == pytest.approx(KAT["gaussian_seed99_first"]["value"], rel=1e-15)


def test_param_count(orc):
    assert orc.param_count([16, 512, 512, 1]) == KAT["param_count_16_512_512_1"]["value"]
    assert orc.param_count([164, 512, 512, 1]) == 347649
    assert orc.param_count([164, 256, 256, 1]) == 108289
    assert orc.param_count([164, 512, 512, 512, 512, 1]) == 872961


def test_init_bounds_and_determinism(orc):
    a = orc.init_random([16, 512, 512, 1], 4)
    b = orc.init_random([16, 512, 512, 1], 4)
    c = orc.init_random([16, 512, 512, 1], 5)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    off = 0
    for fi, fo in ((16, 512), (512, 512), (512, 1)):
        w = a[off:off + fi * fo]
        assert np.abs(w).max() <= math.sqrt(6.0 / (fi + fo))
        assert np.all(a[off + fi * fo: off + fi * fo + fo] == 0.0)
        off += fi * fo + fo
    with pytest.raises(Exception, match="bad-dims"):
        orc.init_random([16, 512, 1], 0)
    with pytest.raises(Exception, match="bad-dims"):
        orc.init_random([16, 512, 512, 2], 0)


def test_golden_model_predictions(orc):
    g = KAT["golden_model_v1"]
    w = orc.init_random(g["dims"], g["seed"])
    x = np.array([[(r + 1) * 0.1 + c * 0.01 for c in range(16)] for r in range(3)])
    s, _ = orc.forward(g["dims"], w, x)
    for got, want in zip(s, g["scores"]):
        assert got == pytest.approx(want, rel=g["rel"])
    # the file form (MOSM v1) pins layout: 12 + 16*P bytes
    blob = orc.serialize(g["dims"], w)
    assert blob[:4] == b"MOSM" and len(blob) == 12 + 16 * 271873


def test_forward_hand_pass(orc):
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 3)
    x = random_rows(5, 4, 10)
    s, h2 = orc.forward(dims, w, x)
    W0 = w[:32].reshape(4, 8).T; b0 = w[32:40]
    W1 = w[40:104].reshape(8, 8).T; b1 = w[104:112]
    w2 = w[112:120]; b2 = w[120]
    for r in range(5):
        h = np.maximum(W0 @ x[r] + b0, 0)
        h = np.maximum(W1 @ h + b1, 0)
        assert s[r] == pytest.approx(w2 @ h + b2, rel=1e-10)
        assert np.allclose(h2[r], h, rtol=1e-12, atol=0)


def test_ranking_loss_hand_cases(orc):
    loss, _, _ = orc.ranking_terms(np.array([2.0, 1.0]), np.array([3.0, 1.0]))
    assert loss == pytest.approx(math.log(1 + math.exp(-1)), rel=1e-12)
    loss, _, _ = orc.ranking_terms(np.array([1.0, 1.0]), np.array([3.0, 1.0]))
    assert loss == pytest.approx(math.log(2), rel=1e-12)
    loss, gs, pairs = orc.ranking_terms(np.array([1.0, 1.0]), np.array([1.0, 1.0]))
    assert loss == 0.0 and pairs == 0 and np.all(gs == 0)


def test_ranking_loss_brute_force(orc):
    rng = np.random.default_rng(14)
    s = rng.uniform(-2, 2, 8)
    y = rng.uniform(0, 1, 8)
    tot, pairs = 0.0, 0
    for i in range(8):
        for j in range(8):
            if y[i] > y[j]:
                tot += math.log(1 + math.exp(-(s[i] - s[j])))
                pairs += 1
    loss, _, p = orc.ranking_terms(s, y)
    assert p == pairs and loss == pytest.approx(tot / pairs, rel=1e-12)
    # translation invariance (test_model.cpp:186-203)
    loss2, _, _ = orc.ranking_terms(s + 17.5, y)
    assert loss2 == pytest.approx(loss, rel=1e-12)


def grazes_kink(dims, w, rows, margin):
    W0 = w[:32].reshape(4, 8); b0 = w[32:40]
    W1 = w[40:104].reshape(8, 8); b1 = w[104:112]
    z1 = rows @ W0 + b0
    if np.abs(z1).min() < margin:
        return True
    z2 = np.maximum(z1, 0) @ W1 + b1
    return np.abs(z2).min() < margin


def test_finite_difference_gradients(orc):
    """test_model.cpp:225-256 / acceptance.cpp:77-127: rel err < 1e-4, beta in {0, 0.01}."""
    dims = [4, 8, 8, 1]
    h = 1e-4
    done, seed, worst = 0, 100, 0.0
    while done < 10:
        seed += 1
        w = orc.init_random(dims, seed)
        x, y = random_batch(6, 4, seed * 3 + 1)
        replay = random_rows(8, 4, seed * 3 + 2)
        adv = (np.zeros(8), 0.0, replay)
        beta = 0.0 if done % 2 == 0 else 0.01
        if grazes_kink(dims, w, np.vstack([x, replay]), 1e-3):
            continue
        # a non-zero discriminator so the adversary term is exercised
        aw = np.linspace(-0.3, 0.4, 8)
        adv = (aw, 0.05, replay)
        g, _ = orc.gradients(dims, w, x, y, adv, beta)
        for i in range(len(w)):
            wp = w.copy(); wp[i] += h
            wm = w.copy(); wm[i] -= h
            fd = (orc.objective(dims, wp, x, y, adv, beta) - orc.objective(dims, wm, x, y, adv, beta)) / (2 * h)
            denom = max(abs(fd), abs(g[i]), 1e-3)
            worst = max(worst, abs(fd - g[i]) / denom)
        done += 1
    assert worst < 1e-4


def test_beta_zero_bit_exact(orc):
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 8)
    x, y = random_batch(6, 4, 21)
    adv = (np.zeros(8), 0.0, random_rows(5, 4, 22))
    a, _ = orc.gradients(dims, w, x, y, adv, 0.0)
    b, _ = orc.gradients(dims, w, x, y, None, 0.0)
    assert np.array_equal(a, b)


def test_objective_matches_gradient_loss(orc):
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 30)
    x, y = random_batch(6, 4, 31)
    adv = (np.linspace(-0.2, 0.2, 8), 0.1, random_rows(7, 4, 32))
    _, loss = orc.gradients(dims, w, x, y, adv, 0.01)
    assert loss == pytest.approx(orc.objective(dims, w, x, y, adv, 0.01), rel=1e-12)


def test_pair_free_batch_zero_gradient(orc):
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 7)
    x, _ = random_batch(4, 4, 20)
    g, _ = orc.gradients(dims, w, x, np.ones(4))
    assert np.all(g == 0)


def test_update_arithmetic(orc):
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 40)
    w[0] = 1.0
    g = np.zeros_like(w); g[0] = 2.0
    w2, _ = orc.apply_update(w, np.zeros_like(w), g, 0.001)
    assert w2[0] == pytest.approx(0.998, rel=1e-15)
    assert np.array_equal(w2[1:], w[1:])
    q = orc.init_random(dims, 41)
    w0 = q[0]
    q1, m1 = orc.apply_update(q, np.zeros_like(q), g, 0.001, 0.9, use_momentum=True)
    q2, _ = orc.apply_update(q1, m1, g, 0.001, 0.9, use_momentum=True)
    assert q2[0] == pytest.approx(w0 - 0.001 * 2.0 - 0.001 * (0.9 * 2.0 + 2.0), rel=1e-15)
    # all-variant mask is a no-op (test_model.cpp:310-326)
    q3, _ = orc.apply_update(q, np.zeros_like(q), np.ones_like(q), 0.001, mask=np.zeros(len(q), bool))
    assert np.array_equal(q3, q)


def test_xi_flat_order_and_normalization(orc):
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 1)
    g = np.zeros_like(w)
    w[0], g[0] = 0.2, 3.0          # w[0](0,0)
    w[1], g[1] = -0.5, 4.0         # w[0](1,0): column-major
    xi = orc.xi_scores(w, g, False)
    assert xi[0] == pytest.approx(0.6, rel=1e-15) and xi[1] == pytest.approx(2.0, rel=1e-15)
    w[32], g[32] = 2.0, 5.0        # b[0](0) at flat 32
    w[40], g[40] = 3.0, 1.0        # w[1](0,0) at flat 40
    xi = orc.xi_scores(w, g, False)
    assert xi[32] == pytest.approx(10.0) and xi[40] == pytest.approx(3.0)
    xin = orc.xi_scores(w, g, True)
    assert xin.max() == pytest.approx(1.0, rel=1e-15)


def test_partition_kats(orc):
    t = KAT["threshold_strict"]
    m = orc.partition(np.array(t["xi"]), True, orc.THRESHOLD, t["theta"])
    assert list(m) == t["mask"]
    with pytest.raises(Exception, match="unnormalized-threshold"):
        orc.partition(np.full(4, 2.0), False, orc.THRESHOLD, 0.5)
    r = KAT["ratio_ties"]
    m = orc.partition(np.array(r["xi"]), False, orc.RATIO, r["rho"])
    assert sorted(np.flatnonzero(m)) == r["kept"]
    for bad in (0.0, 1.5, -0.1):
        with pytest.raises(Exception, match="invalid-ratio"):
            orc.partition(np.ones(4), False, orc.RATIO, bad)
    assert orc.partition(np.zeros(9), False, orc.RATIO, 1.0).sum() == 9


def test_ratio_popcounts_canonical_scale(orc):
    k = KAT["ratio_popcounts_271873"]
    n = 271873
    xi = np.array([(orc.lib().orc_splitmix_at(8, i + 1) >> 11) * 2.0 ** -53 for i in range(n)])
    for rho, want in zip(k["rho"], k["popcount"]):
        assert orc.partition(xi, False, orc.RATIO, rho).sum() == want


def test_variant_decay(orc):
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 4)
    w[0] = 1.0
    mask = np.zeros(len(w), bool)
    w1 = orc.variant_decay(w, mask, 0.001, 0.01)
    assert abs(w1[0] - 0.99999) < 1e-12
    q = orc.init_random(dims, 5)
    i = 40 + 3 * 8 + 3  # w[1](3,3)
    q0 = q[i]
    for _ in range(50):
        q = orc.variant_decay(q, mask, 0.001, 0.01)
    assert abs(q[i] - q0 * (1 - 0.001 * 0.01) ** 50) < 1e-12
    z = orc.variant_decay(w, mask, 0.5, 0.0)
    assert z.tobytes() == w.tobytes()
    for a, l in ((1.0, 1.0), (2.0, 0.5), (0.1, -0.5)):
        with pytest.raises(Exception, match="unstable-decay"):
            orc.variant_decay(w, mask, a, l)


def test_discriminator(orc):
    z = np.zeros(5)
    assert orc.disc_ce(z, z) == pytest.approx(math.log(2), rel=1e-15)
    assert orc.disc_ce(np.full(5, 10.0), np.full(5, -10.0)) < 1e-4
    assert orc.disc_ce(np.full(5, -10.0), np.full(5, 10.0)) > 5.0
    h = random_rows(5, 8, 21)
    aw, ab, loss = orc.adversarial_term(np.zeros(8), 0.0, h, h)
    assert loss == pytest.approx(math.log(2), rel=1e-12)
    # separable toy (test_lottery.cpp:289-312)
    hs = random_rows(32, 2, 31); hs[:, 0] += 2.0
    ht = random_rows(32, 2, 32)
    aw, ab = np.zeros(2), 0.0
    first = None
    for step in range(200):
        aw, ab, l = orc.adversarial_term(aw, ab, hs, ht)
        first = l if first is None else first
    assert l < first and l < 0.35


def test_topk_order(orc):
    s = np.array([0.5, 0.9, 0.5, 0.1, 0.9, 0.5])
    assert list(orc.topk(s, 4)) == [1, 4, 0, 2]


def test_synthetic_generator_matches_rng(orc):
    x = orc.synth_features(1, 5, 2, 4)
    key = orc.lib().orc_fnv_u64s  # noqa: F841  (keyed streams checked via oracle KeyBuilder)
    assert x.shape == (2, 4) and np.all((x >= 0) & (x < 1))
    off = orc.synth_offsets(1, 100, 8)
    lens = np.diff(off)
    assert lens.min() >= 1 and lens.max() <= 8


def test_pooled_gradients_reduce_and_fd(orc):
    """Segment-sum pooling (north-star extension): S == 1 is exactly gradients(); FD agreement otherwise."""
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 3)
    rng = np.random.default_rng(0)
    x, y = rng.random((7, 4)), 0.1 + rng.random(7)
    g1, l1 = orc.gradients_pooled(dims, w, x, np.arange(8), y)
    g2, l2 = orc.gradients(dims, w, x, y)
    assert np.array_equal(g1, g2) and l1 == l2
    off = np.array([0, 2, 3, 6, 7])
    yp = 0.1 + rng.random(4)
    g, _ = orc.gradients_pooled(dims, w, x, off, yp)
    h, worst = 1e-6, 0.0
    for i in range(len(w)):
        wp, wm = w.copy(), w.copy()
        wp[i] += h
        wm[i] -= h
        fd = (orc.gradients_pooled(dims, wp, x, off, yp)[1] - orc.gradients_pooled(dims, wm, x, off, yp)[1]) / (2 * h)
        worst = max(worst, abs(fd - g[i]) / max(abs(fd), abs(g[i]), 1e-3))
    assert worst < 1e-4


# ---------------------------------------------------------------- knob space (space.cpp:140-197)
def test_feature_encoding_reference_vector(orc):
    k = KAT["feature_encoding"]
    knobs = orc.default_knob_template()
    f, h, v = orc.encode_configs(k["task"], knobs, 0, KAT["default_space_size"]["value"])
    i = [j for j in range(len(v)) if list(v[j]) == k["config"]]
    assert len(i) == 1
    got = f[i[0]]
    for a, b in zip(got[:10], k["features"]):
        assert abs(a - b) <= k["eps"] * max(1.0, abs(b))
    assert np.all(got[10:] == 0.0)
    assert int(h[i[0]]) == int(KAT["config_hash_16_32_16_8_32"]["value"], 16)


def test_work_term_clamps(orc):
    k = KAT["work_clamp"]
    knobs = [(n, [c]) for (n, _), c in zip(orc.default_knob_template(), k["config"])]
    for g, want in zip((k["low_gflops"], k["high_gflops"]), k["f7"]):
        f, _, _ = orc.encode_configs((g, 8.0, 9.0, 5.0), knobs, 0, 1)
        assert f[0, 7] == want


def test_enumeration_order_and_completeness(orc):
    k = KAT["enumeration_order"]
    knobs = [(n, d) for (n, _), d in zip(orc.default_knob_template(), k["domains"])]
    _, _, v = orc.encode_configs((2.0, 8.0, 9.0, 5.0), knobs, 0, len(k["configs"]))
    assert v.tolist() == k["configs"]
    n = KAT["default_space_size"]["value"]
    _, h, v = orc.encode_configs((2.0, 8.0, 9.0, 5.0), orc.default_knob_template(), 0, n)
    assert len({tuple(r) for r in v.tolist()}) == n  # no duplicates
    assert v.tolist() == sorted(v.tolist())          # lexicographic
    assert len(set(h.tolist())) == n                 # hashes distinct on the default space


# ---------------------------------------------------------------- simulated hardware (oracle.cpp:33-105)
SIM = json.load(open(os.path.join(HERE, "golden", "simulated_oracle.json")))


def _index_of(orc, knobs, values):
    idx = 0
    for (name, dom), v in zip(knobs, values):
        idx = idx * len(dom) + dom.index(v)
    return idx


def test_reference_measurement_values(orc):
    k = SIM["reference_measurement"]
    knobs = orc.default_knob_template()
    i = _index_of(orc, knobs, k["config"])
    clean, thr, lat, wall = orc.measure_configs(k["device"], k["task"]["id"], k["task"], knobs, k["seed"], i, 1)
    assert clean[0] == pytest.approx(k["clean_latency_ms"], rel=k["eps"])
    assert thr[0] == pytest.approx(k["throughput_gflops"], rel=k["eps"])
    assert lat[0] == pytest.approx(k["latency_ms"], rel=k["eps"])
    assert wall[0] == pytest.approx(k["device"]["measure_overhead_ms"] + 3 * lat[0], rel=1e-15)


def test_golden_true_best_exact(orc):
    """proj/tests/test_oracle.cpp:313-335 compares these exactly; so does the oracle restatement."""
    tasks = {t["id"]: t for t in SIM["tasks"]["list"]}
    knobs = orc.default_knob_template()
    for e in SIM["true_best"]["entries"]:
        dev = SIM["devices"][e["device_id"]]
        values, lat = orc.true_best(dev, tasks[e["task_id"]], knobs)
        assert values == e["values"], e
        assert lat == e["latency_ms"], e
