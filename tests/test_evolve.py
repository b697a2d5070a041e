"""evolve (search.cpp:41-71): the GA's host logic (keyed sample / mutate /
epsilon draws, survivors, sort by score then configuration) bit-exact against the oracle's
restatement with the linear test scorer (no GPU), plus the reference's parameter validation
(test_search.cpp:136-150)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    return moseslab


TASK = (2.0, 8.0, 9.0, 5.0)


def lin_scorer(knobs, w):
    def score(cfgs):
        out = []
        for c in cfgs:
            s = 0.0
            for k, v in enumerate(c):
                s = s + w[k] * float(v)
            out.append(s)
        return out
    return score


@pytest.mark.parametrize("params", [dict(), dict(population=7, generations=6, mutation_count=3, survivors=7),
                                    dict(population=64, generations=3, mutation_count=5, survivors=9,
                                         epsilon_random=0.5, seed=77),
                                    dict(population=16, generations=0, survivors=16, seed=3),
                                    dict(population=32, generations=4, epsilon_random=1.0, survivors=8, seed=9)])
@pytest.mark.parametrize("w", [[1.0, -0.5, 0.25, 2.0, -1.0], [0.0, 0.0, 0.0, 0.0, 0.0], [1e-3, 1.0, 0.0, 0.0, 1.0]])
def test_evolve_matches_oracle(ml, orc, params, w):
    knobs = orc.default_knob_template()
    vals, scores = ml.evolve(None, TASK, knobs, lin_w=w, **params)
    want = orc.evolve(knobs, lin_scorer(knobs, w), **params)
    assert vals.tolist() == [c for c, _ in want]
    assert scores.tolist() == [s for _, s in want]


def test_evolve_sorted_valid_and_elitist(ml, orc):
    # test_search.cpp:82-120: sorted by score then config; every candidate valid; best never lost
    knobs = orc.default_knob_template()
    w = [0.3, 0.7, -0.01, 0.5, 0.2]
    best_prev = None
    for g in range(0, 5):
        vals, scores = ml.evolve(None, TASK, knobs, generations=g, lin_w=w, seed=11)
        keys = [(-s, tuple(v)) for v, s in zip(vals.tolist(), scores.tolist())]
        assert keys == sorted(keys)
        for v in vals.tolist():
            assert all(x in d for x, (_, d) in zip(v, knobs))
        if best_prev is not None:
            assert scores[0] >= best_prev
        best_prev = scores[0]


def test_evolve_validation(ml, orc):
    knobs = orc.default_knob_template()
    for bad in [dict(population=0), dict(mutation_count=0), dict(survivors=0), dict(generations=-1),
                dict(population=4, survivors=5), dict(epsilon_random=1.5), dict(epsilon_random=-0.1)]:
        with pytest.raises(ml.MosesError) as e:
            ml.evolve(None, TASK, knobs, lin_w=[1.0] * 5, **bad)
        assert e.value.code == "invalid-config", bad
    single = [("tile_x", [4]), ("tile_y", [8])]
    with pytest.raises(ml.MosesError) as e:  # mutate_config on an all-singleton space
        ml.evolve(None, TASK, single, lin_w=[1.0, 1.0], population=2, survivors=1, generations=1,
                  epsilon_random=0.0)
    assert e.value.code == "immutable-space"
    vals, _ = ml.evolve(None, TASK, single, lin_w=[1.0, 1.0], population=3, survivors=3, generations=0)
    assert vals.tolist() == [[4, 8]] * 3


def test_evolve_property_vs_oracle(ml, orc):
    """Random SearchParams, linear scorers and knob spaces: bit-exact populations and scores."""
    pytest.importorskip("hypothesis")
    from hypothesis import given, settings
    from hypothesis import strategies as st

    @settings(max_examples=40, deadline=None)
    @given(st.integers(1, 20), st.integers(0, 4), st.integers(1, 4), st.integers(1, 20),
           st.floats(0.0, 1.0), st.integers(0, 2**64 - 1),
           st.lists(st.lists(st.integers(-50, 50), min_size=1, max_size=5, unique=True), min_size=1, max_size=4),
           st.lists(st.floats(-2.0, 2.0, allow_nan=False), min_size=4, max_size=4))
    def check(pop, gens, mc, surv, eps, seed, doms, w):
        surv = min(surv, pop)
        knobs = [("k%d" % i, sorted(d)) for i, d in enumerate(doms)]
        lw = w[:len(knobs)]
        if gens > 0 and all(len(d) == 1 for _, d in knobs) and eps < 1.0:
            return  # mutate_config raises ImmutableSpace on both sides (covered elsewhere)
        params = dict(population=pop, generations=gens, mutation_count=mc, survivors=surv, epsilon_random=eps,
                      seed=seed)
        vals, scores = ml.evolve(None, TASK, knobs, lin_w=lw, **params)
        want = orc.evolve(knobs, lin_scorer(knobs, lw), **params)
        assert vals.tolist() == [c for c, _ in want]
        assert scores.tolist() == [s for _, s in want]

    check()
