"""Candidate generation on the device (space.cu) against the oracle's
restatement of space.cpp:140-197 (itself pinned by the reference's KATs in test_oracle_kat.py):
enumeration order and knob values and FNV-1a hashes bit-exact, feature rows within fp64 rounding
(f64 output) and equal after the single rounding to the model's operand type (f32 output)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TASK = (2.0, 8.0, 9.0, 5.0)  # test_space.cpp:19-28


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0, moseslab.lib().moses_last_error()
    return moseslab


def big_space():
    """6 knobs, 10,223,616 configurations (the 5 template knobs with wider domains + an untemplated one)."""
    return [("tile_x", [1 << i for i in range(16)]), ("tile_y", [1 << i for i in range(16)]),
            ("unroll", [0, 1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 128, 256, 512]),
            ("vectorize", [1 << i for i in range(8)]), ("parallel", [1 << i for i in range(13)]),
            ("split", list(range(1, 25)))]


def run_device(ml, task, knobs, first, n, dtype, D=16, ld=16):
    import torch

    tdt = {ml.DTYPE_F64: torch.float64, ml.DTYPE_F32: torch.float32, ml.DTYPE_BF16: torch.bfloat16}[dtype]
    F = torch.full((n, ld), -7.0, dtype=tdt, device="cuda")
    H = torch.zeros(n, dtype=torch.int64, device="cuda")
    V = torch.zeros((n, len(knobs)), dtype=torch.int64, device="cuda")
    ml.encode_configs_device(task, knobs, first, n, dtype, ctypes.c_void_p(F.data_ptr()), ld, D,
                             ctypes.c_void_p(H.data_ptr()), ctypes.c_void_p(V.data_ptr()))
    torch.cuda.synchronize()
    return F.float().cpu().double().numpy() if dtype == ml.DTYPE_BF16 else F.cpu().numpy(), \
        H.cpu().numpy().view(np.uint64), V.cpu().numpy()


def test_default_space_full_enumeration(ml, orc):
    knobs = orc.default_knob_template()
    f_ref, h_ref, v_ref = orc.encode_configs(TASK, knobs, 0, 8820)
    f, h, v = run_device(ml, TASK, knobs, 0, 8820, ml.DTYPE_F64)
    assert np.array_equal(v, v_ref)
    assert np.array_equal(h, h_ref)
    assert np.max(np.abs(f - f_ref)) <= 1e-15
    f32, _, _ = run_device(ml, TASK, knobs, 0, 8820, ml.DTYPE_F32)
    assert np.array_equal(f32.astype(np.float32), f_ref.astype(np.float32))


def test_reference_vector_and_hash(ml, orc):
    """test_space.cpp:142-157 / 206-208 through the device path."""
    knobs = orc.default_knob_template()
    f, h, v = run_device(ml, TASK, knobs, 0, 8820, ml.DTYPE_F64)
    i = int(np.nonzero((v == [16, 32, 16, 8, 32]).all(1))[0][0])
    want = [0.66666666666666663, 0.83333333333333337, 0.40874628412503389, 0.75, 0.625, 0.75,
            0.66666666666666663, 0.10034333188799373, 0.5625, 0.5]
    assert np.allclose(f[i, :10], want, rtol=1e-14, atol=0)
    assert np.all(f[i, 10:] == 0.0)
    assert int(h[i]) == 0xc27c832e9cdb768d


@pytest.mark.parametrize("first,n", [(0, 1), (12345, 4096), (10_223_616 - 5000, 5000), (5_000_000, 100_000)])
def test_large_space_slices(ml, orc, first, n):
    knobs = big_space()
    f_ref, h_ref, v_ref = orc.encode_configs(TASK, knobs, first, n)
    f, h, v = run_device(ml, TASK, knobs, first, n, ml.DTYPE_F64)
    assert np.array_equal(v, v_ref) and np.array_equal(h, h_ref)
    assert np.max(np.abs(f - f_ref)) <= 2e-15


def test_packed_model_rows_bf16(ml, orc):
    """bf16 rows with the packed layout's constant column (ld > D)."""
    knobs = orc.default_knob_template()
    f_ref, _, _ = orc.encode_configs(TASK, knobs, 100, 300)
    f, _, _ = run_device(ml, TASK, knobs, 100, 300, ml.DTYPE_BF16, D=16, ld=24)
    import torch

    want = torch.from_numpy(f_ref).to(torch.bfloat16).double().numpy()
    assert np.array_equal(f[:, :16], want)
    assert np.all(f[:, 16] == 1.0)


def test_errors(ml):
    knobs = [("tile_x", [1, 2]), ("tile_y", [4])]
    with pytest.raises(ml.MosesError) as e:
        ml.encode_configs_device(TASK, knobs, 1, 2)  # range beyond the 2-config space
    assert e.value.code == "shape-mismatch"
    with pytest.raises(ml.MosesError) as e:
        ml.encode_configs_device(TASK, [("tile_x", [2, 1])], 0, 1)
    assert e.value.code == "invalid-task"  # unsorted domain


def test_score_whole_space_on_device(ml, orc):
    """Exhaustive scorer input path without host features: encode 8820 configs on the device ->
    predict (golden 16-512-512-1 model, TF32) -> scores vs the fp64 oracle on oracle features."""
    import torch

    knobs = orc.default_knob_template()
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 12345)
    dm = ml.DeviceModel(p, ml.PREC_TF32, 8832)
    ld = dm.packed_ld
    F = torch.zeros((8820, ld), dtype=torch.float32, device="cuda")
    ml.encode_configs_device(TASK, knobs, 0, 8820, ml.DTYPE_F32, ctypes.c_void_p(F.data_ptr()), ld, 16)
    S = torch.empty(8820, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ml._ck(ml.lib().moses_predict_device(dm.h, ctypes.c_void_p(F.data_ptr()), ml.DTYPE_F32, ld, 8820,
                                         ctypes.c_void_p(S.data_ptr())))
    torch.cuda.synchronize()
    f_ref, _, _ = orc.encode_configs(TASK, knobs, 0, 8820)
    ref, _ = orc.forward(dims, p.params, f_ref)
    got = S.cpu().double().numpy()
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-3


# ---------------------------------------------------------------- simulated hardware (oracle.cpp:33-105)
import json
import os

SIM = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "simulated_oracle.json")))


def test_golden_true_best_on_device(ml, orc):
    """The 16 frozen optima of proj/tests/golden/true_best_default.json (test_oracle.cpp:313-335):
    configuration bit-exact, latency within 1e-14 (device exp/log2 vs libm)."""
    tasks = {t["id"]: t for t in SIM["tasks"]["list"]}
    knobs = orc.default_knob_template()
    for e in SIM["true_best"]["entries"]:
        values, lat = ml.true_best(SIM["devices"][e["device_id"]], tasks[e["task_id"]], knobs)
        assert values == e["values"], e
        assert lat == pytest.approx(e["latency_ms"], rel=1e-14), e


@pytest.mark.parametrize("first,n", [(0, 8820)])
def test_measure_matches_oracle(ml, orc, first, n):
    import torch

    k = SIM["reference_measurement"]
    knobs = orc.default_knob_template()
    bufs = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(4)]
    lab = torch.zeros(n, dtype=torch.float32, device="cuda")
    ml.measure_configs_device(k["device"], k["task"]["id"], k["task"], knobs, k["seed"], first, n,
                              *(ctypes.c_void_p(b.data_ptr()) for b in bufs), ctypes.c_void_p(lab.data_ptr()))
    torch.cuda.synchronize()
    got = [b.cpu().numpy() for b in bufs]
    ref = orc.measure_configs(k["device"], k["task"]["id"], k["task"], knobs, k["seed"], first, n)
    for g, r in zip(got, ref):
        assert np.max(np.abs(g - r) / np.abs(r)) <= 1e-14
    assert np.array_equal(lab.cpu().numpy(), got[1].astype(np.float32))
    # the reference measurement KAT (test_oracle.cpp:142-156) through the device path
    i = 0
    for (name, dom), v in zip(knobs, k["config"]):
        i = i * len(dom) + dom.index(v)
    assert got[1][i] == pytest.approx(k["throughput_gflops"], rel=k["eps"])
    assert got[2][i] == pytest.approx(k["latency_ms"], rel=k["eps"])


def test_true_best_large_space_matches_oracle(ml, orc):
    """1.4M-configuration space (wider domains): device argmin == oracle argmin."""
    knobs = [("tile_x", [1 << i for i in range(12)]), ("tile_y", [1 << i for i in range(12)]),
             ("unroll", [0, 2, 4, 8, 16, 32, 64, 128, 256, 512]), ("vectorize", [1 << i for i in range(6)]),
             ("parallel", [1 << i for i in range(10)]), ("split", [1, 2, 3, 4])]
    dev = SIM["devices"]["embedded"]
    task = SIM["tasks"]["list"][3]
    v_ref, l_ref = orc.true_best(dev, task, knobs)
    v, l = ml.true_best(dev, task, knobs)
    assert v == v_ref and l == pytest.approx(l_ref, rel=1e-14)


def test_space_property_vs_oracle(ml, orc):
    """Random knob spaces (roles, domain sizes and values), task parameters and index ranges:
    enumeration values and hashes bit-exact, features within fp64 rounding, simulated measurements
    within 1e-14 (device libm), the noise-free optimum identical."""
    pytest.importorskip("hypothesis")
    from hypothesis import given, settings
    from hypothesis import strategies as st

    names = ["tile_x", "tile_y", "unroll", "vectorize", "parallel", "extra"]
    device = {"id": "dev", "peak_gflops": 5000.0, "parallel_units": 24.0, "vector_lanes": 8.0, "cache_bytes": 3e6,
              "measure_overhead_ms": 1.5, "noise_std": 0.07, "repeats": 2}

    @settings(max_examples=12, deadline=None)
    @given(st.lists(st.tuples(st.sampled_from(names),
                              st.lists(st.integers(1, 4096), min_size=1, max_size=9, unique=True)),
                    min_size=1, max_size=6),
           st.tuples(st.floats(0.01, 500.0), st.floats(1.0, 16.0), st.floats(0.0, 14.0), st.floats(0.0, 9.0)),
           st.integers(0, 2**32), st.integers(0, 10**6))
    def check(kn, task, seed, first_raw):
        knobs = [(n, sorted(d)) for n, d in kn]
        space = int(np.prod([len(d) for _, d in knobs]))
        first = first_raw % space
        n = min(space - first, 500)
        f_ref, h_ref, v_ref = orc.encode_configs(task, knobs, first, n)
        f, h, v = run_device(ml, task, knobs, first, n, ml.DTYPE_F64)
        assert np.array_equal(v, v_ref) and np.array_equal(h, h_ref)
        assert np.max(np.abs(f - f_ref)) <= 4e-15
        import torch

        out = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(4)]
        ml.measure_configs_device(device, "t", task, knobs, seed, first, n,
                                  *(ctypes.c_void_p(o.data_ptr()) for o in out))
        torch.cuda.synchronize()
        ref = orc.measure_configs(device, "t", task, knobs, seed, first, n)
        for got, want in zip(out, ref):
            g = got.cpu().numpy()
            # exp() of the large tile-term exponents these random (non-power-of-two) domains reach
            # amplifies the device-libm vs glibc ulp difference; the reference's own domains stay at 1e-14
            assert np.max(np.abs(g - want) / np.abs(want)) <= 2e-13
        if space <= 20000:
            assert ml.true_best(device, task, knobs)[0] == orc.true_best(device, task, knobs)[0]

    check()
