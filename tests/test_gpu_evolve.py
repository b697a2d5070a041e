"""evolve with the model scorer on the device: candidates encoded on the device
from their enumeration indices and scored by the model there. The GA logic itself is pinned
bit-exactly against the oracle in test_evolve.py (linear scorer); here: the scores are the model's
own device scores of the returned configurations (bitwise), the result is sorted, valid,
deterministic per seed and never loses its best candidate across generations."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TASK = (2.0, 8.0, 9.0, 5.0)


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0, moseslab.lib().moses_last_error()
    return moseslab


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
def test_evolve_model_scores(ml, orc, prec):
    import torch

    knobs = orc.default_knob_template()
    dims = [16, 512, 512, 1]
    dm = ml.DeviceModel(ml.init_random(dims, 4), ml.PREC_BF16 if prec == "bf16" else ml.PREC_TF32, 1024)
    vals, scores = ml.evolve(dm, TASK, knobs, seed=5)
    assert len(vals) == 32 * 5
    keys = [(-s, tuple(v)) for v, s in zip(vals.tolist(), scores.tolist())]
    assert keys == sorted(keys)
    for v in vals.tolist():
        assert all(x in d for x, (_, d) in zip(v, knobs))
    v2, s2 = ml.evolve(dm, TASK, knobs, seed=5)
    assert np.array_equal(vals, v2) and np.array_equal(scores, s2)
    # the scores are the model's device scores of these configurations (same encode + predict path)
    sizes = [len(d) for _, d in knobs]
    idx = []
    for v in vals.tolist():
        i = 0
        for k, x in enumerate(v):
            i = i * sizes[k] + knobs[k][1].index(x)
        idx.append(i)
    dt = ml.DTYPE_BF16 if prec == "bf16" else ml.DTYPE_F32
    ld = dm.packed_ld
    F = torch.zeros((len(idx), ld), dtype=torch.bfloat16 if prec == "bf16" else torch.float32, device="cuda")
    for r, i in enumerate(idx):
        ml.encode_configs_device(TASK, knobs, i, 1, dt, ctypes.c_void_p(F[r].data_ptr()), ld, dims[0])
    S = torch.zeros(len(idx), dtype=torch.float32, device="cuda")
    ml._ck(ml.lib().moses_predict_device(dm.h, ctypes.c_void_p(F.data_ptr()), dt, ld, len(idx),
                                         ctypes.c_void_p(S.data_ptr())))
    torch.cuda.synchronize()
    assert np.array_equal(S.cpu().numpy().astype(np.float64), scores)
    # elitism: the best never gets worse with more generations
    best = [ml.evolve(dm, TASK, knobs, generations=g, seed=8)[1][0] for g in range(5)]
    assert all(b1 >= b0 for b0, b1 in zip(best, best[1:]))
