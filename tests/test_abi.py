"""CPU-side checks of the drop-in boundary: the library builds, loads without a
GPU, exports every symbol include/moses_gpu.h declares, and its host-only
entry points (init, files, select_batch) match the oracle byte for byte."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import build as b

    b.build()
    from paper_2201_05752_b200 import moseslab

    moseslab.lib()
    return moseslab


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "moses_gpu.h")).read()
    return sorted(set(re.findall(r"MOSES_API\s+[\w\s\*]+?\b(moses_\w+)\s*\(", src)))


def test_header_symbols_exported(ml):
    syms = declared_symbols()
    assert len(syms) > 40
    lib = ml.lib()
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_no_device_is_reported_not_faked(ml):
    rc = ml.lib().moses_device_check()
    import torch

    if not torch.cuda.is_available():
        assert rc != 0  # no silent CPU path


def test_init_random_bit_exact(ml, orc):
    for dims, seed in (([16, 512, 512, 1], 12345), ([4, 8, 8, 1], 3), ([164, 256, 256, 1], 7)):
        p = ml.init_random(dims, seed)
        assert np.array_equal(p.params, orc.init_random(dims, seed))
    with pytest.raises(ml.MosesError) as e:
        ml.init_random([16, 512, 1], 0)
    assert e.value.code == "bad-dims"
    deep = ml.init_random([164, 512, 512, 512, 512, 1], 1, strict=False)
    assert len(deep.params) == 872961


def test_param_count(ml):
    assert ml.param_count([16, 512, 512, 1]) == 271873
    assert ml.param_count([164, 512, 512, 512, 512, 1]) == 872961


def test_serialize_roundtrip_and_failures(ml, orc):
    p = ml.init_random([16, 512, 512, 1], 60)
    p.momentum[3 * 512 + 5] = 0.25
    p.momentum[-1] = -1.5
    blob = ml.serialize(p)
    assert blob == orc.serialize(p.dims, p.params, p.momentum)
    q = ml.deserialize(blob)
    assert ml.serialize(q) == blob
    bad = bytearray(blob); bad[0] = ord("X")
    with pytest.raises(ml.MosesError) as e:
        ml.deserialize(bytes(bad))
    assert e.value.code == "corrupt-stream"
    bad = bytearray(blob); bad[4] = 9
    with pytest.raises(ml.MosesError) as e:
        ml.deserialize(bytes(bad))
    assert e.value.code == "version-mismatch"
    with pytest.raises(ml.MosesError) as e:
        ml.deserialize(blob[: len(blob) // 2])
    assert e.value.code == "corrupt-stream"
    with pytest.raises(ml.MosesError) as e:
        ml.deserialize(b"")
    assert e.value.code == "corrupt-stream"
    with pytest.raises(ml.MosesError) as e:
        ml.serialize(ml.init_random([16, 256, 256, 1], 0))
    assert e.value.code == "bad-dims"


def test_model_file_io(ml, tmp_path):
    p = ml.init_random([16, 512, 512, 1], 62)
    path = str(tmp_path / "m.bin")
    ml.save_model(p, path)
    assert ml.serialize(ml.load_model(path)) == ml.serialize(p)
    os.remove(path)
    with pytest.raises(ml.MosesError) as e:
        ml.load_model(path)
    assert e.value.code == "io-error"


def test_mask_file_roundtrip(ml, orc, tmp_path):
    rng = np.random.default_rng(40)
    mask = ml.ParamMask(rng.random(1001) < 0.3, 4, ml.THRESHOLD, 0.75)
    path = str(tmp_path / "k.bin")
    ml.write_mask(mask, path)
    blob = open(path, "rb").read()
    assert blob == orc.write_mask_bytes(mask.transferable, 4, orc.THRESHOLD, 0.75)
    back = ml.read_mask(path)
    assert back.phase == 4 and back.mode == ml.THRESHOLD and back.value == 0.75
    assert np.array_equal(back.transferable, mask.transferable)
    open(path, "wb").write(blob[: len(blob) // 2])
    with pytest.raises(ml.MosesError) as e:
        ml.read_mask(path)
    assert e.value.code == "corrupt-stream"
    os.remove(path)
    with pytest.raises(ml.MosesError) as e:
        ml.read_mask(path)
    assert e.value.code == "io-error"


def test_select_batch(ml, orc):
    # search_test.cpp:161-187 with hashes standing in for configs
    a, b, c = orc.fnv_u64s([8, 8, 0, 1, 1]), orc.fnv_u64s([16, 8, 0, 1, 1]), orc.fnv_u64s([32, 8, 0, 1, 1])
    pos = ml.select_batch([a, b, a, c], {b}, 10)
    assert list(pos) == [0, 3]
    hs = [orc.fnv_u64s([i]) for i in range(6)]
    assert list(ml.select_batch(hs, set(), 3)) == [0, 1, 2]
    one = orc.fnv_u64s([1])
    assert len(ml.select_batch([one], {one}, 5)) == 0
    with pytest.raises(ml.MosesError) as e:
        ml.select_batch([one], {one}, 0)
    assert e.value.code == "invalid-config"
