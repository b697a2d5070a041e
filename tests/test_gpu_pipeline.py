"""Device side of the training-data pipeline: generate_dataset on the device
(data.cpp:49-65), encode_features over device rows of knob values (space.cpp:69-81,140-159) and one
pretrain epoch over a ranking-batch plan (tuner.cpp:140-155) against the oracle's restatements.

Bars: configurations and knob values bit-exact (integer draws); measured throughput / latency /
wall cost within 1e-14 relative (device libm vs glibc); feature rows within fp64 rounding; the plan epoch bitwise
equal to the same batches stepped one by one through moses_train_step_device (bf16), and within
1e-5 of the fp64 oracle's pretrain epoch on an FP32 (3xTF32) handle."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOY_DEVICE = {"id": "toy", "peak_gflops": 1000.0, "parallel_units": 16.0, "vector_lanes": 8.0,
              "cache_bytes": 1e6, "measure_overhead_ms": 1.0, "noise_std": 0.05, "repeats": 3}
TASKS = [("a", (1.0, 4.0, 6.0, 3.0)), ("b", (1.0, 4.0, 9.0, 3.0)), ("conv2d_big", (300.0, 2.0, 10.0, 4.0))]


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0, moseslab.lib().moses_last_error()
    return moseslab


def vp(t):
    return ctypes.c_void_p(t.data_ptr())


def gen_device(ml, tid, task, knobs, n, seed, dtype=None, ld=16, D=16):
    import torch

    dtype = ml.DTYPE_F64 if dtype is None else dtype
    tdt = {ml.DTYPE_F64: torch.float64, ml.DTYPE_F32: torch.float32, ml.DTYPE_BF16: torch.bfloat16}[dtype]
    F = torch.full((n, ld), -7.0, dtype=tdt, device="cuda")
    V = torch.zeros((n, len(knobs)), dtype=torch.int64, device="cuda")
    thr, lat, wall = (torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(3))
    lab = torch.zeros(n, dtype=torch.float32, device="cuda")
    ml.generate_dataset_device(TOY_DEVICE, tid, task, knobs, n, seed, dtype, vp(F), ld, D, vp(V), vp(thr), vp(lat),
                               vp(wall), vp(lab))
    torch.cuda.synchronize()
    return F, V, thr, lat, wall, lab


def test_generate_dataset_matches_oracle(ml, orc):
    knobs = orc.default_knob_template()
    recs = orc.generate_dataset(TOY_DEVICE, TASKS, knobs, 300, 7)
    for t, (tid, task) in enumerate(TASKS):
        F, V, thr, lat, wall, lab = gen_device(ml, tid, task, knobs, 300, 7)
        want = recs[t * 300:(t + 1) * 300]
        assert V.cpu().numpy().tolist() == [r["values"] for r in want]
        # measure(): the device's exp / log / sqrt / cos vs glibc differ in the last bits (as in
        # test_gpu_space.py); everything upstream of them (configs, hashes, noise keys) is exact
        for got, key in ((thr, "throughput_gflops"), (lat, "latency_ms"), (wall, "wall_cost_ms")):
            r = np.array([x[key] for x in want])
            assert np.max(np.abs(got.cpu().numpy() - r) / np.abs(r)) <= 1e-14, key
        assert np.array_equal(lab.cpu().numpy(), thr.cpu().numpy().astype(np.float32))
        f_ref = np.stack([r["features"] for r in want])
        assert np.max(np.abs(F.cpu().numpy() - f_ref)) <= 1e-15


def test_generate_dataset_wide_space_and_serial_walk(ml, orc):
    """6 knobs (10.2M configurations), 50k samples: draws equal the oracle's; the exact sequential
    walk (taken when a below() call would reject) reproduces the parallel draws."""
    knobs = [("tile_x", [1 << i for i in range(16)]), ("tile_y", [1 << i for i in range(16)]),
             ("unroll", [0, 1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 128, 256, 512]),
             ("vectorize", [1 << i for i in range(8)]), ("parallel", [1 << i for i in range(13)]),
             ("split", list(range(1, 25)))]
    n = 50_000
    _, V, thr, _, _, _ = gen_device(ml, "wide", TASKS[2][1], knobs, n, 99)
    idx = orc.sample_config_indices(99, "wide", knobs, n)
    sizes = [len(d) for _, d in knobs]
    want = np.zeros((n, len(knobs)), dtype=np.int64)
    for i, x in enumerate(idx):
        for k in range(len(knobs) - 1, -1, -1):
            want[i, k] = knobs[k][1][x % sizes[k]]
            x //= sizes[k]
    assert np.array_equal(V.cpu().numpy(), want)
    ml.lib().moses_debug_force_serial_sampling(1)
    try:
        _, V2, thr2, _, _, _ = gen_device(ml, "wide", TASKS[2][1], knobs, 4000, 99)
    finally:
        ml.lib().moses_debug_force_serial_sampling(0)
    assert np.array_equal(V2.cpu().numpy(), want[:4000])
    assert np.array_equal(thr2.cpu().numpy(), thr.cpu().numpy()[:4000])


def test_generate_dataset_validation(ml, orc):
    knobs = orc.default_knob_template()
    with pytest.raises(ml.MosesError) as e:
        gen_device(ml, "a", TASKS[0][1], knobs, 0, 1)
    assert e.value.code == "invalid-config"
    with pytest.raises(ml.MosesError) as e:
        gen_device(ml, "a", TASKS[0][1], [("tile_x", [4, 2])], 5, 1)
    assert e.value.code == "invalid-task"


def test_encode_values_device(ml, orc):
    import torch

    knobs = orc.default_knob_template()
    F, V, *_ = gen_device(ml, "b", TASKS[1][1], knobs, 5000, 3, ml.DTYPE_F32)
    G = torch.full_like(F, -1.0)
    ml.encode_values_device(TASKS[1][1], knobs, vp(V), 5000, ml.DTYPE_F32, vp(G), 16, 16)
    torch.cuda.synchronize()
    assert torch.equal(F, G)
    V[37, 2] = 17  # not in the unroll domain
    V[4000, 0] = 3
    with pytest.raises(ml.MosesError) as e:
        ml.encode_values_device(TASKS[1][1], knobs, vp(V), 5000, ml.DTYPE_F32, vp(G), 16, 16)
    assert e.value.code == "invalid-config" and "record 37" in str(e.value)


def _dataset(ml, orc, dm, per_task, seed, dtype):
    """Device-resident packed dataset (rows of stride packed_ld with the constant column) over TASKS."""
    import torch

    knobs = orc.default_knob_template()
    ld = dm.packed_ld
    tdt = torch.bfloat16 if dtype == ml.DTYPE_BF16 else torch.float32
    n = per_task * len(TASKS)
    X = torch.zeros((n, ld), dtype=tdt, device="cuda")
    Y = torch.zeros(n, dtype=torch.float32, device="cuda")
    esz = X.element_size()
    for t, (tid, task) in enumerate(TASKS):
        r0 = t * per_task
        ml.generate_dataset_device(TOY_DEVICE, tid, task, knobs, per_task, seed, dtype,
                                   ctypes.c_void_p(X.data_ptr() + r0 * ld * esz), ld, 16, None, None, None, None,
                                   ctypes.c_void_p(Y.data_ptr() + r0 * 4))
    torch.cuda.synchronize()
    task_of = [tid for tid, _ in TASKS for _ in range(per_task)]
    return X, Y, task_of


@pytest.mark.parametrize("per_task,batch", [(700, 64), (300, 512), (129, 8)])
def test_train_plan_matches_eager_steps(ml, orc, per_task, batch):
    import torch

    dims = [16, 512, 512, 1]  # pretrain's model (tuner.cpp:133)
    p = ml.init_random(dims, 11)
    a = ml.DeviceModel(p, ml.PREC_BF16, 512)
    b = ml.DeviceModel(p, ml.PREC_BF16, 512)
    X, Y, task_of = _dataset(ml, orc, a, per_task, 5, ml.DTYPE_BF16)
    ld = a.packed_ld
    L = ml.lib()
    for epoch in range(2):
        plan = ml.make_ranking_batches(task_of, [t for t, _ in TASKS], batch, ml.epoch_seed(1, epoch))
        mean = ml.train_plan_device(a, vp(X), ld, vp(Y), len(task_of), plan, 0.001, 0.9)
        losses = []
        for k in range(len(plan)):
            _, rows = plan.batch(k)
            ri = torch.as_tensor(rows, device="cuda")
            xb, yb = X[ri].contiguous(), Y[ri].contiguous()
            torch.cuda.synchronize()  # the handle's stream does not wait on torch's
            out = ctypes.c_double()
            ml._ck(L.moses_train_step_device(b.h, xb.data_ptr(), ld, yb.data_ptr(), len(rows), 0.001, 0.9,
                                             ctypes.byref(out)))
            losses.append(out.value)
        pa, pb = a.download(), b.download()
        assert np.array_equal(pa.params, pb.params) and np.array_equal(pa.momentum, pb.momentum), epoch
        acc = 0.0
        for x in losses:  # left to right, like the device accumulator (Python's sum() compensates)
            acc += x
        assert mean == acc / len(losses)


def test_train_plan_fp32_matches_oracle_epoch(ml, orc):
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 21)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 64)
    X, Y, task_of = _dataset(ml, orc, dm, 60, 9, ml.DTYPE_F32)
    plan_ids = [t for t, _ in TASKS]
    seed = orc.epoch_seed(4, 0)
    plan = ml.make_ranking_batches(task_of, plan_ids, 16, seed)
    batches, _ = orc.make_ranking_batches(task_of, 16, seed)
    mean = ml.train_plan_device(dm, vp(X), dm.packed_ld, vp(Y), len(task_of), plan, 0.01, 0.9)
    feats = X[:, :16].double().cpu().numpy()
    labels = Y.double().cpu().numpy()
    w, mom, mean_ref = orc.pretrain_epoch(dims, p.params.copy(), p.momentum.copy(), feats, labels, batches, 0.01, 0.9)
    got = dm.download()
    assert abs(mean - mean_ref) <= 1e-5 * max(1.0, abs(mean_ref))
    assert np.max(np.abs(got.params - w)) <= 1e-5 * max(1.0, np.max(np.abs(w)))
    assert np.max(np.abs(got.momentum - mom)) <= 1e-5 * max(1e-3, np.max(np.abs(mom)))


def test_train_plan_validation(ml, orc):
    import torch

    dims = [16, 512, 512, 1]
    dm = ml.DeviceModel(ml.init_random(dims, 1), ml.PREC_BF16, 64)
    ld = dm.packed_ld
    X = torch.zeros((10, ld), dtype=torch.bfloat16, device="cuda")
    Y = torch.ones(10, dtype=torch.float32, device="cuda")
    bad = ml.RankingPlan(np.array([0, 1, 12]), np.array([0, 3]), np.array([0]), ["a"], 0)
    with pytest.raises(ml.MosesError) as e:
        ml.train_plan_device(dm, vp(X), ld, vp(Y), 10, bad, 0.001)
    assert e.value.code == "shape-mismatch"
    single = ml.RankingPlan(np.array([0, 1, 2]), np.array([0, 2, 3]), np.array([0, 0]), ["a"], 0)
    with pytest.raises(ml.MosesError) as e:
        ml.train_plan_device(dm, vp(X), ld, vp(Y), 10, single, 0.001)
    assert e.value.code == "invalid-argument"
    big = ml.RankingPlan(np.arange(1000) % 10, np.array([0, 1000]), np.array([0]), ["a"], 0)
    with pytest.raises(ml.MosesError) as e:
        ml.train_plan_device(dm, vp(X), ld, vp(Y), 10, big, 0.001)
    assert e.value.code == "capacity"
    empty = ml.RankingPlan(np.zeros(0, dtype=np.int64), np.array([0]), np.zeros(0), ["a"], 0)
    assert ml.train_plan_device(dm, vp(X), ld, vp(Y), 10, empty, 0.001) == 0.0


def test_pretrain_device_equals_plan_epochs(ml, orc):
    """moses_pretrain_device (plans overlapped with device epochs) == explicit per-epoch plans through
    moses_train_plan_device, bit for bit, with the same per-epoch losses and PretrainLog drop count."""
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 3)
    a = ml.DeviceModel(p, ml.PREC_BF16, 512)
    b = ml.DeviceModel(p, ml.PREC_BF16, 512)
    X, Y, task_of = _dataset(ml, orc, a, 1025, 2, ml.DTYPE_BF16)  # 1025 = 2 x 512 + a singleton per task
    ids = [t for t, _ in TASKS]
    losses, dropped = ml.pretrain_device(a, vp(X), a.packed_ld, vp(Y), task_of, ids, 512, 17, 4, 0.001, 0.9)
    assert dropped == len(TASKS)
    for e in range(4):
        plan = ml.make_ranking_batches(task_of, ids, 512, ml.epoch_seed(17, e))
        assert ml.train_plan_device(b, vp(X), b.packed_ld, vp(Y), len(task_of), plan, 0.001, 0.9) == losses[e]
    pa, pb = a.download(), b.download()
    assert np.array_equal(pa.params, pb.params) and np.array_equal(pa.momentum, pb.momentum)
    with pytest.raises(ml.MosesError) as e:
        ml.pretrain_device(a, vp(X), a.packed_ld, vp(Y), [], ids, 512, 17, 1)
    assert e.value.code == "empty-dataset"


def test_pretrain_device_fp32_matches_oracle(ml, orc):
    """Two epochs of the reference's pretrain loop on an FP32 handle vs the fp64 oracle (tuner.cpp:130-156)."""
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 5)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 64)
    X, Y, task_of = _dataset(ml, orc, dm, 50, 6, ml.DTYPE_F32)
    losses, _ = ml.pretrain_device(dm, vp(X), dm.packed_ld, vp(Y), task_of, [t for t, _ in TASKS], 16, 8, 2,
                                   0.01, 0.9)
    feats, labels = X[:, :16].double().cpu().numpy(), Y.double().cpu().numpy()
    w, mom = p.params.copy(), p.momentum.copy()
    for e in range(2):
        batches, _ = orc.make_ranking_batches(task_of, 16, orc.epoch_seed(8, e))
        w, mom, mean_ref = orc.pretrain_epoch(dims, w, mom, feats, labels, batches, 0.01, 0.9)
        assert abs(losses[e] - mean_ref) <= 1e-5 * max(1.0, abs(mean_ref))
    got = dm.download()
    assert np.max(np.abs(got.params - w)) <= 1e-5 * max(1.0, np.max(np.abs(w)))


@pytest.mark.parametrize("threads", [1, 3])
def test_pretrain_jobs_equal_sequential_runs(ml, orc, threads):
    """The native job pool (tuner.cpp:331-374 shape): every job's parameters and epoch losses equal
    its own sequential moses_pretrain_device run, bit for bit, whatever the worker count."""
    dims = [16, 512, 512, 1]
    seeds = [11, 12, 13, 14, 15]
    pool = [ml.DeviceModel(ml.init_random(dims, s), ml.PREC_BF16, 512) for s in seeds]
    X, Y, task_of = _dataset(ml, orc, pool[0], 600, 4, ml.DTYPE_BF16)
    ids = [t for t, _ in TASKS]
    ld = pool[0].packed_ld
    losses, dropped = ml.pretrain_jobs(pool, seeds, vp(X), ld, vp(Y), task_of, ids, 128, 3, 0.001, 0.9, threads)
    for j, s in enumerate(seeds):
        ref = ml.DeviceModel(ml.init_random(dims, s), ml.PREC_BF16, 512)
        l_ref, d_ref = ml.pretrain_device(ref, vp(X), ld, vp(Y), task_of, ids, 128, s, 3, 0.001, 0.9)
        assert losses[j].tolist() == l_ref and dropped[j] == d_ref
        a, b = pool[j].download(), ref.download()
        assert np.array_equal(a.params, b.params) and np.array_equal(a.momentum, b.momentum)


def test_pretrain_jobs_mapped_per_job_stores(ml, orc):
    """moses_pretrain_jobs_mapped (the f4 job grid across GPUs: job j over its own device's copy of the
    store): with two copies of the store on this device, every job equals its sequential run; a job whose
    store is on another device than its handle is refused (single-GPU box: checked only when >1 GPU)."""
    import torch

    dims = [16, 512, 512, 1]
    seeds = [21, 22, 23, 24]
    pool = [ml.DeviceModel(ml.init_random(dims, s), ml.PREC_BF16X3, 512) for s in seeds]
    X, Y, task_of = _dataset(ml, orc, pool[0], 400, 4, ml.DTYPE_F32)
    X2, Y2 = X.clone(), Y.clone()
    torch.cuda.synchronize()
    ids = [t for t, _ in TASKS]
    ld = pool[0].packed_ld
    xs = [vp(X), vp(X2), vp(X), vp(X2)]
    ys = [vp(Y), vp(Y2), vp(Y), vp(Y2)]
    losses, dropped = ml.pretrain_jobs_mapped(pool, seeds, xs, ld, ys, task_of, ids, 128, 2, 0.001, 0.9, 4)
    for j, s in enumerate(seeds):
        ref = ml.DeviceModel(ml.init_random(dims, s), ml.PREC_BF16X3, 512)
        l_ref, d_ref = ml.pretrain_device(ref, vp(X), ld, vp(Y), task_of, ids, 128, s, 2, 0.001, 0.9)
        assert losses[j].tolist() == l_ref and dropped[j] == d_ref
        assert np.array_equal(pool[j].download().params, ref.download().params)


def test_pretrain_from_records_matches_oracle(ml, orc):
    """moses_pretrain (host records -> device staging grouped by task -> encode -> epochs) on an FP32
    handle vs the fp64 oracle's pretrain over the same records (tuner.cpp:130-156): same batches,
    epoch losses and parameters within 1e-5."""
    knobs = orc.default_knob_template()
    recs = orc.generate_dataset(TOY_DEVICE, TASKS, knobs, 40, 3)
    order = [2, 0, 1]  # interleave tasks in the store: grouping must not change batch composition
    recs = [r for k in range(40) for t in order for r in [recs[t * 40 + k]]]
    ids = [t for t, _ in TASKS]
    rt = [ids.index(r["task_id"]) for r in recs]
    dims = [16, 512, 512, 1]
    p = ml.init_random(dims, 6)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 64)
    losses, dropped = ml.pretrain(dm, TASKS, knobs, rt, [r["values"] for r in recs],
                                  [r["throughput_gflops"] for r in recs], 16, 6, 2, 0.01, 0.9)
    feats = np.stack([r["features"] for r in recs]).astype(np.float32).astype(np.float64)
    labels = np.array([r["throughput_gflops"] for r in recs], dtype=np.float32).astype(np.float64)
    w, mom = p.params.copy(), p.momentum.copy()
    task_of = [r["task_id"] for r in recs]
    for e in range(2):
        batches, drop = orc.make_ranking_batches(task_of, 16, orc.epoch_seed(6, e))
        if e == 0:
            assert dropped == drop
        w, mom, mean_ref = orc.pretrain_epoch(dims, w, mom, feats, labels, batches, 0.01, 0.9)
        assert abs(losses[e] - mean_ref) <= 1e-5 * max(1.0, abs(mean_ref))
    got = dm.download()
    assert np.max(np.abs(got.params - w)) <= 1e-5 * max(1.0, np.max(np.abs(w)))
    bad = [list(r["values"]) for r in recs]
    bad[7][2] = 17
    with pytest.raises(ml.MosesError) as e:
        ml.pretrain(dm, TASKS, knobs, rt, bad, [r["throughput_gflops"] for r in recs], 16, 6, 1)
    assert e.value.code == "invalid-config" and "record 7" in str(e.value)


def test_generate_dataset_property(ml, orc):
    """Random seeds, task ids (any UTF-8) and sample counts: the device's keyed draws equal the
    oracle's sample_config walk value for value."""
    pytest.importorskip("hypothesis")
    from hypothesis import given, settings
    from hypothesis import strategies as st

    knobs = orc.default_knob_template()
    ids = st.text(alphabet=st.characters(blacklist_categories=("Cs",), blacklist_characters="\x00"), max_size=10)

    @settings(max_examples=15, deadline=None)
    @given(st.integers(0, 2**64 - 1), ids, st.integers(1, 300))
    def check(seed, tid, n):
        _, V, *_ = gen_device(ml, tid, TASKS[0][1], knobs, n, seed)
        idx = orc.sample_config_indices(seed, tid, knobs, n)
        sizes = [len(d) for _, d in knobs]
        want = []
        for x in idx:
            row = [0] * len(knobs)
            for k in range(len(knobs) - 1, -1, -1):
                row[k] = knobs[k][1][x % sizes[k]]
                x //= sizes[k]
            want.append(row)
        assert V.cpu().numpy().tolist() == want

    check()
