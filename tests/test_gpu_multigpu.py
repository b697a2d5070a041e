"""Library-level multi-GPU paths (csrc/comm.cu + capi.cu) on the one GPU this build can reach:
NCCL communicators at world size 1 (the collectives run; averages and sums of one rank are identities),
and the exact-batch data-parallel phases with two virtual ranks on one device (two handles, the
all-gather / all-reduce done by the test), which must reproduce the gradient of the concatenated batch.
The multi-rank host logic runs over real gloo collectives in test_distributed_gloo.py."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = [164, 512, 512, 1]


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0, moseslab.lib().moses_last_error()
    return moseslab


@pytest.fixture(scope="module")
def comm1(ml):
    import torch

    from paper_2201_05752_b200.distributed import Comm

    torch.cuda.init()
    c = Comm.init_all([torch.cuda.current_device()])[0]
    yield c
    c.close()


def nrel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _rows(ml, n, seed, ld):
    import torch

    L = ml.lib()
    X = torch.empty((n, ld), dtype=torch.float32, device="cuda")
    Y = torch.empty(n, dtype=torch.float32, device="cuda")
    assert L.moses_synth_features_device(seed, 0, n, DIMS[0], ml.DTYPE_F32, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(seed, 0, n, Y.data_ptr()) == 0
    Y.copy_(torch.round(Y * 10) / 10)  # label ties, as single-task batches have
    torch.cuda.synchronize()
    return X, Y


def test_comm_info(ml, comm1):
    import torch

    assert comm1.info() == (1, 0, torch.cuda.current_device())


@pytest.mark.parametrize("prec", ["BF16X3", "FP32"])
def test_exact_batch_two_virtual_ranks_equals_full_batch(ml, prec):
    """Exact-batch DP phases: ranks 0 and 1 (two handles on this GPU) each forward 256 rows of a
    512-row batch into their slots, the test plays the all-gather, each takes the pair terms of its rows,
    the test sums the (loss, pairs) partials and the gradient shares. == the full-batch gradient of one
    handle up to summation order (the forward is row-wise and the per-row pair terms are the same sums)."""
    import torch

    L = ml.lib()
    p = ml.init_random(DIMS, 7)
    P = getattr(ml, "PREC_" + prec)
    full = ml.DeviceModel(p, P, 512)
    ld = full.packed_ld
    X, Y = _rows(ml, 512, 3, ld)
    loss_full = C.c_double()
    ml._ck(L.moses_gradients_device(full.h, X.data_ptr(), ld, Y.data_ptr(), 512, C.byref(loss_full)))
    g_full = full.gradients()
    ranks = [ml.DeviceModel(p, P, 256) for _ in range(2)]
    S = torch.zeros(512, dtype=torch.float32, device="cuda")
    YG = torch.zeros(512, dtype=torch.float32, device="cuda")
    for r, dm in enumerate(ranks):
        ml._ck(L.moses_dp_exact_forward(dm.h, X[256 * r:].data_ptr(), ld, Y[256 * r:].data_ptr(), 256,
                                        S[256 * r:].data_ptr(), YG[256 * r:].data_ptr()))
        ml._ck(L.moses_model_synchronize(dm.h))
    tots = [torch.zeros(2, dtype=torch.float64, device="cuda") for _ in ranks]
    for r, dm in enumerate(ranks):
        ml._ck(L.moses_dp_exact_rank(dm.h, S.data_ptr(), YG.data_ptr(), 512, 256 * r, tots[r].data_ptr()))
        ml._ck(L.moses_model_synchronize(dm.h))
    tot = tots[0] + tots[1]
    losses = []
    for dm in ranks:
        lo = C.c_double()
        ml._ck(L.moses_dp_exact_backward(dm.h, 512, tot.data_ptr(), C.byref(lo)))
        losses.append(lo.value)
    g = ranks[0].gradients() + ranks[1].gradients()
    assert losses[0] == losses[1]
    assert abs(losses[0] - loss_full.value) <= 1e-6 * abs(loss_full.value)
    assert nrel(g, g_full) < 1e-5


def test_world1_average_step_equals_local_step(ml, comm1):
    """Throughput-mode DP over a 1-rank NCCL communicator == the local training step, bit for bit
    (the average of one rank is the identity; the update has the fused step's arithmetic)."""
    import torch

    from paper_2201_05752_b200.distributed import DP_AVERAGE, set_data_parallel

    L = ml.lib()
    p = ml.init_random(DIMS, 9)
    a = ml.DeviceModel(p, ml.PREC_BF16X3, 512)
    b = ml.DeviceModel(p, ml.PREC_BF16X3, 512)
    ld = a.packed_ld
    X, Y = _rows(ml, 512, 4, ld)
    set_data_parallel(a, comm1, DP_AVERAGE)
    for _ in range(3):
        ml._ck(L.moses_dp_train_step(a.h, X.data_ptr(), ld, Y.data_ptr(), 512, 0.001, 0.9, None))
        ml._ck(L.moses_train_step_device(b.h, X.data_ptr(), ld, Y.data_ptr(), 512, 0.001, 0.9, None))
    pa, pb = a.download(), b.download()
    assert np.array_equal(pa.params, pb.params) and np.array_equal(pa.momentum, pb.momentum)
    torch.cuda.synchronize()


def test_world1_exact_step_and_graph(ml, comm1):
    """Exact-batch DP over a 1-rank communicator: the step (all-gather, pair terms of the own rows,
    all-reduces inside) == the local step within fp32 summation order; the captured graph == eager."""
    import torch

    from paper_2201_05752_b200.distributed import DP_EXACT, set_data_parallel

    L = ml.lib()
    p = ml.init_random(DIMS, 11)
    a = ml.DeviceModel(p, ml.PREC_BF16X3, 512)
    b = ml.DeviceModel(p, ml.PREC_BF16X3, 512)
    ld = a.packed_ld
    X, Y = _rows(ml, 3 * 512, 5, ld)
    set_data_parallel(a, comm1, DP_EXACT)
    la, lb = C.c_double(), C.c_double()
    for s in range(3):
        ml._ck(L.moses_dp_train_step(a.h, X[512 * s:].data_ptr(), ld, Y[512 * s:].data_ptr(), 512, 0.001, 0.9,
                                     C.byref(la)))
        ml._ck(L.moses_train_step_device(b.h, X[512 * s:].data_ptr(), ld, Y[512 * s:].data_ptr(), 512, 0.001, 0.9,
                                         C.byref(lb)))
        assert abs(la.value - lb.value) <= 1e-6 * abs(lb.value)
    pa, pb = a.download(), b.download()
    assert nrel(pa.params - p.params, pb.params - p.params) < 1e-4
    # graph replay of the exact step (gather + collectives + update captured) == the eager DP steps
    c = ml.DeviceModel(p, ml.PREC_BF16X3, 512)
    d = ml.DeviceModel(p, ml.PREC_BF16X3, 512)
    set_data_parallel(c, comm1, DP_EXACT)
    set_data_parallel(d, comm1, DP_EXACT)
    ml._ck(L.moses_train_graph_create(c.h, X.data_ptr(), ld, Y.data_ptr(), 3, 512, 0.001, 0.9, 1))
    ml._ck(L.moses_train_graph_launch(c.h, 3))
    for s in range(3):
        ml._ck(L.moses_dp_train_step(d.h, X[512 * s:].data_ptr(), ld, Y[512 * s:].data_ptr(), 512, 0.001, 0.9, None))
    ml._ck(L.moses_model_synchronize(c.h))
    assert np.array_equal(c.download().params, d.download().params)
    torch.cuda.synchronize()


def test_world1_pooled_graph_with_comm_equals_plain_graph(ml, comm1):
    """The cfg2 training graph with throughput-mode DP (all-reduce + update captured) at world size 1 ==
    the plain fused graph, bit for bit."""
    import torch

    from paper_2201_05752_b200.distributed import DP_AVERAGE, set_data_parallel

    L = ml.lib()
    dims = [164, 512, 512, 512, 512, 1]
    p = ml.init_random(dims, 12345, strict=False)
    B, nb = 256, 3
    off = ml.synth_offsets(2, B * nb, 8)
    rows_pad = (max(int(off[(b + 1) * B] - off[b * B]) for b in range(nb)) + 127) // 128 * 128
    a = ml.DeviceModel(p, ml.PREC_BF16X3, rows_pad)
    b = ml.DeviceModel(p, ml.PREC_BF16X3, rows_pad)
    ld = a.packed_ld
    X = torch.empty((int(off[-1]), ld), dtype=torch.float32, device="cuda")
    Y = torch.empty(B * nb, dtype=torch.float32, device="cuda")
    assert L.moses_synth_features_device(2, 0, int(off[-1]), 164, ml.DTYPE_F32, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(2, 0, B * nb, Y.data_ptr()) == 0
    OFF = torch.from_numpy(off).cuda()
    torch.cuda.synchronize()
    set_data_parallel(a, comm1, DP_AVERAGE)
    for dm in (a, b):
        ml._ck(L.moses_train_graph_create_pooled(dm.h, X.data_ptr(), ld, Y.data_ptr(), OFF.data_ptr(), nb, B,
                                                 rows_pad, 0.001, 0.9, 1))
        ml._ck(L.moses_train_graph_launch(dm.h, 5))
        ml._ck(L.moses_model_synchronize(dm.h))
    assert np.array_equal(a.download().params, b.download().params)


def test_topk_sharded_world1_equals_device_topk(ml, comm1):
    import torch

    from paper_2201_05752_b200.distributed import topk_sharded

    L = ml.lib()
    n, k = 300_000, 1024
    s = torch.from_numpy(np.round(np.random.default_rng(0).normal(0, 1, n), 3).astype(np.float32)).cuda()
    torch.cuda.synchronize()
    got = topk_sharded(comm1, s.data_ptr(), n, 1000, k)
    want = (C.c_int64 * k)()
    ml._ck(L.moses_topk_device(s.data_ptr(), n, k, want))
    assert np.array_equal(got, np.frombuffer(want, dtype=np.int64) + 1000)
