"""World-size-2 gloo tests of the multi-GPU host logic (CPU): sharded top-k merge and
gradient averaging give the single-device answers."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, q):
    import torch
    import torch.distributed as dist

    from paper_2201_05752_b200.distributed import gather_merge_topk, local_topk_host, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(123)
    pool = np.round(rng.normal(0, 1, n), 2).astype(np.float32)  # heavy ties across shards
    lo, hi = shard_range(n, rank, world)
    li = local_topk_host(pool[lo:hi], k)
    merged = gather_merge_topk(pool[lo:hi][li], li + lo, k)
    # data-parallel (throughput mode) gradient average: each rank's oracle gradient of its own batch,
    # averaged by the library helper
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle as orc

    from paper_2201_05752_b200.distributed import allreduce_gradients_

    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 7)
    xr = np.random.default_rng(10 + rank).random((9, 4))
    yr = 0.1 + np.random.default_rng(20 + rank).random(9)
    g_local, _ = orc.gradients(dims, w, xr, yr)
    g = torch.from_numpy(g_local.copy())
    allreduce_gradients_(g)
    q.put((rank, merged.tolist(), g.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,k", [(1001, 17), (50, 40), (7, 10)])
def test_sharded_topk_merge_equals_single_device(n, k):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    pool = np.round(np.random.default_rng(123).normal(0, 1, n), 2).astype(np.float32)
    want = orc.topk(pool, k)  # single-device reference order (score desc, index asc)
    dims = [4, 8, 8, 1]
    w = orc.init_random(dims, 7)
    g_mean = np.mean([orc.gradients(dims, w, np.random.default_rng(10 + r).random((9, 4)),
                                    0.1 + np.random.default_rng(20 + r).random(9))[0] for r in range(2)], axis=0)
    for rank, merged, g in res:
        assert merged == list(want)
        assert np.allclose(g, g_mean, rtol=0, atol=1e-15)


def test_shard_range_covers_everything():
    from paper_2201_05752_b200.distributed import shard_range

    for n in (0, 1, 7, 1000, 10_000_001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _exact_worker(rank, world, port, q):
    """SURVEY.md §8(e) exact-batch data parallelism over real collectives (gloo): every rank forwards its
    rows of the global batch, all-gathers scores and labels, takes the pair terms of its own rows
    against the whole batch, all-reduces (loss, pairs), normalises, backprops its rows; the all-reduced
    shares are the gradient of the concatenated batch. The same phases run on the GPU around NCCL
    (moses_dp_train_step mode 2 / moses_dp_exact_*)."""
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle as orc

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dims = [12, 32, 32, 1]
    w = orc.init_random(dims, 5, strict=False)
    n_local = 24
    x = np.random.default_rng(100 + rank).random((n_local, 12))
    y = np.round(0.1 + np.random.default_rng(200 + rank).random(n_local), 1)  # label ties across ranks
    s_local, _ = orc.forward(dims, w, x)
    s_all = [torch.zeros(n_local, dtype=torch.float64) for _ in range(world)]
    y_all = [torch.zeros(n_local, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(s_all, torch.from_numpy(s_local))
    dist.all_gather(y_all, torch.from_numpy(y))
    s_g, y_g = torch.cat(s_all).numpy(), torch.cat(y_all).numpy()
    p0 = rank * n_local
    gs, loss, pairs = orc.pair_terms_rows(s_g, y_g, p0, p0 + n_local)
    tot = torch.tensor([loss, float(pairs)], dtype=torch.float64)
    dist.all_reduce(tot)
    share = orc.gradients_from_score_grads(dims, w, x, gs / tot[1].item())
    g = torch.from_numpy(share)
    dist.all_reduce(g)
    q.put((rank, g.numpy().tolist(), float(tot[0] / tot[1])))
    dist.barrier()
    dist.destroy_process_group()


def test_exact_batch_dp_equals_single_device_gradient():
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle as orc

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exact_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    dims = [12, 32, 32, 1]
    w = orc.init_random(dims, 5, strict=False)
    x = np.concatenate([np.random.default_rng(100 + r).random((24, 12)) for r in range(world)])
    y = np.concatenate([np.round(0.1 + np.random.default_rng(200 + r).random(24), 1) for r in range(world)])
    g_full, loss_full = orc.gradients(dims, w, x, y)
    for rank, g, loss in res:
        g = np.asarray(g)
        assert np.max(np.abs(g - g_full)) <= 1e-13 * np.max(np.abs(g_full))  # summation order only
        assert abs(loss - loss_full) <= 1e-13 * abs(loss_full)
