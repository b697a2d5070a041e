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
