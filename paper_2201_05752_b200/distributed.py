"""Multi-GPU plumbing for the two paths that shard.

* Candidate scoring (cfg4): programs are independent (predict is row-wise pure,
  model.cpp:169-175), so the pool is split into contiguous index ranges, one per
  rank; each rank scores and top-k's its shard on its own GPU; the k winners
  (score, global index) of every rank are all-gathered and merged with the
  reference comparator (score desc, then index asc — search.cpp:32-37). This is
  the only exchange (k * 12 bytes per rank).
* Training (cfg5): data parallel; the flat fp32 gradient buffer of the device
  handle is averaged across ranks between gradients and update.

The collectives of the data path live in the library (libmoses_gpu.so over NCCL, csrc/comm.cu):
`Comm` wraps a moses_comm_t, created per rank from an id distributed through torch.distributed
(`Comm.from_torch`) or for several GPUs of one process (`Comm.init_all`). torch.distributed is only the
rendezvous here, and the transport of the gloo CPU tests of the host logic.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of n items for `rank` (the first n % world ranks get one more)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def merge_topk(scores: np.ndarray, indices: np.ndarray, k: int) -> np.ndarray:
    """Exact merge of gathered candidates: order (score desc, global index asc), first k.

    Scores are compared as float32 (the device's score type), so the merge agrees
    bit-for-bit with a single-device top-k over the concatenated pool."""
    s = np.asarray(scores, dtype=np.float32)
    i = np.asarray(indices, dtype=np.int64)
    keep = i >= 0  # padding slots from ranks with fewer than k candidates
    s, i = s[keep], i[keep]
    order = np.lexsort((i, -s.astype(np.float64)))
    return i[order[:k]]


def local_topk_host(scores_f32: np.ndarray, k: int) -> np.ndarray:
    """Reference-order top-k of one shard (numpy; the device path uses moses_topk_device)."""
    s = np.asarray(scores_f32, dtype=np.float32)
    order = np.lexsort((np.arange(len(s)), -s.astype(np.float64)))
    return order[: min(k, len(s))]


def gather_merge_topk(local_scores: np.ndarray, local_global_idx: np.ndarray, k: int, group=None) -> np.ndarray:
    """All-gather each rank's (score, global index) winners and merge them identically on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    s = np.full(k, -np.inf, dtype=np.float32)
    i = np.full(k, -1, dtype=np.int64)
    m = min(k, len(local_scores))
    s[:m] = np.asarray(local_scores, dtype=np.float32)[:m]
    i[:m] = np.asarray(local_global_idx, dtype=np.int64)[:m]
    ts, ti = torch.from_numpy(s).to(dev), torch.from_numpy(i).to(dev)
    gs = [torch.empty_like(ts) for _ in range(world)]
    gi = [torch.empty_like(ti) for _ in range(world)]
    dist.all_gather(gs, ts, group=group)
    dist.all_gather(gi, ti, group=group)
    return merge_topk(torch.cat(gs).cpu().numpy(), torch.cat(gi).cpu().numpy(), k)


def sharded_score_topk(model, x_dev_shard, ld: int, row0: int, n_local: int, k: int, dtype: int, group=None):
    """One rank's part of cfg4: score the local shard on device, local top-k, gather + merge.

    `model` is a moseslab.DeviceModel, `x_dev_shard` a device pointer to the shard's packed rows."""
    import ctypes as C

    import torch

    from . import moseslab as ml

    L = ml.lib()
    scores = torch.empty(n_local, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()  # the shard rows were written on torch's stream
    ml._ck(L.moses_predict_device(model.h, x_dev_shard, dtype, ld, n_local, scores.data_ptr()))
    # predict only queues work on the handle's stream; top-k reads the scores on another stream
    ml._ck(L.moses_model_synchronize(model.h))
    kk = min(k, n_local)
    idx = (C.c_int64 * max(kk, 1))()
    ml._ck(L.moses_topk_device(scores.data_ptr(), n_local, kk, idx))
    local_idx = np.frombuffer(idx, dtype=np.int64)[:kk].copy()
    # only the k winning scores leave the device
    local_scores = scores[torch.from_numpy(local_idx).to(scores.device)].cpu().numpy()
    return gather_merge_topk(local_scores, local_idx + row0, k, group)


def allreduce_gradients_(grad_tensor, group=None):
    """Average the device gradient buffer across data-parallel ranks (in place)."""
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        dist.all_reduce(grad_tensor, op=dist.ReduceOp.AVG, group=group)
    else:  # gloo has no AVG
        dist.all_reduce(grad_tensor, op=dist.ReduceOp.SUM, group=group)
        grad_tensor.div_(dist.get_world_size(group))
    return grad_tensor


def device_gradient_tensor(model):
    """Zero-copy torch view of a DeviceModel's fp32 gradient buffer (for NCCL)."""
    import ctypes as C

    import torch

    from . import moseslab as ml

    g = C.POINTER(C.c_float)()
    ml._ck(ml.lib().moses_model_device_ptrs(model.h, None, C.byref(g), None))

    class _CAI:
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}

    return torch.as_tensor(_CAI(C.cast(g, C.c_void_p).value, model.P), device="cuda")


class Comm:
    """A library NCCL communicator (moses_comm_t)."""

    ID_BYTES = 128

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def from_torch(cls, group=None):
        """One communicator per rank of a torch.distributed group, on the current CUDA device: rank 0 makes
        the NCCL id, torch.distributed broadcasts it, every rank calls moses_comm_init_rank."""
        import ctypes as C

        import torch.distributed as dist

        from . import moseslab as ml

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = (C.c_uint8 * cls.ID_BYTES)()
        if rank == 0:
            ml._ck(ml.lib().moses_comm_unique_id(buf, cls.ID_BYTES))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        idb = (C.c_uint8 * cls.ID_BYTES).from_buffer_copy(obj[0])
        h = C.c_void_p()
        ml._ck(ml.lib().moses_comm_init_rank(idb, world, rank, C.byref(h)))
        return cls(h)

    @classmethod
    def init_all(cls, devices):
        """ncclCommInitAll: one communicator per listed device, driven from this process."""
        import ctypes as C

        from . import moseslab as ml

        n = len(devices)
        devs = (C.c_int32 * n)(*devices)
        hs = (C.c_void_p * n)()
        ml._ck(ml.lib().moses_comm_init_all(n, devs, hs))
        return [cls(C.c_void_p(hs[i])) for i in range(n)]

    def info(self):
        import ctypes as C

        from . import moseslab as ml

        n, r, d = C.c_int32(), C.c_int32(), C.c_int32()
        ml._ck(ml.lib().moses_comm_info(self.h, C.byref(n), C.byref(r), C.byref(d)))
        return n.value, r.value, d.value

    def close(self):
        from . import moseslab as ml

        if getattr(self, "h", None):
            ml.lib().moses_comm_destroy(self.h)
            self.h = None


DP_NONE, DP_AVERAGE, DP_EXACT = 0, 1, 2


def set_data_parallel(model, comm, mode):
    """moses_model_set_comm: DP_AVERAGE (each rank its own batch, averaged gradients) or DP_EXACT (one global
    batch, the rank-ordered concatenation of the ranks' rows)."""
    from . import moseslab as ml

    ml._ck(ml.lib().moses_model_set_comm(model.h, comm.h if comm is not None else None, mode))


def topk_sharded(comm, scores_dev_ptr, n_local: int, row0: int, k: int) -> np.ndarray:
    """moses_topk_sharded: the global top-k of a pool sharded by contiguous ranges (same on every rank)."""
    import ctypes as C

    from . import moseslab as ml

    out = (C.c_int64 * k)()
    ml._ck(ml.lib().moses_topk_sharded(comm.h, scores_dev_ptr, n_local, row0, k, out))
    return np.frombuffer(out, dtype=np.int64).copy()
