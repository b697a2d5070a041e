"""Graph-step time of the bench workload with the fused kernels toggled (chain fwd/dZ, grouped
wgrad+update). Per-step CUDA events, L2 flushed between steps like bench.py."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench as B
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
import os
for f in ("moses_debug_set_chain", "moses_debug_set_group", "moses_debug_set_cluster", "moses_debug_set_rank_fused"):
    getattr(L, f).argtypes = [C.c_int]
off = ml.synth_offsets(B.SEED_DATA, B.PROGRAMS, B.MAX_STMTS)
nb = B.PROGRAMS // B.BATCH
off = off[: nb * B.BATCH + 1]
n_rows = int(off[-1])
rows_pad = int((np.diff(off[::B.BATCH]).max() + 127) // 128 * 128)
params = ml.init_random(B.DIMS, B.SEED_MODEL, strict=False)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
CONFIGS = [tuple(int(c) for c in x) for x in os.environ.get("ABL", "111,101,011,001,110").split(",")]
for chain, group, rankf in CONFIGS:
    L.moses_debug_set_chain(chain)
    L.moses_debug_set_group(group)
    L.moses_debug_set_rank_fused(rankf)
    dm = ml.DeviceModel(params, ml.PREC_BF16, max_rows=rows_pad)
    ld = dm.packed_ld
    X = torch.empty((n_rows, ld), dtype=torch.bfloat16, device="cuda")
    Y = torch.empty(nb * B.BATCH, dtype=torch.float32, device="cuda")
    OFF = torch.from_numpy(off).cuda()
    assert L.moses_synth_features_device(B.SEED_DATA, 0, n_rows, B.DIMS[0], ml.DTYPE_BF16, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(B.SEED_DATA, 0, nb * B.BATCH, Y.data_ptr()) == 0
    torch.cuda.synchronize()
    L.moses_set_async(1)
    ml._ck(L.moses_train_graph_create_pooled(dm.h, X.data_ptr(), ld, Y.data_ptr(), OFF.data_ptr(), nb, B.BATCH,
                                             rows_pad, B.LR, B.MU, 1))
    sp = C.c_void_p()
    L.moses_model_stream(dm.h, C.byref(sp))
    st = torch.cuda.ExternalStream(sp.value)
    res = {}
    with torch.cuda.stream(st):
        for _ in range(20):
            ml._ck(L.moses_train_graph_launch(dm.h, 1))
        for mode in ("flush", "warm"):
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for k in range(steps):
                if mode == "flush":
                    flush.fill_(float(k))
                evs[k][0].record(st)
                ml._ck(L.moses_train_graph_launch(dm.h, 1))
                evs[k][1].record(st)
            torch.cuda.synchronize()
            t = sorted(a.elapsed_time(b) for a, b in evs)
            res[mode] = (sum(t) / steps * 1e3, t[len(t) // 2] * 1e3)
        # back-to-back graph launches, one event pair around all
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        ml._ck(L.moses_train_graph_launch(dm.h, steps))
        b.record(st)
        torch.cuda.synchronize()
        res["b2b"] = a.elapsed_time(b) / steps * 1e3
    print(f"chain={chain} group={group} rank_fused={rankf}: flushed mean {res['flush'][0]:.1f} us (median {res['flush'][1]:.1f}); "
          f"warm mean {res['warm'][0]:.1f} us (median {res['warm'][1]:.1f}); back-to-back {res['b2b']:.1f} us", flush=True)
    dm.close()
