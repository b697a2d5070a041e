"""Kernel timeline (torch profiler / CUPTI) of the bench training step (pooled CUDA graph),
with and without the 256 MiB L2 flush between steps."""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench as B
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
PREC = getattr(ml, "PREC_" + os.environ.get("PREC", "BF16X3"))
CFG = os.environ.get("CFG", "2")
DT = ml.input_dtype(PREC)
if CFG == "5":  # cfg5: {164,512,512,1}, 4096 single-statement programs per step (bench_cfg5)
    dims, batch, nb = [164, 512, 512, 1], 4096, 64
    dm = ml.DeviceModel(ml.init_random(dims, B.SEED_MODEL), PREC, max_rows=batch)
    ld = dm.packed_ld
    X = torch.empty((nb * batch, ld), dtype=torch.bfloat16 if DT == ml.DTYPE_BF16 else torch.float32, device="cuda")
    Y = torch.empty(nb * batch, dtype=torch.float32, device="cuda")
    assert L.moses_synth_features_device(B.SEED_DATA + 5, 0, nb * batch, dims[0], DT, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(B.SEED_DATA + 5, 0, nb * batch, Y.data_ptr()) == 0
    torch.cuda.synchronize()
    L.moses_set_async(1)
    ml._ck(L.moses_train_graph_create(dm.h, X.data_ptr(), ld, Y.data_ptr(), nb, batch, B.LR, B.MU, 1))
else:
    off = ml.synth_offsets(B.SEED_DATA, B.PROGRAMS, B.MAX_STMTS)
    nb = B.PROGRAMS // B.BATCH
    off = off[: nb * B.BATCH + 1]
    n_rows = int(off[-1])
    rows_pad = int((np.diff(off[::B.BATCH]).max() + 127) // 128 * 128)
    params = ml.init_random(B.DIMS, B.SEED_MODEL, strict=False)
    dm = ml.DeviceModel(params, PREC, max_rows=rows_pad)
    ld = dm.packed_ld
    X = torch.empty((n_rows, ld), dtype=torch.bfloat16 if DT == ml.DTYPE_BF16 else torch.float32, device="cuda")
    Y = torch.empty(nb * B.BATCH, dtype=torch.float32, device="cuda")
    OFF = torch.from_numpy(off).cuda()
    assert L.moses_synth_features_device(B.SEED_DATA, 0, n_rows, B.DIMS[0], DT, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(B.SEED_DATA, 0, nb * B.BATCH, Y.data_ptr()) == 0
    torch.cuda.synchronize()
    L.moses_set_async(1)
    ml._ck(L.moses_train_graph_create_pooled(dm.h, X.data_ptr(), ld, Y.data_ptr(), OFF.data_ptr(), nb, B.BATCH,
                                             rows_pad, B.LR, B.MU, 1))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(20):
    ml._ck(L.moses_train_graph_launch(dm.h, 1))
torch.cuda.synchronize()
for do_flush in (False,):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for k in range(4):
            if do_flush:
                flush.fill_(float(k))
            ml._ck(L.moses_train_graph_launch(dm.h, 1))
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    # last step only
    # step period: between the ends of the last kernel of consecutive steps (the weight update)
    ends = sorted(e.time_range.end for e in evs if "wgrad" in e.name)
    last_ends, prev = [], None
    for t_end in ends:  # one update per step: the latest wgrad end within each step
        if prev is not None and t_end - prev > 40:
            last_ends.append(prev)
        prev = t_end
    if prev is not None:
        last_ends.append(prev)
    if len(last_ends) >= 2:
        per = [b - a for a, b in zip(last_ends, last_ends[1:])]
        print("step period (us):", " ".join(f"{p:.1f}" for p in per))
    starts = [i for i, e in enumerate(evs) if "gather" in e.name]
    # the last step: from the kernel after the previous step's update (the forward may start before the gather)
    lo = starts[-1] if starts else 0
    if len(last_ends) >= 2:
        lo = min(i for i, e in enumerate(evs) if e.time_range.start >= last_ends[-2] - 1)
    evs = evs[lo:]
    t0 = evs[0].time_range.start
    print(f"--- flush={do_flush}")
    for e in evs:
        if "FillFunctor" in e.name:
            continue
        print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.elapsed_us():7.1f}  {e.name[:70]}")
