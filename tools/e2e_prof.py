"""Timeline of the pipelined host-input training step (bench e2e leg): copies vs kernels."""
import ctypes as C
import sys
import os
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench as B
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
off = ml.synth_offsets(B.SEED_DATA, 4 * B.BATCH, B.MAX_STMTS)
params = ml.init_random(B.DIMS, B.SEED_MODEL, strict=False)
dm = ml.DeviceModel(params, getattr(ml, "PREC_" + os.environ.get("PREC", "BF16X3")), max_rows=2560)
batches = []
rng = np.random.default_rng(0)
for b in range(4):
    lo, hi = int(off[b * B.BATCH]), int(off[(b + 1) * B.BATCH])
    batches.append((torch.from_numpy(rng.random((hi - lo, 164))).pin_memory(),
                    torch.from_numpy(np.ascontiguousarray(off[b * B.BATCH:(b + 1) * B.BATCH + 1] - lo)).pin_memory(),
                    torch.from_numpy(0.1 + rng.random(B.BATCH)).pin_memory()))
losses = torch.zeros(4096, dtype=torch.float64).pin_memory()


import os

WANT_LOSS = os.environ.get("LOSS", "1") == "1"


def step(k):
    x, o, y = batches[k % 4]
    ml._ck(L.moses_train_step_pooled_async(dm.h, x.data_ptr(), x.shape[0], 164, o.data_ptr(), B.BATCH, y.data_ptr(),
                                           B.LR, B.MU, losses[k:k + 1].data_ptr() if WANT_LOSS else None))


for k in range(10):
    step(k)
ml._ck(L.moses_model_synchronize(dm.h))
t0 = time.perf_counter()
for k in range(200):
    step(k)
ml._ck(L.moses_model_synchronize(dm.h))
dt = (time.perf_counter() - t0) / 200
print(f"e2e {dt * 1e6:.1f} us/step -> {B.BATCH / dt / 1e6:.2f} M samples/s")
t0 = time.perf_counter()
for k in range(200):
    step(k)
host_us = (time.perf_counter() - t0) / 200 * 1e6
ml._ck(L.moses_model_synchronize(dm.h))
print(f"host enqueue (no sync inside) {host_us:.1f} us/step")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(6):
        step(k)
    ml._ck(L.moses_model_synchronize(dm.h))
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs[-40:]:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.elapsed_us():8.1f}  {e.name[:60]}")

# per-call host cost of the API (GPU kept busy so the host is never throttled by slot reuse)
ts = []
for k in range(300):
    t0 = time.perf_counter()
    step(k)
    ts.append(time.perf_counter() - t0)
ml._ck(L.moses_model_synchronize(dm.h))
ts = np.array(ts[50:]) * 1e6
print(f"per-call host time: median {np.median(ts):.1f} us, p10 {np.percentile(ts, 10):.1f}, p90 {np.percentile(ts, 90):.1f}")
