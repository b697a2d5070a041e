"""The resident (single cooperative launch) lottery step at the cost model's own size (cfg2 dims,
P = 872,961): device time per step (CUDA events) and CTA 0's phase stamps, ratio and threshold modes."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
dims = [164, 512, 512, 512, 512, 1]
p = ml.init_random(dims, 7, strict=False)
dm = ml.DeviceModel(p, ml.PREC_BF16X3, max_rows=512)
rng = np.random.default_rng(1)
x, y = rng.random((512, dims[0])), 0.1 + rng.random(512)
ml.gradients(dm, ml.RankingBatch(x, y))  # a real gradient in the handle
sp = C.c_void_p()
L.moses_model_stream(dm.h, C.byref(sp))
st = torch.cuda.ExternalStream(sp.value)
pop = C.c_int64()
tr = (C.c_uint64 * 8)()
for mode, name in ((2, "ratio 0.5"), (1, "threshold 0.5")):
    L.moses_set_async(1)
    for _ in range(5):
        ml._ck(L.moses_lottery_step(dm.h, mode, 0.5, 0, 1e-9, 1.0, None, 0, C.byref(pop)))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    a.record(st)
    for _ in range(reps):
        ml._ck(L.moses_lottery_step(dm.h, mode, 0.5, 0, 1e-9, 1.0, None, 0, C.byref(pop)))
    b.record(st)
    torch.cuda.synchronize()
    L.moses_set_async(0)
    ml._ck(L.moses_debug_lottery_trace(tr))
    d = [(tr[i + 1] - tr[i]) / 1e3 for i in range(5)]
    print(f"{name}: {1e3 * a.elapsed_time(b) / reps:.1f} us per step (device, back to back); CTA 0 phases (us): "
          f"loads+level1 {d[0]:.1f}, level2 {d[1]:.1f}, level3 {d[2]:.1f}, ties {d[3]:.1f}, apply {d[4]:.1f}")

from torch.profiler import ProfilerActivity, profile  # noqa: E402

for mode, name in ((2, "ratio 0.5"), (1, "threshold 0.5")):
    L.moses_set_async(1)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            ml._ck(L.moses_lottery_step(dm.h, mode, 0.5, 0, 1e-9, 1.0, None, 0, C.byref(pop)))
        torch.cuda.synchronize()
    L.moses_set_async(0)
    evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    if not evs:  # CUPTI taken (e.g. running under ncu): no timeline
        break
    t0 = evs[0].time_range.start
    print("---", name)
    for e in evs:
        print(f"{e.time_range.start - t0:9.1f} {e.time_range.elapsed_us():7.1f}  {e.name[:90]}")
