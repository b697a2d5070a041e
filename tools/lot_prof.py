"""One fused ratio-mode lottery step on a 268M-scalar synthetic model (bench.py's HBM case), for
ncu launch lists: python tools/lot_prof.py [ratio|threshold] [reps]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml
from paper_2201_05752_b200.distributed import device_gradient_tensor

L = ml.lib()
mode = 2 if (len(sys.argv) < 2 or sys.argv[1] == "ratio") else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dims = [32768, 8192, 8, 1]
P = ml.param_count(dims)
dm = ml.DeviceModel(ml.CostModelParams(dims, np.zeros(P)), ml.PREC_BF16, max_rows=128)
wptr = C.POINTER(C.c_float)()
L.moses_model_device_ptrs(dm.h, C.byref(wptr), None, None)


class _CAI:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


w = torch.as_tensor(_CAI(C.cast(wptr, C.c_void_p).value, P), device="cuda")
g = device_gradient_tensor(dm)
gen = torch.Generator(device="cuda").manual_seed(0)
w.normal_(0, 0.05, generator=gen)
g.normal_(0, 1e-2, generator=gen)
g[torch.rand(P, device="cuda", generator=gen) < 0.4] = 0.0
torch.cuda.synchronize()
pop = C.c_int64()
for _ in range(reps):
    ml._ck(L.moses_lottery_step(dm.h, mode, 0.5, 0, 1e-3, 1e-2, None, 0, C.byref(pop)))
torch.cuda.synchronize()
print("popcount", pop.value, "of", P)

if len(sys.argv) > 3 and sys.argv[3] == "torchprof":
    from torch.profiler import ProfilerActivity, profile

    L.moses_set_async(1)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            ml._ck(L.moses_lottery_step(dm.h, mode, 0.5, 0, 1e-3, 1e-2, None, 0, C.byref(pop)))
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    for e in evs:
        print(f"{e.time_range.start - t0:10.1f} {e.time_range.elapsed_us():9.1f}  {e.name[:80]}")
    sp = C.c_void_p()
    L.moses_model_stream(dm.h, C.byref(sp))
    st = torch.cuda.ExternalStream(sp.value)
    for async_ in (1, 0):
        L.moses_set_async(async_)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(5):
            ml._ck(L.moses_lottery_step(dm.h, mode, 0.5, 0, 1e-3, 1e-2, None, 0, C.byref(pop)))
        b.record(st)
        torch.cuda.synchronize()
        print(f"async={async_}: {a.elapsed_time(b) / 5:.3f} ms per step")
