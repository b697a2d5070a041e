"""CUPTI timeline of the cfg3 fine-tune steps (bench_sections.bench_finetune): the Moses branch with the
adversary and the MMD^2 variant, one step each after warm-up."""
import ctypes as C
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_2201_05752_b200 import moseslab as ml  # noqa: E402

DIMS = [164, 512, 512, 512, 512, 1]
L = ml.lib()
params = ml.init_random(DIMS, 12345, strict=False)
dm = ml.DeviceModel(params, ml.PREC_BF16X3, max_rows=1024)
rng = np.random.default_rng(3)
replay = rng.random((256, DIMS[0]))
adv = ml.AdversaryState(replay, DIMS[-2])
xt = np.ascontiguousarray(rng.random((512, DIMS[0])))
yt = np.ascontiguousarray(0.1 + rng.random(512))
src = np.ascontiguousarray(rng.random((256, DIMS[0])))
loss, dl, cf, pop = C.c_double(), C.c_double(), C.c_double(), C.c_int64()


def moses():
    ml._ck(L.moses_gradients(dm.h, xt.ctypes.data, yt.ctypes.data, 512, DIMS[0], adv.h, 0.01, C.byref(loss)))
    ml._ck(L.moses_adversarial_step(adv.h, dm.h, xt.ctypes.data, 512, DIMS[0], 0.01, C.byref(dl), C.byref(cf)))
    ml._ck(L.moses_lottery_step(dm.h, 2, 0.5, 0, 1e-3, 1e-2, None, 0, C.byref(pop)))


def mmd():
    ml._ck(L.moses_gradients_mmd(dm.h, xt.ctypes.data, yt.ctypes.data, 512, DIMS[0], src.ctypes.data, 256, 0.01,
                                 float(np.sqrt(DIMS[-2] / 6.0)), C.byref(loss)))
    ml._ck(L.moses_lottery_step(dm.h, 2, 0.5, 0, 1e-3, 1e-2, None, 0, C.byref(pop)))


def fused():
    ml._ck(L.moses_moses_step(dm.h, adv.h, xt.ctypes.data, yt.ctypes.data, 512, DIMS[0], 0.01, 2, 0.5, 0, 1e-3, 1e-2,
                              C.byref(loss), C.byref(dl), C.byref(pop)))


for name, fn in (("moses (adversary)", moses), ("mmd", mmd), ("moses_moses_step (fused)", fused)):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    print(f"--- {name}: {evs[-1].time_range.end - t0:.1f} us device span")
    for e in evs:
        print(f"{e.time_range.start - t0:8.1f} {e.time_range.elapsed_us():7.1f}  {e.name[:70]}")
