"""Kernel timeline of moses_topk_device over a 100M-score pool (bench.py's HBM case)."""
import ctypes as C
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
n = 100_000_000
gen = torch.Generator(device="cuda").manual_seed(0)
S = torch.empty(n, dtype=torch.float32, device="cuda").normal_(generator=gen)
idx = (C.c_int64 * 1024)()
for _ in range(3):
    ml._ck(L.moses_topk_device(S.data_ptr(), n, 1024, idx))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    ml._ck(L.moses_topk_device(S.data_ptr(), n, 1024, idx))
print(f"wall {1e3 * (time.perf_counter() - t0) / 10:.3f} ms per call")
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        ml._ck(L.moses_topk_device(S.data_ptr(), n, 1024, idx))
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{e.time_range.start - t0:10.1f} {e.time_range.elapsed_us():9.1f}  {e.name[:80]}")
tr = (C.c_uint64 * 16)()
ml._ck(L.moses_debug_topk_trace(tr))
names = ["sample+hist", "level 1", "level 2", "pass", "barrier", "final"]
print("phases (us):", ", ".join(f"{names[i]} {(tr[i + 1] - tr[i]) / 1e3:.1f}" for i in range(6)),
      f"(sample loop {(tr[7] - tr[0]) / 1e3:.1f}); candidates {tr[8]}; pass end over CTAs "
      f"{(tr[9] - tr[3]) / 1e3:.1f}-{(tr[10] - tr[3]) / 1e3:.1f} us after its start")
