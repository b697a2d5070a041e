"""Host runtime-API timeline (CUPTI via torch.profiler) of one moses_moses_step call next to its kernels."""
import sys
sys.argv = ["x"]
exec(open("tools/finetune_prof.py").read().split("for name, fn in")[0])
for _ in range(5):
    fused()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    fused()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events()], key=lambda e: e.time_range.start)
t0 = min(e.time_range.start for e in evs)
for e in evs:
    print(f"{e.device_type.name[:4]} {e.time_range.start - t0:8.1f} {e.time_range.elapsed_us():7.1f}  {e.name[:60]}")

import time  # noqa: E402

for name, fn in (("moses (three calls)", moses), ("mmd", mmd), ("moses_moses_step", fused)):
    for _ in range(10):
        fn()
    t0 = time.perf_counter()
    for _ in range(100):
        fn()
    print(f"{name}: {1e6 * (time.perf_counter() - t0) / 100:.1f} us per call (wall)")
