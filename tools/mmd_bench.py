"""cfg3 MMD^2 between 50k source and 5k target 512-d representations (device-resident fp32)."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
m, n, w = 50_000, 5_000, 512
gen = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((m + n, w), device="cuda", generator=gen)
X[m:] += 0.1
out = C.c_double()
for _ in range(2):
    ml._ck(L.moses_mmd2_device(C.c_void_p(X.data_ptr()), m, C.c_void_p(X[m:].data_ptr()), n, w, w, 22.6, C.byref(out)))
torch.cuda.synchronize()
t0 = time.perf_counter()
reps = 5
for _ in range(reps):
    ml._ck(L.moses_mmd2_device(C.c_void_p(X.data_ptr()), m, C.c_void_p(X[m:].data_ptr()), n, w, w, 22.6, C.byref(out)))
dt = (time.perf_counter() - t0) / reps
flops = 2 * w * (m * (m + 1) / 2 + n * (n + 1) / 2 + m * n)
print(f"mmd2 {out.value:.6e}: {dt * 1e3:.3f} ms, {flops / dt / 1e12:.1f} TFLOP/s (unique pairs, tf32)")
