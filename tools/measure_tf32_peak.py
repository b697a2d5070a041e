"""Dense TF32 tensor-core peak of this B200, measured the way the driver measures bf16 for
MEASURED_PEAKS.json (torch.matmul 8192^3, 2*N^3 FLOPs): best of 10 (burst) and back to back for 4 s
(sustained). Writes profiles/measured_tf32_peak.json (bench.py quotes TF32 fractions against it)."""
import json
import os
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
torch.backends.cuda.matmul.fp32_precision = "tf32" if hasattr(torch.backends.cuda.matmul, "fp32_precision") else None
N = 8192
a = torch.randn(N, N, device="cuda")
b = torch.randn(N, N, device="cuda")
c = a @ b
torch.cuda.synchronize()
flops = 2.0 * N ** 3
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c = a @ b
    e1.record()
    torch.cuda.synchronize()
    best = max(best, flops / (e0.elapsed_time(e1) / 1e3) / 1e12)
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
while time.perf_counter() - t0 < 4.0:
    for _ in range(10):
        c = a @ b
    n += 10
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sustained = n * flops / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"tf32_tflops": best, "tf32_tflops_sustained": sustained, "gpu": torch.cuda.get_device_name(0),
       "how": "torch.matmul fp32 with TF32 tensor cores, 8192^3 (2*N^3): best of 10 (burst) and back to back "
              "for 4 s (sustained), CUDA events"}
os.makedirs("profiles", exist_ok=True)
json.dump(out, open("profiles/measured_tf32_peak.json", "w"), indent=1)
print(json.dumps(out))
