"""The f1 candidate encoder over bench_search's 10.2M-config knob space (packed bf16 rows + FNV-1a
hashes): device time per call (CUDA events on the launching stream), for ncu captures."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
knobs = [("tile_x", [1 << i for i in range(16)]), ("tile_y", [1 << i for i in range(16)]),
         ("unroll", [0, 1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 128, 256, 512]),
         ("vectorize", [1 << i for i in range(8)]), ("parallel", [1 << i for i in range(13)]),
         ("split", list(range(1, 25)))]
n = int(np.prod([len(d) for _, d in knobs]))
task = (2.0, 8.0, 9.0, 5.0)
ld = 24
F = torch.empty((n, ld), dtype=torch.bfloat16, device="cuda")
Hh = torch.empty(n, dtype=torch.int64, device="cuda")


def encode():
    ml.encode_configs_device(task, knobs, 0, n, ml.DTYPE_BF16, C.c_void_p(F.data_ptr()), ld, 16,
                             C.c_void_p(Hh.data_ptr()))


for _ in range(3):
    encode()
torch.cuda.synchronize()
reps = 20
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    encode()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print(f"encode {n} configs: {ms * 1e3:.1f} us per call, {n * (ld * 2 + 8) / ms / 1e6:.0f} GB/s written")
