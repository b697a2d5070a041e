import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml
L = ml.lib()
dims = [164, 512, 512, 512, 512, 1]
dm = ml.DeviceModel(ml.init_random(dims, 1, strict=False), ml.PREC_BF16, 4096)
off = ml.synth_offsets(3, 512, 8)
x = np.random.default_rng(0).random((int(off[-1]), 164)); y = 0.1 + np.random.default_rng(1).random(512)
for _ in range(5):
    ml.gradients_pooled(dm, x, off, y)
buf = (C.c_ulonglong * 16)()
ml._ck(L.moses_debug_rank_trace(buf))
t = np.array(buf[:7], dtype=np.int64)
names = ["start", "rows summed", "seg sums", "pairs", "cta reduce", "cluster sync", "coef"]
print(" | ".join(f"{names[k]} {(t[k]-t[0])/1e3:.2f}" for k in range(7)))
