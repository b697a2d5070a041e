"""Fused ranking step in the pooled bench configuration: event-bracketed time per call of the
default policy (cluster form at n = 512) with CTA 0's phase timestamps, or of the grid form (--grid)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml  # noqa: E402

L = ml.lib()
cluster = "--grid" not in sys.argv
L.moses_debug_set_rank_grid(0 if cluster else 1)  # 0: default policy
dims = [164, 512, 512, 512, 512, 1]
dm = ml.DeviceModel(ml.init_random(dims, 1, strict=False), getattr(ml, "PREC_" + (sys.argv[sys.argv.index("--prec") + 1] if "--prec" in sys.argv else "BF16X3")), 4096)
off = ml.synth_offsets(3, 512, 8)
x = np.random.default_rng(0).random((int(off[-1]), 164))
y = 0.1 + np.random.default_rng(1).random(512)
for _ in range(5):
    ml.gradients_pooled(dm, x, off, y)
buf = (C.c_ulonglong * 16)()
ml._ck(L.moses_debug_rank_trace(buf))
t = np.array(buf[:16], dtype=np.int64)
if cluster:
    names = ["start", "scores", "all-gather", "pairs", "cta reduce", "cluster sync", "coef"]
    print(" | ".join(f"{names[k]} {(t[k] - t[0]) / 1e3:.2f}" for k in range(7)))
ms = np.zeros(9)
cnt = np.zeros(9, dtype=np.int64)
ml._ck(L.moses_profile_begin())
for _ in range(20):
    ml.gradients_pooled(dm, x, off, y)
ml._ck(L.moses_profile_end(ms.ctypes.data, cnt.ctypes.data, 9))
print("rank category (event-bracketed, per call): %.2f us" % (ms[3] / max(cnt[3], 1) * 1e3))
