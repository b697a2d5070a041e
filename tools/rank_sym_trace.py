"""Symmetric ranking step at cfg5 size (n = 4096 plain rows): CTA 0's phase stamps (globaltimer, us)
and the event-bracketed rank time per call, against the grid form."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml  # noqa: E402

L = ml.lib()
dims = [164, 512, 512, 1]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dm = ml.DeviceModel(ml.init_random(dims, 1), ml.PREC_BF16X3, n)
x = np.random.default_rng(0).random((n, 164))
y = 0.1 + np.random.default_rng(1).random(n)
for grid in (0, 1):
    L.moses_debug_set_rank_grid(grid)
    for _ in range(5):
        ml.gradients(dm, ml.RankingBatch(x, y))
    if grid == 0:
        buf = (C.c_ulonglong * 16)()
        ml._ck(L.moses_debug_rank_trace(buf))
        t = np.array(buf[:16], dtype=np.int64)
        names = {8: "start", 9: "scores", 10: "pairs", 11: "grid sync", 12: "rows"}
        print(" | ".join(f"{names[k]} {(t[k] - t[8]) / 1e3:.2f}" for k in range(8, 13)))
    ms = np.zeros(9)
    cnt = np.zeros(9, dtype=np.int64)
    ml._ck(L.moses_profile_begin())
    for _ in range(20):
        ml.gradients(dm, ml.RankingBatch(x, y))
    ml._ck(L.moses_profile_end(ms.ctypes.data, cnt.ctypes.data, 9))
    print(("grid" if grid else "sym") + " rank (event-bracketed, per call): %.2f us" % (ms[3] / max(cnt[3], 1) * 1e3))
L.moses_debug_set_rank_grid(0)
L.moses_debug_set_rank_grid(0)
ml.gradients(dm, ml.RankingBatch(x, y))
buf = (C.c_ulonglong * 2560)()
ml._ck(L.moses_debug_rank_cta_trace(buf))
t = np.array(buf[:], dtype=np.int64).reshape(512, 5)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
print("ctas", len(t))
for k, nm in enumerate(["start", "scores", "pairs", "grid sync", "rows"]):
    c = rel[:, k]
    print(f"{nm:10s} min {c.min():6.2f} med {np.median(c):6.2f} max {c.max():6.2f}  argmax {int(np.argmax(c))}")
print("pairs duration: min %.2f med %.2f max %.2f" % tuple(np.percentile(rel[:, 2] - rel[:, 1], [0, 50, 100])))
slow = np.argsort(rel[:, 2] - rel[:, 1])[-8:]
print("slowest pair phases (cta, dur):", [(int(b), round(float(rel[b, 2] - rel[b, 1]), 2)) for b in slow])
