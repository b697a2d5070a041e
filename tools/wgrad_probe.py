"""Weight-gradient GEMM shape (M=513, N=512, K=rows) per-launch time vs K and operand majorness."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml
import tools.gemm_latency as GL  # noqa: F401  (argtypes)

L = ml.lib()
t = GL.t
bf = torch.bfloat16
for R in (256, 576, 1152, 2304):
    act = torch.randn(R, 520, device="cuda").to(bf)
    dz = torch.randn(R, 512, device="cuda").to(bf)
    actT = act.t().contiguous()  # [520][R]: K-major view for M
    dzT = dz.t().contiguous()
    g = torch.empty(513 * 512, device="cuda", dtype=torch.float32)
    for bn in (64, 128):
        mn = t(513, 512, R, act, 520, 1, dz, 512, 1, 2, g, 512, bn=bn)
        km = t(513, 512, R, actT, R, 0, dzT, R, 0, 2, g, 512, bn=bn)
        print(f"rows={R:5d} bn={bn:3d}: MN/MN {mn:7.2f} us   K/K {km:7.2f} us", flush=True)
