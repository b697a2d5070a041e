import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import oracle as orc
from paper_2201_05752_b200 import moseslab as ml

def blocks(dims):
    off = 0
    out = []
    for l in range(len(dims) - 1):
        nw = dims[l] * dims[l + 1]
        out.append((f"W{l}", off, off + nw)); out.append((f"b{l}", off + nw, off + nw + dims[l + 1]))
        off += nw + dims[l + 1]
    return out

for dims, n in (([16, 512, 512, 1], 64), ([4, 8, 8, 1], 6), ([16, 512, 512, 1], 300)):
    p = ml.init_random(dims, 12345)
    rng = np.random.default_rng(0)
    x = rng.random((n, dims[0])); y = 0.1 + rng.random(n)
    g_ref, loss_ref = orc.gradients(dims, p.params, x, y)
    for prec in (ml.PREC_TF32, ml.PREC_BF16):
        dm = ml.DeviceModel(p, prec, 512)
        g, loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
        print(dims, n, "prec", prec, "loss", loss, loss_ref)
        for name, a, b in blocks(dims):
            r = g_ref[a:b]; q = g[a:b]
            err = np.max(np.abs(q - r)) / max(np.max(np.abs(r)), 1e-30)
            print(f"   {name}: rel {err:.3e}  ref[:4] {r[:4]}  got[:4] {q[:4]}")
