import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
from paper_2201_05752_b200 import moseslab as ml
from precision_model import device_gradients, nrel

def blocks(dims):
    off = 0; out = []
    for l in range(len(dims) - 1):
        nw = dims[l] * dims[l + 1]
        out.append((f"W{l}", off, off + nw)); out.append((f"b{l}", off + nw, off + nw + dims[l + 1]))
        off += nw + dims[l + 1]
    return out

for dims, n in (([164, 512, 512, 512, 512, 1], 512), ([164, 512, 512, 512, 512, 1], 256), ([16, 512, 512, 512, 1], 512), ([164, 512, 512, 1], 512)):
    p = ml.init_random(dims, 21, strict=False)
    x = np.random.default_rng(7).random((n, dims[0])); y = 0.1 + np.random.default_rng(8).random(n)
    for mode, prec in (("tf32", 1), ("bf16", 0)):
        g_ref, _ = device_gradients(dims, p.params, x, y, mode)
        dm = ml.DeviceModel(p, prec, 1024)
        g = ml.gradients(dm, ml.RankingBatch(x, y))
        g2 = ml.gradients(dm, ml.RankingBatch(x, y))
        print(dims, n, mode, "total", f"{nrel(g, g_ref):.2e}", "det", np.array_equal(g, g2))
        for name, a, b in blocks(dims):
            e = nrel(g[a:b], g_ref[a:b])
            if e > 1e-3:
                d = np.abs(g[a:b] - g_ref[a:b]); i = int(np.argmax(d))
                print(f"   {name}: rel {e:.2e} at {i} ref {g_ref[a+i]:.4e} got {g[a+i]:.4e}")
