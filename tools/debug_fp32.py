"""Per-level error of the FP32 (3xTF32) path vs the fp64 oracle (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
import numpy as np
import oracle as orc
from paper_2201_05752_b200 import moseslab as ml

def f32(a): return np.asarray(a, np.float32).astype(np.float64)
def levels(dims):
    out, o = [], 0
    for l in range(len(dims) - 1):
        out.append((f"W{l}", o, o + dims[l] * dims[l + 1])); o += dims[l] * dims[l + 1]
        out.append((f"b{l}", o, o + dims[l + 1])); o += dims[l + 1]
    return out

import json
CASES = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [[[164, 512, 512, 1], 12], [[164, 512, 512, 1], 512],
                                                          [[164, 512, 512, 512, 512, 1], 300]]
PRECS = [ml.PREC_FP32] if len(sys.argv) > 2 else [ml.PREC_FP32, ml.PREC_TF32]
for dims, n in CASES:
    p = ml.CostModelParams(dims, f32(orc.init_random(dims, 21, strict=False)))
    x = f32(np.random.default_rng(7).random((n, dims[0]))); y = f32(0.1 + np.random.default_rng(8).random(n))
    s64, h64 = orc.forward(dims, p.params, x, threads=8)
    for prec in PRECS:
        dm = ml.DeviceModel(p, prec, 1024)
        s = ml.predict(dm, x); h = ml.penultimate_activations(dm, x)
        print(dims, n, "prec", prec, "scores nrel %.3g" % (np.max(np.abs(s - s64)) / np.max(np.abs(s64))),
              "h nrel %.3g" % (np.max(np.abs(h - h64)) / np.max(np.abs(h64))))
        g64, l64 = orc.gradients(dims, p.params, x, y, threads=8)
        g, l = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
        print("   loss rel %.3g" % (abs(l - l64) / abs(l64)))
        for name, a, b in levels(dims):
            d = np.abs(g[a:b] - g64[a:b]); mx = np.max(np.abs(g64[a:b]))
            print("   %-3s max|ref| %.3g  nrel %.3g  frob %.3g  argmax %d" % (name, mx, d.max() / mx,
                  np.linalg.norm(g[a:b] - g64[a:b]) / np.linalg.norm(g64[a:b]), int(np.argmax(d))))
