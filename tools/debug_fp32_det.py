import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
import numpy as np
import oracle as orc
from paper_2201_05752_b200 import moseslab as ml
def f32(a): return np.asarray(a, np.float32).astype(np.float64)
for dims in ([16, 512, 512, 1], [164, 512, 512, 512, 512, 1], [33, 72, 40, 1]):
  for n in (12, 512):
    p = ml.CostModelParams(dims, f32(orc.init_random(dims, 21, strict=False)))
    x = f32(np.random.default_rng(7).random((n, dims[0]))); y = f32(0.1 + np.random.default_rng(8).random(n))
    g64, _ = orc.gradients(dims, p.params, x, y, threads=8)
    dm = ml.DeviceModel(p, ml.PREC_FP32, 1024)
    errs = []; base = None; ndiff = 0
    for it in range(30):
        g = ml.gradients(dm, ml.RankingBatch(x, y))
        if base is None: base = g
        ndiff += int(not np.array_equal(g, base))
        errs.append(float(np.max(np.abs(g - g64)) / np.max(np.abs(g64))))
    print(dims, n, "nondeterministic runs", ndiff, "max err %.3g" % max(errs), flush=True)
