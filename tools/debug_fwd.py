import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2201_05752_b200 import moseslab as ml
from precision_model import device_forward
dims = [164, 512, 512, 1]
p = ml.init_random(dims, 21, strict=False)
x = np.random.default_rng(7).random((512, 164))
for mode, prec in (("tf32", 1), ("bf16", 0)):
    dm = ml.DeviceModel(p, prec, 1024)
    h = ml.penultimate_activations(dm, x)
    s_model, h_full, acts, _, _ = device_forward(dims, p.params, x, mode)
    flips = np.sum((h > 0) != (h_full > 0))
    err = np.abs(h - h_full).max() / np.abs(h_full).max()
    d = np.abs(h - h_full)
    i = np.unravel_index(np.argmax(d), d.shape)
    print(mode, "flips", flips, "max rel", err, "at", i, h[i], h_full[i])
    # first layer check
    z1 = acts[0] @ acts[0][:0].T if False else None
    print("  mean |h|", np.abs(h_full).mean(), "frac relative err >1e-5:", np.mean(d > 1e-5 * np.abs(h_full).max()))
