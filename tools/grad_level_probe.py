"""Per-level gradient error of each precision vs the fp64 oracle on the cfg2 shape, plus the error
of a numpy emulation of the same operand rounding with exact (fp64) accumulation — separates operand
rounding from tensor-core accumulation error."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from paper_2201_05752_b200 import moseslab as ml  # noqa: E402
import oracle as orc  # noqa: E402

dims = [164, 512, 512, 512, 512, 1]
p = ml.init_random(dims, 12345, strict=False)
off = ml.synth_offsets(1, 512, 8)
x = np.random.default_rng(1).random((int(off[-1]), 164))
y = 0.1 + np.random.default_rng(2).random(512)
g_ref, _ = orc.gradients_pooled(dims, p.params, x, off, y, threads=16)
offs = [0]
for l in range(len(dims) - 1):
    offs.append(offs[-1] + dims[l] * dims[l + 1] + dims[l + 1])


def per_level(g):
    out = []
    for l in range(len(dims) - 1):
        a, b = offs[l], offs[l + 1]
        wb = a + dims[l] * dims[l + 1]
        ref_w, ref_b = g_ref[a:wb], g_ref[wb:b]
        out.append({"lvl": l, "w_nrel": float(np.max(np.abs(g[a:wb] - ref_w)) / np.max(np.abs(ref_w))),
                    "w_frob": float(np.linalg.norm(g[a:wb] - ref_w) / np.linalg.norm(ref_w)),
                    "b_nrel": float(np.max(np.abs(g[wb:b] - ref_b)) / np.max(np.abs(ref_b)))})
    return out


for name, prec in (("bf16x3", ml.PREC_BF16X3), ("fp32", ml.PREC_FP32), ("tf32", ml.PREC_TF32)):
    dm = ml.DeviceModel(p, prec, int(off[-1]) + 128)
    g = ml.gradients_pooled(dm, x, off, y)
    print(json.dumps({"prec": name, "levels": per_level(g)}), flush=True)

# error distribution of the bf16x3 level-3 gradient (ReLU-kink flips give a few large entries)
dm = ml.DeviceModel(p, ml.PREC_BF16X3, int(off[-1]) + 128)
g = ml.gradients_pooled(dm, x, off, y)
for lvl in (1, 3):
    a = offs[lvl]
    wb = a + dims[lvl] * dims[lvl + 1]
    b = offs[lvl + 1]
    for name, sl in (("w", slice(a, wb)), ("b", slice(wb, b))):
        d = np.abs(g[sl] - g_ref[sl]) / np.max(np.abs(g_ref[sl]))
        q = np.quantile(d, [0.5, 0.9, 0.99, 0.999, 1.0])
        print(json.dumps({"lvl": lvl, "part": name, "quantiles_50_90_99_999_max": [float(v) for v in q],
                          "n_above_1e-4": int(np.sum(d > 1e-4))}), flush=True)
