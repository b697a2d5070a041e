"""Device time per category (CUDA events, moses_profile_*) of one pooled gradient call on the cfg2
shape, per operand precision. Quick comparison tool, not a bench line."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml  # noqa: E402

dims = [164, 512, 512, 512, 512, 1]
p = ml.init_random(dims, 12345, strict=False)
off = ml.synth_offsets(1, 512, 8)
x = np.random.default_rng(1).random((int(off[-1]), 164))
y = 0.1 + np.random.default_rng(2).random(512)
precs = [("bf16", ml.PREC_BF16), ("tf32", ml.PREC_TF32), ("fp32", ml.PREC_FP32)]
if hasattr(ml, "PREC_BF16X3"):
    precs.append(("bf16x3", ml.PREC_BF16X3))
for name, prec in precs:
    dm = ml.DeviceModel(p, prec, int(off[-1]) + 128)
    for _ in range(5):
        ml.gradients_pooled(dm, x, off, y)
    ml.profile_begin()
    K = 20
    for _ in range(K):
        ml.gradients_pooled(dm, x, off, y)
    prof = ml.profile_end()
    out = {c: round(v[0] / K * 1000, 1) for c, v in prof.items() if v[1]}
    out["total_us"] = round(sum(v[0] for v in prof.values()) / K * 1000, 1)
    print(json.dumps({"prec": name, "us_per_call": out}), flush=True)
