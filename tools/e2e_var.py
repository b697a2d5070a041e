"""Repeatability of the bench e2e leg (moses_train_step_pooled_async, 1000 steps, 4 host batches)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench as B  # noqa: E402
from paper_2201_05752_b200 import moseslab as ml  # noqa: E402

L = ml.lib()
off = ml.synth_offsets(B.SEED_DATA, 4 * B.BATCH, B.MAX_STMTS)
dm = ml.DeviceModel(ml.init_random(B.DIMS, B.SEED_MODEL, strict=False), ml.PREC_BF16, max_rows=2560)
rng = np.random.default_rng(0)
hb = []
for b in range(4):
    lo, hi = int(off[b * B.BATCH]), int(off[(b + 1) * B.BATCH])
    hb.append((torch.from_numpy(rng.random((hi - lo, 164))).pin_memory(),
               torch.from_numpy(np.ascontiguousarray(off[b * B.BATCH:(b + 1) * B.BATCH + 1] - lo)).pin_memory(),
               torch.from_numpy(0.1 + rng.random(B.BATCH)).pin_memory()))
losses = torch.zeros(1100, dtype=torch.float64).pin_memory()
ptrs = [(x.data_ptr(), x.shape[0], o.data_ptr(), y.data_ptr()) for x, o, y in hb]
lp = [losses[k:k + 1].data_ptr() for k in range(1100)]
f = L.moses_train_step_pooled_async
for rep in range(6):
    for k in range(5):
        xp, n, op, yp = ptrs[k % 4]
        f(dm.h, xp, n, 164, op, B.BATCH, yp, B.LR, B.MU, lp[k])
    L.moses_model_synchronize(dm.h)
    t0 = time.perf_counter()
    for k in range(1000):
        xp, n, op, yp = ptrs[k % 4]
        f(dm.h, xp, n, 164, op, B.BATCH, yp, B.LR, B.MU, lp[k])
    L.moses_model_synchronize(dm.h)
    dt = (time.perf_counter() - t0) / 1000
    print(f"rep {rep}: {dt * 1e6:.1f} us/step -> {B.BATCH / dt / 1e6:.2f} M samples/s", flush=True)
