"""Fine-tune sized steps (768 / 1280 / 2560 rows) with the split chain on 4-CTA clusters (default) vs CTA
pairs on 8-CTA clusters (moses_debug_set_chain_pair): wall time per moses_moses_step call."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml  # noqa: E402

DIMS = [164, 512, 512, 512, 512, 1]
L = ml.lib()
params = ml.init_random(DIMS, 12345, strict=False)
rng = np.random.default_rng(3)
for n, rep in ((512, 256), (1024, 256), (2048, 512)):
    dm = ml.DeviceModel(params, ml.PREC_BF16X3, max_rows=n + rep)
    adv = ml.AdversaryState(rng.random((rep, DIMS[0])), DIMS[-2])
    xt = np.ascontiguousarray(rng.random((n, DIMS[0])))
    yt = np.ascontiguousarray(0.1 + rng.random(n))
    loss, dl, pop = C.c_double(), C.c_double(), C.c_int64()
    for pair in (0, 1):
        L.moses_debug_set_chain_pair(pair)
        f = lambda: ml._ck(L.moses_moses_step(dm.h, adv.h, xt.ctypes.data, yt.ctypes.data, n, DIMS[0], 0.01, 2, 0.5, 0,
                                               1e-3, 1e-2, C.byref(loss), C.byref(dl), C.byref(pop)))
        for _ in range(10):
            f()
        t0 = time.perf_counter()
        for _ in range(50):
            f()
        print(f"rows {n + rep}: chain_pair={pair}: {1e6 * (time.perf_counter() - t0) / 50:.1f} us per Moses step")
    L.moses_debug_set_chain_pair(0)
    dm.close()
