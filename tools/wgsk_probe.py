"""Split-K wgrad probe: wgrad device time (profiler category gemm_wgrad, CUDA events) of the cfg2 / cfg5
training step for several TMEM promotion intervals (kc k-blocks of 64 rows) and cluster widths, plus a
clock64 trace of block 0 (producer issue, MMA stage start, drain chunk end) for the default setting."""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench as B
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
L.moses_debug_set_wgrad_sk.argtypes = [C.c_int, C.c_int]
L.moses_debug_wgrad_sk_probe.argtypes = [C.c_int, C.c_void_p]
out = {}
for name, dims, n in (("cfg5", [164, 512, 512, 1], 4096), ("cfg2", [164, 512, 512, 512, 512, 1], 2560)):
    dm = ml.DeviceModel(ml.init_random(dims, B.SEED_MODEL, strict=False), ml.PREC_BF16X3, max_rows=n)
    ld = dm.packed_ld
    X = torch.empty((n, ld), dtype=torch.float32, device="cuda")
    Y = torch.empty(n, dtype=torch.float32, device="cuda")
    assert L.moses_synth_features_device(B.SEED_DATA + 5, 0, n, dims[0], ml.DTYPE_F32, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(B.SEED_DATA + 5, 0, n, Y.data_ptr()) == 0
    torch.cuda.synchronize()
    L.moses_set_async(1)

    def step():
        ml._ck(L.moses_train_step_device(dm.h, X.data_ptr(), ld, Y.data_ptr(), n, C.c_double(0.0), C.c_double(0.9), None))

    res = {}
    for sk, splits, kc in [(0, 0, 0), (1, 0, 2), (1, 0, 4), (1, 0, 8), (1, 1, 2), (1, 2, 2), (1, 4, 2), (1, 8, 2),
                           (1, 0, 64)]:
        L.moses_debug_set_wgrad_sk(sk, splits)
        L.moses_debug_wgrad_sk_probe(kc, None)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ml.profile_begin()
        for _ in range(20):
            step()
        torch.cuda.synchronize()
        prof = ml.profile_end()
        res[f"sk{sk}_S{splits}_kc{kc}"] = prof["gemm_wgrad"][0] / 20 * 1e3
    tr = torch.zeros(131 + 2 * 148, dtype=torch.int64, device="cuda")
    L.moses_debug_set_wgrad_sk(1, 0)
    L.moses_debug_wgrad_sk_probe(2, tr.data_ptr())
    step()
    torch.cuda.synchronize()
    L.moses_debug_wgrad_sk_probe(0, None)
    t = tr.cpu().numpy().astype(np.int64)
    t0 = t[130]
    rel = lambda a: [int(v - t0) if v else None for v in a]
    st, en = t[131::2][:148], t[132::2][:148]
    live = [(b, int(st[b]), int(en[b])) for b in range(148) if st[b] and en[b]]
    g0 = min(x[1] for x in live)
    ctas = {"n": len(live), "start_ns": sorted(x[1] - g0 for x in live)[::12],
            "end_ns": sorted(x[2] - g0 for x in live)[::12],
            "slowest": sorted(((x[2] - x[1], x[0]) for x in live))[-6:]}
    out[name] = {"ctas": ctas, "wgrad_us": res, "trace": {"prod_hi": rel(t[0:32]), "prod_lo": rel(t[32:64]), "mma_start": rel(t[64:96]),
                                             "drain_end": rel(t[96:126]), "published": rel(t[127:128]), "barrier_done": rel(t[126:127]), "mainloop_end": rel(t[128:129]),
                                             "reduce_end": rel(t[129:130])}}
    L.moses_set_async(0)
    dm.close()
print(json.dumps(out, indent=1))
