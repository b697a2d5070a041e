"""Phase timeline of the fused chain kernels (cluster 0), from %globaltimer stamps."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
L.moses_debug_set_chain_trace.argtypes = [C.c_void_p]
dims = [164, 512, 512, 512, 512, 1]
R = int(sys.argv[1]) if len(sys.argv) > 1 else 2560
PREC = getattr(ml, "PREC_" + os.environ.get("PREC", "BF16X3"))
DT = ml.input_dtype(PREC)
dm = ml.DeviceModel(ml.init_random(dims, 1, strict=False), PREC, R)
ld = dm.packed_ld
X = torch.zeros((R, ld), dtype=torch.bfloat16 if DT == ml.DTYPE_BF16 else torch.float32, device="cuda")
X[:, :164] = torch.rand(R, 164, device="cuda").to(X.dtype)
X[:, 164] = 1
Y = torch.rand(R, device="cuda") + 0.1
S = torch.empty(R, device="cuda")
tr = torch.zeros(4 * 8 * 8, dtype=torch.int64, device="cuda")
EV = ["mma_start", "mma_issued", "acc_seen", "stores_fenced", "cl_wait_done", "mc_issued", "k_start", "k_end"]
if os.environ.get("PREC", "BF16X3") == "BF16X3":  # streamed split chain: its own event meanings
    EV = ["mma_start", "mma_issued", "acc_seen", "slice_written", "ready_seen", "-", "k_start", "k_end"]


def show(title):
    t = tr.cpu().numpy().reshape(4, 8, 8).astype(np.int64)
    t0 = t[:, 0, 6][t[:, 0, 6] > 0].min()
    for row, nm in ((5, "W issued"), (6, "A issued"), (4, "MMA start")):
        if t[0, row, 0] > 0 and t[0, row, 0] - t0 < 10**9:
            print(f"  layer-1 positions {nm:9s}: " + " ".join(f"{(v - t0) / 1e3:6.2f}" for v in t[0, row]))
    print(f"--- {title} (us from kernel start of CTA 0..3)")
    for q in range(4):
        print(f"  CTA{q} start {(t[q,0,6]-t0)/1e3:.2f} end {(t[q,0,7]-t0)/1e3:.2f}")
    for l in range(8):
        if t[0, l, 0] == 0:
            continue
        row = []
        for e in range(6):
            v = t[0, l, e]
            row.append(f"{EV[e]} {(v - t0) / 1e3:6.2f}" if v > 0 else f"{EV[e]}   -   ")
        print(f"  L{l}: " + " | ".join(row))
        for e in (0, 2, 3, 4):
            print(f"      {EV[e]:14s} per CTA: " + " ".join(f"{(t[q, l, e] - t0) / 1e3:6.2f}" if t[q, l, e] > 0 else "   -  "
                                                        for q in range(4)))


for _ in range(3):
    ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), DT, ld, R, S.data_ptr()))
torch.cuda.synchronize()
tr.zero_()
L.moses_debug_set_chain_trace(tr.data_ptr())
ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), DT, ld, R, S.data_ptr()))
torch.cuda.synchronize()
show("forward chain")
tr.zero_()
ml._ck(L.moses_gradients_device(dm.h, X.data_ptr(), ld, Y.data_ptr(), R, None))
torch.cuda.synchronize()
show("dZ chain")
L.moses_debug_set_chain_trace(None)
