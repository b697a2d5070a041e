"""Short scoring run for ncu: 2 chunks of 64K programs through the per-layer scoring kernels
(PREC=BF16 env: bf16 weight-resident pairs; default BF16X3: the split-bf16 pairs)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml  # noqa: E402

DIMS = [164, 512, 512, 512, 512, 1]
L = ml.lib()
n = 131072
P = getattr(ml, "PREC_" + os.environ.get("PREC", "BF16X3"))
DT = ml.input_dtype(P)
dm = ml.DeviceModel(ml.init_random(DIMS, 1, strict=False), P, max_rows=65536)
ld = dm.packed_ld
X = torch.empty((n, ld), dtype=torch.bfloat16 if DT == ml.DTYPE_BF16 else torch.float32, device="cuda")
S = torch.empty(n, dtype=torch.float32, device="cuda")
assert L.moses_synth_features_device(3, 0, n, DIMS[0], DT, X.data_ptr(), ld) == 0
for _ in range(3):
    ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), DT, ld, n, S.data_ptr()))
torch.cuda.synchronize()
