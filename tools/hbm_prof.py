"""The HBM-bound kernels of bench.py once each at L2-exceeding sizes (for ncu --set full):
momentum update over 268M parameters, segment-sum pooling of 4M statement rows."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
dims = [32768, 8192, 8, 1]
P = ml.param_count(dims)
dm = ml.DeviceModel(ml.CostModelParams(dims, np.zeros(P)), ml.PREC_BF16, max_rows=128)
L.moses_set_async(1)
for _ in range(2):
    ml._ck(L.moses_apply_update(dm.h, 1e-3, 0.9, None, 0, 1))
torch.cuda.synchronize()
dm.close()
gen = torch.Generator(device="cuda").manual_seed(0)
off = ml.synth_offsets(11, 900_000, 8)
H = torch.empty((int(off[-1]), 512), dtype=torch.bfloat16, device="cuda").normal_(generator=gen)
OFF = torch.from_numpy(off).cuda()
PO = torch.empty((900_000, 512), dtype=torch.float32, device="cuda")
for _ in range(2):
    ml._ck(L.moses_segment_sum_device(H.data_ptr(), ml.DTYPE_BF16, 512, 512, OFF.data_ptr(), 900_000, PO.data_ptr()))
torch.cuda.synchronize()
print("ok")
