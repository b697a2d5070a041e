"""Time the forward GEMM kernels on the scoring shape (64K-row chunk) with each kernel family."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml
import ctypes as C
L = ml.lib()
L.moses_debug_set_cluster.argtypes = [C.c_int]; L.moses_debug_set_persistent.argtypes = [C.c_int]
DIMS = [164, 512, 512, 512, 512, 1]
n = 1 << 20
dm = ml.DeviceModel(ml.init_random(DIMS, 1, strict=False), ml.PREC_BF16, max_rows=65536)
ld = dm.packed_ld
X = torch.empty((n, ld), dtype=torch.bfloat16, device="cuda")
S = torch.empty(n, dtype=torch.float32, device="cuda")
assert L.moses_synth_features_device(3, 0, n, DIMS[0], ml.DTYPE_BF16, X.data_ptr(), ld) == 0
sp = C.c_void_p(); L.moses_model_stream(dm.h, C.byref(sp)); st = torch.cuda.ExternalStream(sp.value)
flops = n * sum(2 * DIMS[l] * DIMS[l + 1] for l in range(len(DIMS) - 2))
for cl, pe in ((1, 1), (0, 1), (0, 0)):
    L.moses_debug_set_cluster(cl); L.moses_debug_set_persistent(pe)
    for _ in range(2):
        ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), ml.DTYPE_BF16, ld, n, S.data_ptr()))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(5):
        ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), ml.DTYPE_BF16, ld, n, S.data_ptr()))
    b.record(st); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"cluster={cl} persistent={pe}: {ms:.3f} ms per 1M programs -> {flops / ms / 1e9:.0f} TFLOP/s, {n / ms / 1e3:.1f} M programs/s")
