"""Time the scoring forward (64K-row chunks, {164,512x4,1} bf16) with each kernel family:
chain (fused 4-CTA cluster chain), cluster GEMM, persistent GEMM, plain GEMM."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
for f in ("moses_debug_set_cluster", "moses_debug_set_persistent", "moses_debug_set_chain", "moses_debug_set_fwd", "moses_debug_set_pair"):
    getattr(L, f).argtypes = [C.c_int]
DIMS = [164, 512, 512, 512, 512, 1]
n = 1 << 20
dm = ml.DeviceModel(ml.init_random(DIMS, 1, strict=False), ml.PREC_BF16, max_rows=65536)
ld = dm.packed_ld
X = torch.empty((n, ld), dtype=torch.bfloat16, device="cuda")
S = torch.empty(n, dtype=torch.float32, device="cuda")
assert L.moses_synth_features_device(3, 0, n, DIMS[0], ml.DTYPE_BF16, X.data_ptr(), ld) == 0
sp = C.c_void_p()
L.moses_model_stream(dm.h, C.byref(sp))
st = torch.cuda.ExternalStream(sp.value)
flops = n * sum(2 * DIMS[l] * DIMS[l + 1] for l in range(len(DIMS) - 2))
ref = None
FAMILIES = (("pair", 1, 1, 1, 1, 1), ("fwd", 0, 0, 1, 1, 0), ("persistent", 0, 0, 1, 0, 0), ("plain", 0, 0, 0, 0, 0))
only = sys.argv[1] if len(sys.argv) > 1 else None
for name, ch, cl, pe, fw, pa in FAMILIES:
    if only and name != only:
        continue
    L.moses_debug_set_chain(ch)
    L.moses_debug_set_cluster(cl)
    L.moses_debug_set_persistent(pe)
    L.moses_debug_set_fwd(fw)
    L.moses_debug_set_pair(pa)
    for _ in range(2):
        ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), ml.DTYPE_BF16, ld, n, S.data_ptr()))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(5):
        ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), ml.DTYPE_BF16, ld, n, S.data_ptr()))
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    if ref is None:
        ref = S.clone()
    dev = float((S - ref).abs().max() / ref.abs().max())
    print(f"{name:10s}: {ms:.3f} ms per 1M programs -> {flops / ms / 1e9:.0f} TFLOP/s, "
          f"{n / ms / 1e3:.1f} M programs/s (max rel dev vs first {dev:.2e})", flush=True)
L.moses_debug_set_chain(1)
L.moses_debug_set_cluster(1)
L.moses_debug_set_persistent(1)
L.moses_debug_set_fwd(1)
L.moses_debug_set_pair(1)
