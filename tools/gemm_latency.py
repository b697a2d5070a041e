"""Per-launch device time of the GEMM kernel families on the training-step shapes (back-to-back
launches, warm L2). Used to pick tiles / split-K for the latency-bound batch-512 step."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml

L = ml.lib()
L.moses_debug_gemm_timed.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_int,
                                     C.c_void_p, C.c_longlong, C.c_int, C.c_int, C.c_void_p, C.c_longlong,
                                     C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_int,
                                     C.POINTER(C.c_float)]
L.moses_debug_set_cluster.argtypes = [C.c_int]
L.moses_debug_set_persistent.argtypes = [C.c_int]
dev = "cuda"
R = int(sys.argv[1]) if len(sys.argv) > 1 else 2560


def t(M, N, K, a, lda, amn, b, ldb, bmn, epi, out, ldo, bias=None, relu=0, bn=0, mask=None, ldm=0, iters=200):
    ms = C.c_float()
    rc = L.moses_debug_gemm_timed(2, M, N, K, a.data_ptr(), lda, amn, b.data_ptr(), ldb, bmn, epi, out.data_ptr(), ldo,
                                  bias.data_ptr() if bias is not None else None, relu, bn,
                                  mask.data_ptr() if mask is not None else None, ldm, iters, C.byref(ms))
    assert rc == 0, L.moses_last_error()
    return ms.value * 1e3


bf = torch.bfloat16
act = torch.randn(R, 520, device=dev).to(bf)
x0 = torch.randn(R, 168, device=dev).to(bf)
w = torch.randn(512 * 512, device=dev).to(bf)
w0 = torch.randn(164 * 512, device=dev).to(bf)
dz = torch.randn(R, 512, device=dev).to(bf)
out = torch.empty(R, 520, device=dev).to(bf)
g = torch.empty(513 * 512, device=dev, dtype=torch.float32)
bias = torch.randn(512, device=dev)
EPI_FWD, EPI_DGRAD, EPI_F32 = 0, 1, 2
if __name__ != "__main__":
    pass
else:
  for cl, pe in ((1, 1), (0, 1), (0, 0)):
        L.moses_debug_set_cluster(cl)
        L.moses_debug_set_persistent(pe)
        print(f"--- cluster={cl} persistent={pe}  rows={R}")
        for K in (64, 128, 256, 512):
            us = t(R, 512, K, act, 520, 0, w, 512, 1, EPI_FWD, out, 520, bias, 1)
            print(f"fwd  K={K:4d}: {us:7.2f} us  {2 * R * 512 * K / us / 1e6:7.1f} TF/s")
        us = t(R, 512, 164, x0, 168, 0, w0, 512, 1, EPI_FWD, out, 520, bias, 1)
        print(f"fwd0 K=164 : {us:7.2f} us")
        us = t(R, 512, 512, dz, 512, 0, w, 512, 0, EPI_DGRAD, out, 520, None, 0, 0, act, 520)
        print(f"dgrad      : {us:7.2f} us")
        for bn in (0, 64, 128, 256):
            try:
                us = t(513, 512, R, act, 520, 1, dz, 512, 1, EPI_F32, g, 512, bn=bn)
                print(f"wgrad bn={bn:3d}: {us:7.2f} us  {2 * R * 512 * 513 / us / 1e6:7.1f} TF/s")
            except AssertionError as e:
                print("wgrad bn", bn, e)
