"""Dev probe: raw tcgen05 GEMM cases vs torch (run on a B200)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml

VERB = False
L = ml.lib()
L.moses_debug_gemm.restype = C.c_int
L.moses_debug_gemm.argtypes = [C.c_int] * 4 + [C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_longlong, C.c_int,
                                               C.c_int, C.c_void_p, C.c_longlong, C.c_void_p, C.c_int, C.c_int,
                                               C.c_void_p, C.c_longlong]


def case(elem, M, N, K, a_mn, b_mn, bn, epi=2, relu=0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dt = torch.bfloat16 if elem == 2 else torch.float32
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    A = A.to(dt)
    B = B.to(dt)
    # stored layouts
    As = A.t().contiguous() if a_mn else A.contiguous()  # MN-major: [K][M]
    Bs = B.t().contiguous() if b_mn else B.contiguous()
    lda = M if a_mn else K
    ldb = N if b_mn else K
    pad = lambda x: x
    ref = (A.float() @ B.float().t())
    bias = torch.randn(N, device="cuda", generator=g)
    if epi == 2:
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
        rc = L.moses_debug_gemm(elem, M, N, K, As.data_ptr(), lda, a_mn, Bs.data_ptr(), ldb, b_mn, 2, out.data_ptr(), N,
                                None, 0, bn, None, 0)
    else:
        out = torch.zeros(M, N, device="cuda", dtype=dt)
        rc = L.moses_debug_gemm(elem, M, N, K, As.data_ptr(), lda, a_mn, Bs.data_ptr(), ldb, b_mn, 0, out.data_ptr(), N,
                                bias.data_ptr(), relu, bn, None, 0)
        ref = ref + bias
        if relu:
            ref = ref.clamp_min(0)
    torch.cuda.synchronize()
    if rc:
        print("rc", rc, L.moses_last_error())
        return
    o = out.float()
    err = (o - ref).abs().max().item() / ref.abs().max().item()
    nz = (o != 0).float().mean().item()
    print(f"elem={elem} M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn} bn={bn} epi={epi}: rel={err:.3e} nonzero={nz:.3f}")
    if err > 1e-2 and VERB:
        print("  out[0,:8]", o[0, :8].tolist())
        print("  ref[0,:8]", ref[0, :8].tolist())
        print("  out[1,:8]", o[1, :8].tolist())
        print("  ref[1,:8]", ref[1, :8].tolist())
        # find relation: is out = ref permuted?
        print("  out[8,:4]", o[8, :4].tolist(), "ref[8,:4]", ref[8, :4].tolist())


for elem in (4, 2):
    bk = 128 // elem
    case(elem, 128, 64, bk, 0, 0, 64)
    case(elem, 128, 64, 4 * bk, 0, 0, 64)
    case(elem, 128, 128, 4 * bk, 0, 0, 128)
    case(elem, 128, 256, 4 * bk, 0, 0, 256)
    case(elem, 128, 64, 4 * bk, 0, 1, 64)
    case(elem, 128, 64, 4 * bk, 1, 1, 64)
    case(elem, 300, 200, 100, 0, 1, 64)
    case(elem, 300, 200, 100, 1, 1, 128)
    case(elem, 300, 200, 100, 0, 0, 0, epi=0, relu=1)
