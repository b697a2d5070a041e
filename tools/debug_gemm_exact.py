"""Raw GEMM cases on tf32/bf16-exact inputs vs fp64: any error > ~1e-5 is a layout bug."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2201_05752_b200 import moseslab as ml
from precision_model import tf32_rna, bf16_rn
L = ml.lib()

def case(elem, M, N, K, a_mn, b_mn, bn, seed=0):
    rng = np.random.default_rng(seed)
    rnd = tf32_rna if elem == 4 else bf16_rn
    A = rnd(rng.normal(0, 1, (M, K)))
    B = rnd(rng.normal(0, 1, (N, K)))
    ref = A @ B.T
    dt = torch.float32 if elem == 4 else torch.bfloat16
    pad = 16 // elem
    if a_mn:
        lda = (M + pad - 1) // pad * pad
        As = torch.zeros((K, lda), dtype=torch.float64); As[:, :M] = torch.from_numpy(A.T)
    else:
        lda = (K + pad - 1) // pad * pad
        As = torch.zeros((M, lda), dtype=torch.float64); As[:, :K] = torch.from_numpy(A)
    if b_mn:
        ldb = (N + pad - 1) // pad * pad
        Bs = torch.zeros((K, ldb), dtype=torch.float64); Bs[:, :N] = torch.from_numpy(B.T)
    else:
        ldb = (K + pad - 1) // pad * pad
        Bs = torch.zeros((N, ldb), dtype=torch.float64); Bs[:, :K] = torch.from_numpy(B)
    As = As.to(dt).cuda(); Bs = Bs.to(dt).cuda()
    out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    rc = L.moses_debug_gemm(elem, M, N, K, As.data_ptr(), lda, a_mn, Bs.data_ptr(), ldb, b_mn, 2, out.data_ptr(), N,
                            None, 0, bn, None, 0)
    assert rc == 0, L.moses_last_error()
    o = out.cpu().double().numpy()
    err = np.abs(o - ref).max() / np.abs(ref).max()
    bad = np.argwhere(np.abs(o - ref) > 1e-4 * np.abs(ref).max())
    print(f"elem={elem} M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn} bn={bn}: rel={err:.2e} bad={len(bad)}"
          + (f" first bad {bad[:3].tolist()} rows {sorted(set(bad[:,0].tolist()))[:8]} cols {sorted(set(bad[:,1].tolist()))[:8]}" if len(bad) else ""))

for elem in (4, 2):
    for (M, N, K) in ((128, 64, 128), (256, 128, 256), (513, 512, 512), (165, 512, 512), (512, 512, 512), (512, 512, 40), (300, 200, 100)):
        for a_mn, b_mn in ((0, 0), (0, 1), (1, 1)):
            for bn in (64, 128, 256):
                case(elem, M, N, K, a_mn, b_mn, bn)
