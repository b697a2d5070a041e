"""The tcgen05 GEMM kernels on bf16/tf32-representable inputs against fp64: with exact operands the
only error is fp32 accumulation, so anything above ~1e-5 relative is a layout/pipeline bug.
Covers K-/MN-major operands, all N tiles, ragged M/N/K, and the persistent double-buffered kernel."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(ml, elem, M, N, K, a_mn, b_mn, bn, epi=2, seed=0):
    import torch

    from precision_model import bf16_rn, tf32_rna

    L = ml.lib()
    rng = np.random.default_rng(seed)
    rnd = tf32_rna if elem == 4 else bf16_rn
    A = rnd(rng.normal(0, 1, (M, K)))
    B = rnd(rng.normal(0, 1, (N, K)))
    ref = A @ B.T
    dt = torch.float32 if elem == 4 else torch.bfloat16
    pad = 16 // elem
    rp = lambda v: (v + pad - 1) // pad * pad
    if a_mn:
        As = torch.zeros((K, rp(M)), dtype=torch.float64); As[:, :M] = torch.from_numpy(A.T); lda = rp(M)
    else:
        As = torch.zeros((M, rp(K)), dtype=torch.float64); As[:, :K] = torch.from_numpy(A); lda = rp(K)
    if b_mn:
        Bs = torch.zeros((K, rp(N)), dtype=torch.float64); Bs[:, :N] = torch.from_numpy(B.T); ldb = rp(N)
    else:
        Bs = torch.zeros((N, rp(K)), dtype=torch.float64); Bs[:, :K] = torch.from_numpy(B); ldb = rp(K)
    As, Bs = As.to(dt).cuda(), Bs.to(dt).cuda()
    mask = None
    if epi == 2:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        bias = None
    elif epi == 1:  # ReLU'-masked store
        out = torch.zeros((M, rp(N)), dtype=dt, device="cuda")
        bias = None
        mk = (rng.random((M, N)) < 0.5).astype(np.float64) * rng.random((M, N))
        mask = torch.zeros((M, rp(N)), dtype=torch.float64)
        mask[:, :N] = torch.from_numpy(mk)
        mask = mask.to(dt).cuda()
        ref = ref * (mk > 0)
    else:
        out = torch.zeros((M, rp(N)), dtype=dt, device="cuda")
        bias = torch.from_numpy(rng.normal(0, 1, rp(N)).astype(np.float32)).cuda()
        ref = np.maximum(ref + bias.cpu().numpy()[:N].astype(np.float64), 0.0)
    rc = L.moses_debug_gemm(elem, M, N, K, As.data_ptr(), lda, a_mn, Bs.data_ptr(), ldb, b_mn, epi, out.data_ptr(),
                            out.shape[1], None if bias is None else bias.data_ptr(), 1 if epi == 0 else 0, bn,
                            None if mask is None else mask.data_ptr(), 0 if mask is None else mask.shape[1])
    assert rc == 0, L.moses_last_error()
    o = out.float().cpu().double().numpy()[:, :N]
    tol = 1e-5 if epi == 2 else (2 ** -8 if elem == 2 else 2 ** -10)  # epi 0 stores rounded outputs
    err = np.abs(o - ref).max() / np.abs(ref).max()
    assert err < tol, (elem, M, N, K, a_mn, b_mn, bn, err)


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    assert moseslab.lib().moses_device_check() == 0
    return moseslab


@pytest.mark.parametrize("elem", [2, 4])
@pytest.mark.parametrize("shape", [(128, 64, 128), (513, 512, 512), (165, 512, 300), (300, 200, 100), (7, 40, 9)])
@pytest.mark.parametrize("majors", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("bn", [64, 128, 256])
def test_gemm_exact(ml, elem, shape, majors, bn):
    _case(ml, elem, *shape, *majors, bn)


@pytest.mark.parametrize("elem", [2, 4])
@pytest.mark.parametrize("majors,epi", [((0, 1), 0), ((0, 0), 0), ((0, 0), 2), ((0, 1), 2)])
def test_persistent_gemm_exact(ml, elem, majors, epi):
    """M large enough for the persistent kernel (>= 2 tiles per SM), incl. a ragged last tile."""
    _case(ml, elem, 65536 + 77, 512, 512 if elem == 2 else 256, *majors, 0, epi)
    _case(ml, elem, 40000, 200, 100, *majors, 0, epi)


@pytest.mark.parametrize("M", [7, 300, 2304, 70000 + 5])
@pytest.mark.parametrize("K", [164, 512])
@pytest.mark.parametrize("b_mn,epi", [(1, 0), (0, 0), (0, 1)])
def test_cluster_gemm_exact(ml, M, K, b_mn, epi):
    """N = 512 bf16 hidden-layer shapes route to the weight-resident 4-CTA multicast kernel."""
    _case(ml, 2, M, 512, K, 0, b_mn, 0, epi, seed=M + K)
