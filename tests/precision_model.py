"""Operand-precision model of the device path (test helper).

The tensor-core GEMMs consume bf16 (kind::f16) or tf32-rounded fp32 (kind::tf32)
operands. Near a ReLU kink the sign of a pre-activation can differ between an
fp64 reference and any reduced-precision evaluation, which moves whole rows of
the backward pass — so raw gradients of the device are compared here against
the reference algorithm (model.cpp:54-62,110-120,192-244, restated in fp64 numpy)
evaluated on *the operands the device actually sees*: every value the device
rounds before a GEMM (features, weight shadow, stored activations, stored dZ)
is rounded identically here; all arithmetic is fp64. What remains is fp32
accumulation order on the device (~1e-7 relative).

Used only by tests (it is a checker, not a product path).
"""
import numpy as np


def tf32_rna(a):
    """cvt.rna.tf32.f32: round to nearest, ties away from zero, keep 10 mantissa bits."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def bf16_rn(a):
    """__float2bfloat16_rn: round to nearest even."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def _blocks(dims, w):
    out, off = [], 0
    for l in range(len(dims) - 1):
        fi, fo = dims[l], dims[l + 1]
        W = w[off:off + fi * fo].reshape(fi, fo)  # flat block = W^T ([in][out])
        b = w[off + fi * fo: off + fi * fo + fo]
        out.append((W, b, off))
        off += fi * fo + fo
    return out


def ranking_coef(s, y):
    """gs / pairs of model.cpp:71-106 (vectorised, fp64)."""
    n = len(s)
    if n == 0:
        return np.zeros(0), 0.0, 0
    d = s[:, None] - s[None, :]
    hi = y[:, None] > y[None, :]
    sig = 1.0 / (1.0 + np.exp(d))  # sigma(-(s_i - s_j)) for i hi over j
    pairs = int(hi.sum())
    if pairs == 0:
        return np.zeros(n), 0.0, 0
    gs = -(sig * hi).sum(1) + (sig * hi).sum(0)
    loss = np.logaddexp(0.0, -d)[hi].sum() / pairs
    return gs / pairs, loss, pairs


def _sigmoid(v):
    return 0.5 * (1.0 + np.tanh(0.5 * v))


def _softplus(v):
    return np.logaddexp(0.0, v)


def device_forward(dims, w64, x, mode):
    """Scores and stored activations as the device produces them."""
    rnd, w, f32_ = _mode(mode, w64)
    L = len(dims) - 1
    blocks = _blocks(dims, w)
    ops = [(rnd(W), b) for (W, b, _) in blocks[:-1]]
    acts = [rnd(f32_(x))]
    h = acts[0]
    for l in range(L - 1):
        z = h @ ops[l][0] + ops[l][1]
        hv = np.maximum(f32_(z), 0.0)
        if l == L - 2:
            h_full = hv
            stored = bf16_rn(hv) if mode == "bf16" else hv
        else:
            stored = rnd(hv)
        acts.append(stored)
        h = stored
    wh, bh, _ = blocks[-1]
    s = f32_(h_full @ wh[:, 0] + bh[0])
    return s, h_full, acts, ops, blocks


def _mode(mode, w64):
    rnd = {"tf32": tf32_rna, "bf16": bf16_rn, "none": lambda a: np.asarray(a, np.float64)}[mode]
    w = f32(w64) if mode != "none" else np.asarray(w64, np.float64)
    f32_ = f32 if mode != "none" else (lambda a: np.asarray(a, np.float64))
    return rnd, w, f32_


def device_gradients(dims, w64, x, y, mode, adv=None, beta=0.0):
    """Gradient of model.cpp:192-244 as the device computes it (mode 'tf32', 'bf16' or 'none').

    adv = (u, c, replay): replay rows go first (rows [0, m)), like the device layout."""
    rnd, w, f32_ = _mode(mode, w64)
    active = adv is not None and beta != 0.0 and len(y) > 0
    n = len(y)
    m = len(adv[2]) if active else 0
    xs = np.vstack([adv[2], x]) if active else np.asarray(x, np.float64)
    s_all, h_full, acts, ops, blocks = device_forward(dims, w64, xs, mode)
    L = len(dims) - 1
    wh, bh, offh = blocks[-1]
    s = s_all[m:]
    coef_b, loss, pairs = ranking_coef(s, np.asarray(y, np.float64))
    coefA = np.concatenate([np.zeros(m), f32_(coef_b)])
    coefB = np.zeros(m + n)
    u = None
    if active:
        u = f32_(adv[0])
        z = f32_(h_full @ u + f32_(adv[1]))
        coefB[:m] = f32_(0.5 * beta * _sigmoid(-z[:m]) / m)
        coefB[m:] = f32_(-0.5 * beta * _sigmoid(z[m:]) / n)
        ce = 0.5 * (_softplus(-z[:m]).mean() + _softplus(z[m:]).mean())
        loss += beta * -ce
    g = np.zeros(len(w))
    Hst = acts[-1]
    g[offh:offh + dims[L - 1]] = coefA @ Hst
    g[offh + dims[L - 1]] = coefA.sum()
    v = np.outer(coefA, wh[:, 0])
    if u is not None:
        v = v + np.outer(coefB, u)
    dz = rnd(f32_(v) * (Hst > 0))
    for l in range(L - 2, -1, -1):
        Wop, _ = ops[l]
        _, _, off = blocks[l]
        fi, fo = dims[l], dims[l + 1]
        g[off:off + fi * fo] = (acts[l].T @ dz).reshape(-1)
        g[off + fi * fo: off + fi * fo + fo] = dz.sum(0)
        if l > 0:
            dh = dz @ Wop.T
            dz = rnd(f32_(dh) * (acts[l] > 0))
    return g, loss


def device_gradients_pooled(dims, w64, x, offsets, y, mode):
    """Pooled (TenSet-shaped) gradient as the device computes it: statement rows, CSR program offsets."""
    rnd, w, f32_ = _mode(mode, w64)
    off = np.asarray(offsets, np.int64)
    P = len(off) - 1
    s_rows, h_full, acts, ops, blocks = device_forward(dims, w64, x, mode)
    L = len(dims) - 1
    wh, bh, offh = blocks[-1]
    dots = h_full @ wh[:, 0]
    s = np.array([dots[off[q]:off[q + 1]].sum() for q in range(P)]) + bh[0]
    coef_p, loss, _ = ranking_coef(f32_(s), np.asarray(y, np.float64))
    coef_p = f32_(coef_p)
    seg = np.repeat(np.arange(P), np.diff(off))
    coefA = coef_p[seg]
    g = np.zeros(len(w))
    Hst = acts[-1]
    g[offh:offh + dims[L - 1]] = coefA @ Hst
    g[offh + dims[L - 1]] = coef_p.sum()
    dz = rnd(f32_(np.outer(coefA, wh[:, 0])) * (Hst > 0))
    for l in range(L - 2, -1, -1):
        Wop, _ = ops[l]
        _, _, o = blocks[l]
        fi, fo = dims[l], dims[l + 1]
        g[o:o + fi * fo] = (acts[l].T @ dz).reshape(-1)
        g[o + fi * fo: o + fi * fo + fo] = dz.sum(0)
        if l > 0:
            dz = rnd(f32_(dz @ Wop.T) * (acts[l] > 0))
    return g, loss


def nrel(got, ref):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))
