"""ctypes view of the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg. The product package
(paper_2201_05752_b200) never imports this module.

Every function mirrors a reference symbol; see moses_oracle.hpp for the
file:line each one restates.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")

# moseslab::ErrorCode ordinals (errors.hpp:10-36)
ERROR_NAMES = [
    "invalid-task", "invalid-config", "space-too-large", "immutable-space", "bad-dims",
    "dim-mismatch", "shape-mismatch", "version-mismatch", "corrupt-stream", "empty-dataset",
    "invalid-ratio", "unnormalized-threshold", "adversary-disabled", "unstable-decay",
    "infeasible-split", "zero-mean", "insufficient-batches", "budget-infeasible",
    "missing-reference-strategy", "mismatched-runs", "empty-rows", "parse-error",
    "missing-field", "io-error", "usage-error",
]

THRESHOLD, RATIO = 1, 2


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = ERROR_NAMES[code - 1] if 1 <= code <= len(ERROR_NAMES) else f"status-{code}"
        super().__init__(f"{self.code}: {msg}")


def build() -> str:
    if not os.path.exists(_SO) or any(
        os.path.getmtime(os.path.join(_HERE, f)) > os.path.getmtime(_SO)
        for f in ("moses_oracle.hpp", "oracle_capi.cpp")
    ):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build() if not os.path.exists(_SO) else None
        _lib = C.CDLL(_SO)
        _lib.orc_last_error.restype = C.c_char_p
        vp, ci, cd = C.c_void_p, C.c_int, C.c_double
        _lib.orc_mmd2_grad_f64.argtypes = [vp, ci, vp, ci, ci, cd, vp, vp, vp]
        _lib.orc_gradients_mmd_f64.argtypes = [vp, ci, vp, vp, vp, ci, vp, ci, cd, cd, vp, vp, ci]
        _lib.orc_gradients_from_score_grads_f64.argtypes = [vp, ci, vp, vp, ci, vp, vp, ci]
        for name in ("orc_splitmix_draw", "orc_splitmix_at", "orc_fnv_u64s", "orc_fnv_str", "orc_fnv_u64_str"):
            getattr(_lib, name).restype = C.c_uint64
        _lib.orc_splitmix_draw.argtypes = [C.c_uint64, C.c_int]
        _lib.orc_splitmix_at.argtypes = [C.c_uint64, C.c_uint64]
        _lib.orc_fnv_u64_str.argtypes = [C.c_uint64, C.c_char_p]
        _lib.orc_fnv_u64s.argtypes = [C.c_void_p, C.c_int]
        _lib.orc_fnv_str.argtypes = [C.c_char_p]
        _lib.orc_param_count.argtypes = [C.c_void_p, C.c_int]
        _lib.orc_uniform01_first.restype = C.c_double
        _lib.orc_uniform01_first.argtypes = [C.c_uint64]
        _lib.orc_gaussian_first.restype = C.c_double
        _lib.orc_gaussian_first.argtypes = [C.c_uint64]
        for name in ("orc_param_count", "orc_ranking_terms_f64", "orc_ranking_terms_f32", "orc_ratio_keep",
                     "orc_serialize", "orc_write_mask_bytes"):
            getattr(_lib, name).restype = C.c_longlong
        _lib.orc_ratio_keep.argtypes = [C.c_double, C.c_longlong]
        _lib.orc_init_random.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_int, C.c_void_p]
        for s in ("f64", "f32"):
            rt = C.c_double if s == "f64" else C.c_float
            getattr(_lib, f"orc_forward_{s}").argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                                         C.c_void_p, C.c_void_p, C.c_int]
            getattr(_lib, f"orc_ranking_terms_{s}").argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                                               C.c_void_p]
            getattr(_lib, f"orc_accuracy_counts_{s}").argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                                                 C.c_void_p]
            getattr(_lib, f"orc_disc_ce_{s}").argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
            getattr(_lib, f"orc_disc_ce_{s}").restype = rt
            getattr(_lib, f"orc_mmd2_{s}").restype = rt
            getattr(_lib, f"orc_mmd2_{s}").argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, rt]
            getattr(_lib, f"orc_gradients_{s}").argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                                           C.c_int, C.c_void_p, rt, C.c_void_p, C.c_int, rt,
                                                           C.c_void_p, C.c_void_p, C.c_int]
            getattr(_lib, f"orc_objective_{s}").argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                                           C.c_int, C.c_void_p, rt, C.c_void_p, C.c_int, rt,
                                                           C.c_void_p]
            getattr(_lib, f"orc_apply_update_{s}").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong,
                                                              C.c_double, C.c_double, C.c_void_p, C.c_int]
            getattr(_lib, f"orc_xi_{s}").argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_int, C.c_void_p]
            getattr(_lib, f"orc_partition_{s}").argtypes = [C.c_void_p, C.c_longlong, C.c_int, C.c_int, C.c_double,
                                                            C.c_void_p]
            getattr(_lib, f"orc_variant_decay_{s}").argtypes = [C.c_void_p, C.c_longlong, C.c_void_p, C.c_double,
                                                               C.c_double]
            getattr(_lib, f"orc_adversarial_term_{s}").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                                                  C.c_void_p, C.c_int, C.c_int, rt, C.c_void_p]
            getattr(_lib, f"orc_topk_{s}").argtypes = [C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p]
            getattr(_lib, f"orc_segment_sum_{s}").argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_longlong,
                                                             C.c_void_p]
            getattr(_lib, f"orc_adam_{s}").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong,
                                                      C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double,
                                                      C.c_int]
        _lib.orc_gradients_pooled_f64.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                                  C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _lib.orc_synth_features.argtypes = [C.c_uint64, C.c_longlong, C.c_longlong, C.c_int, C.c_void_p]
        _lib.orc_measure_configs.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_char_p, C.c_void_p, C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_longlong,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_true_best.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                       C.c_void_p, C.c_void_p]
        _lib.orc_encode_configs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_uint64,
                                            C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_synth_labels.argtypes = [C.c_uint64, C.c_longlong, C.c_longlong, C.c_void_p]
        _lib.orc_synth_offsets.argtypes = [C.c_uint64, C.c_longlong, C.c_int, C.c_void_p]
        _lib.orc_serialize.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong]
        _lib.orc_write_mask_bytes.argtypes = [C.c_void_p, C.c_longlong, C.c_uint, C.c_int, C.c_double, C.c_void_p,
                                              C.c_longlong]
        _lib.orc_train_step_f64.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _sfx(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def _dims(dims):
    return np.ascontiguousarray(dims, dtype=np.int32)


# ---------------------------------------------------------------- rng
def splitmix_draw(seed: int, k: int) -> int:
    return lib().orc_splitmix_draw(seed, k)


def uniform01_first(seed: int) -> float:
    return lib().orc_uniform01_first(seed)


def gaussian_first(seed: int) -> float:
    return lib().orc_gaussian_first(seed)


def fnv_u64s(vals) -> int:
    a = np.ascontiguousarray(vals, dtype=np.uint64)
    return lib().orc_fnv_u64s(_p(a), len(a))


def fnv_str(s: str) -> int:
    return lib().orc_fnv_str(s.encode())


# ---------------------------------------------------------------- model
def param_count(dims) -> int:
    d = _dims(dims)
    return lib().orc_param_count(_p(d), len(d))


def init_random(dims, seed: int, strict: bool = True) -> np.ndarray:
    d = _dims(dims)
    out = np.zeros(param_count(dims), dtype=np.float64)
    _check(lib().orc_init_random(_p(d), len(d), seed, int(strict), _p(out)))
    return out


def forward(dims, w, x, threads: int = 1):
    """Returns (scores n, penultimate n x dims[-2])."""
    d = _dims(dims)
    w = np.ascontiguousarray(w)
    x = np.ascontiguousarray(x, dtype=w.dtype)
    n = x.shape[0]
    s = np.zeros(n, dtype=w.dtype)
    h = np.zeros((n, dims[-2]), dtype=w.dtype)
    _check(getattr(lib(), f"orc_forward_{_sfx(w.dtype)}")(_p(d), len(d), _p(w), _p(x), n, _p(s), _p(h), threads))
    return s, h


def ranking_terms(scores, labels):
    s = np.ascontiguousarray(scores)
    y = np.ascontiguousarray(labels, dtype=s.dtype)
    loss = np.zeros(1, dtype=s.dtype)
    gs = np.zeros(len(s), dtype=s.dtype)
    pairs = getattr(lib(), f"orc_ranking_terms_{_sfx(s.dtype)}")(_p(s), _p(y), len(s), _p(loss), _p(gs))
    return float(loss[0]), gs, pairs


def gradients(dims, w, x, y, adv=None, beta=0.0, want_loss=True, threads=1):
    """adv = (weight, bias, replay) or None. Returns (g_flat, loss)."""
    d = _dims(dims)
    w = np.ascontiguousarray(w)
    dt = w.dtype
    x = np.ascontiguousarray(x, dtype=dt)
    y = np.ascontiguousarray(y, dtype=dt)
    g = np.zeros_like(w)
    loss = np.zeros(1, dtype=dt)
    rt = C.c_double if dt == np.float64 else C.c_float
    if adv is not None:
        aw = np.ascontiguousarray(adv[0], dtype=dt)
        rep = np.ascontiguousarray(adv[2], dtype=dt)
        args = (_p(aw), rt(adv[1]), _p(rep), rep.shape[0])
    else:
        args = (None, rt(0.0), None, 0)
    _check(getattr(lib(), f"orc_gradients_{_sfx(dt)}")(_p(d), len(d), _p(w), _p(x), _p(y), x.shape[0], *args,
                                                      rt(beta), _p(g), _p(loss) if want_loss else None, threads))
    return g, float(loss[0])


def gradients_pooled(dims, w, x, offsets, y, threads=1):
    """Statement rows x, CSR program offsets, per-program labels y -> (g_flat, loss), fp64."""
    d = _dims(dims)
    w = np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    g = np.zeros_like(w)
    loss = np.zeros(1)
    _check(lib().orc_gradients_pooled_f64(_p(d), len(d), _p(w), _p(x), x.shape[0], _p(off), len(off) - 1, _p(y),
                                          _p(g), _p(loss), threads))
    return g, float(loss[0])


def gradients_from_score_grads(dims, w, x, gs, threads=1):
    """gradients() with a caller-supplied score gradient (model.cpp:201-244 after ranking_terms), fp64."""
    d = _dims(dims)
    w = np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    gs = np.ascontiguousarray(gs, dtype=np.float64)
    g = np.zeros_like(w)
    _check(lib().orc_gradients_from_score_grads_f64(_p(d), len(d), _p(w), _p(x), x.shape[0], _p(gs), _p(g), threads))
    return g


def mmd2_grad(xs, xt, sigma):
    """Biased Gaussian MMD^2 and its gradient w.r.t. every source / target row (fp64)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    xt = np.ascontiguousarray(xt, dtype=np.float64)
    gs, gt = np.zeros_like(xs), np.zeros_like(xt)
    v = C.c_double()
    _check(lib().orc_mmd2_grad_f64(_p(xs), xs.shape[0], _p(xt), xt.shape[0], xs.shape[1], C.c_double(sigma),
                                   C.byref(v), _p(gs), _p(gt)))
    return v.value, gs, gt


def gradients_mmd(dims, w, x, y, src, beta, sigma, threads=1):
    """gradients() with beta * MMD^2(H_src, H_batch) as the domain term -> (g_flat, loss), fp64."""
    d = _dims(dims)
    w = np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    src = np.ascontiguousarray(src, dtype=np.float64)
    g = np.zeros_like(w)
    loss = C.c_double()
    _check(lib().orc_gradients_mmd_f64(_p(d), len(d), _p(w), _p(x), _p(y), x.shape[0], _p(src), src.shape[0],
                                       C.c_double(beta), C.c_double(sigma), _p(g), C.byref(loss), threads))
    return g, loss.value


def pair_terms_rows(s_global, y_global, r0, r1):
    """Pair terms of rows [r0, r1) against the whole batch (model.cpp:71-106's rule, each distinct-label
    pair's loss counted at its hi row): (unnormalised gs of those rows, loss sum, pair count)."""
    s = np.asarray(s_global, dtype=np.float64)
    y = np.asarray(y_global, dtype=np.float64)
    gs = np.zeros(r1 - r0)
    loss, pairs = 0.0, 0
    for i in range(r0, r1):
        hi = y[i] > y  # i is the hi row of (i, j)
        lo = y[i] < y
        d_hi = s[i] - s[hi]
        e = np.exp(-np.abs(d_hi))
        sig = np.where(d_hi >= 0, e / (1 + e), 1 / (1 + e))
        d_lo = s[lo] - s[i]
        e2 = np.exp(-np.abs(d_lo))
        sig2 = np.where(d_lo >= 0, e2 / (1 + e2), 1 / (1 + e2))
        gs[i - r0] = -sig.sum() + sig2.sum()
        loss += np.sum(np.where(d_hi >= 0, np.log1p(e), -d_hi + np.log1p(e)))
        pairs += int(hi.sum())
    return gs, loss, pairs


def objective(dims, w, x, y, adv=None, beta=0.0):
    d = _dims(dims)
    w = np.ascontiguousarray(w)
    dt = w.dtype
    x = np.ascontiguousarray(x, dtype=dt)
    y = np.ascontiguousarray(y, dtype=dt)
    out = np.zeros(1, dtype=dt)
    rt = C.c_double if dt == np.float64 else C.c_float
    if adv is not None:
        aw = np.ascontiguousarray(adv[0], dtype=dt)
        rep = np.ascontiguousarray(adv[2], dtype=dt)
        args = (_p(aw), rt(adv[1]), _p(rep), rep.shape[0])
    else:
        args = (None, rt(0.0), None, 0)
    _check(getattr(lib(), f"orc_objective_{_sfx(dt)}")(_p(d), len(d), _p(w), _p(x), _p(y), x.shape[0], *args,
                                                      rt(beta), _p(out)))
    return float(out[0])


def apply_update(w, mom, g, lr, mu=0.9, mask=None, use_momentum=False):
    """In place on copies; returns (w, mom)."""
    w = np.array(w, copy=True)
    mom = np.array(mom, copy=True, dtype=w.dtype)
    g = np.ascontiguousarray(g, dtype=w.dtype)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    getattr(lib(), f"orc_apply_update_{_sfx(w.dtype)}")(_p(w), _p(mom), _p(g), len(w), lr, mu, _p(m),
                                                        int(use_momentum))
    return w, mom


def xi_scores(w, g, normalize):
    w = np.ascontiguousarray(w)
    g = np.ascontiguousarray(g, dtype=w.dtype)
    out = np.zeros_like(w)
    getattr(lib(), f"orc_xi_{_sfx(w.dtype)}")(_p(w), _p(g), len(w), int(normalize), _p(out))
    return out


def partition(xi, normalized, mode, value):
    xi = np.ascontiguousarray(xi)
    out = np.zeros(len(xi), dtype=np.uint8)
    _check(getattr(lib(), f"orc_partition_{_sfx(xi.dtype)}")(_p(xi), len(xi), int(normalized), mode, value, _p(out)))
    return out.astype(bool)


def ratio_keep(value, n):
    return lib().orc_ratio_keep(value, n)


def variant_decay(w, mask, alpha, lam):
    w = np.array(w, copy=True)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    _check(getattr(lib(), f"orc_variant_decay_{_sfx(w.dtype)}")(_p(w), len(w), _p(m), alpha, lam))
    return w


def accuracy_counts(scores, labels):
    s = np.ascontiguousarray(scores)
    y = np.ascontiguousarray(labels, dtype=s.dtype)
    pairs = C.c_longlong(0)
    conc = C.c_longlong(0)
    getattr(lib(), f"orc_accuracy_counts_{_sfx(s.dtype)}")(_p(s), _p(y), len(s), C.byref(pairs), C.byref(conc))
    return pairs.value, conc.value


def disc_ce(zs, zt):
    zs = np.ascontiguousarray(zs)
    zt = np.ascontiguousarray(zt, dtype=zs.dtype)
    return getattr(lib(), f"orc_disc_ce_{_sfx(zs.dtype)}")(_p(zs), len(zs), _p(zt), len(zt))


def adversarial_term(weight, bias, hs, ht, step=0.1):
    """Returns (new_weight, new_bias, discriminator_loss)."""
    aw = np.array(weight, copy=True)
    dt = aw.dtype
    rt = C.c_double if dt == np.float64 else C.c_float
    ab = np.array([bias], dtype=dt)
    hs = np.ascontiguousarray(hs, dtype=dt)
    ht = np.ascontiguousarray(ht, dtype=dt)
    loss = np.zeros(1, dtype=dt)
    _check(getattr(lib(), f"orc_adversarial_term_{_sfx(dt)}")(_p(aw), _p(ab), _p(hs), hs.shape[0], _p(ht),
                                                              ht.shape[0], len(aw), rt(step), _p(loss)))
    return aw, float(ab[0]), float(loss[0])


def topk(scores, k):
    s = np.ascontiguousarray(scores)
    k = min(k, len(s))
    out = np.zeros(k, dtype=np.int64)
    getattr(lib(), f"orc_topk_{_sfx(s.dtype)}")(_p(s), len(s), k, _p(out))
    return out


def segment_sum(h, offsets):
    h = np.ascontiguousarray(h)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    out = np.zeros((len(off) - 1, h.shape[1]), dtype=h.dtype)
    getattr(lib(), f"orc_segment_sum_{_sfx(h.dtype)}")(_p(h), h.shape[1], _p(off), len(off) - 1, _p(out))
    return out


def mmd2(xs, xt, sigma):
    xs = np.ascontiguousarray(xs)
    xt = np.ascontiguousarray(xt, dtype=xs.dtype)
    return getattr(lib(), f"orc_mmd2_{_sfx(xs.dtype)}")(_p(xs), xs.shape[0], _p(xt), xt.shape[0], xs.shape[1],
                                                       sigma)


def adam(w, m1, m2, g, lr, b1, b2, eps, t, mask=None):
    w, m1, m2 = (np.array(a, copy=True) for a in (w, m1, m2))
    g = np.ascontiguousarray(g, dtype=w.dtype)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    getattr(lib(), f"orc_adam_{_sfx(w.dtype)}")(_p(w), _p(m1), _p(m2), _p(g), len(w), _p(m), lr, b1, b2, eps, t)
    return w, m1, m2


def synth_features(seed, row0, rows, D):
    out = np.zeros((rows, D), dtype=np.float64)
    lib().orc_synth_features(seed, row0, rows, D, _p(out))
    return out


def synth_labels(seed, row0, rows):
    out = np.zeros(rows, dtype=np.float64)
    lib().orc_synth_labels(seed, row0, rows, _p(out))
    return out


def synth_offsets(seed, programs, max_stmts=8):
    out = np.zeros(programs + 1, dtype=np.int64)
    lib().orc_synth_offsets(seed, programs, max_stmts, _p(out))
    return out


def serialize(dims, w, mom=None):
    d = _dims(dims)
    w = np.ascontiguousarray(w, dtype=np.float64)
    mom = np.zeros_like(w) if mom is None else np.ascontiguousarray(mom, dtype=np.float64)
    n = lib().orc_serialize(_p(d), len(d), _p(w), _p(mom), None, 0)
    if n < 0:
        raise OracleError(-n, lib().orc_last_error().decode())
    buf = C.create_string_buffer(n)
    lib().orc_serialize(_p(d), len(d), _p(w), _p(mom), buf, n)
    return buf.raw


def write_mask_bytes(mask, phase, mode, value):
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    n = lib().orc_write_mask_bytes(_p(m), len(m), phase, mode, value, None, 0)
    buf = C.create_string_buffer(n)
    lib().orc_write_mask_bytes(_p(m), len(m), phase, mode, value, buf, n)
    return buf.raw


def train_step_f64(dims, w, mom, x, y, lr=0.001, mu=0.9, threads=1):
    """In place on w, mom (float64 arrays). Returns the batch loss."""
    d = _dims(dims)
    loss = np.zeros(1)
    _check(lib().orc_train_step_f64(_p(d), len(d), _p(w), _p(mom), _p(np.ascontiguousarray(x)),
                                    _p(np.ascontiguousarray(y)), x.shape[0], lr, mu, _p(loss), threads))
    return float(loss[0])


# ---------------------------------------------------------------- knob space (space.cpp:28-197)
TEMPLATE_ROLES = {"tile_x": 0, "tile_y": 1, "unroll": 2, "vectorize": 3, "parallel": 4}


def default_knob_template():
    """space.cpp:28-36 — (name, domain) of the 5 template knobs."""
    return [("tile_x", [1, 2, 4, 8, 16, 32, 64]), ("tile_y", [1, 2, 4, 8, 16, 32, 64]), ("unroll", [0, 16, 64, 512]),
            ("vectorize", [1, 2, 4, 8, 16]), ("parallel", [1, 2, 4, 8, 16, 32, 64, 128, 256])]


def encode_configs(task, knobs, first, n):
    """encode_features + config_hash over configs [first, first+n) of enumerate_configs' order.
    task = (work_gflops, bytes_per_unit, ideal_log2_tiles, ideal_log2_unroll); knobs = [(name, domain)].
    Returns (features n x 16 float64, hashes uint64, values n x nk int64)."""
    t = np.ascontiguousarray(task, dtype=np.float64)
    dom = np.ascontiguousarray([v for _, d in knobs for v in d], dtype=np.int64)
    sizes = np.ascontiguousarray([len(d) for _, d in knobs], dtype=np.int32)
    roles = np.ascontiguousarray([TEMPLATE_ROLES.get(k, -1) for k, _ in knobs], dtype=np.int32)
    f = np.zeros((n, 16))
    h = np.zeros(n, dtype=np.uint64)
    v = np.zeros((n, len(knobs)), dtype=np.int64)
    _check(lib().orc_encode_configs(_p(t), _p(dom), _p(sizes), _p(roles), len(knobs), first, n, _p(f), _p(h), _p(v)))
    return f, h, v


# ---------------------------------------------------------------- simulated hardware (oracle.cpp:33-105)
def _dev6(device):
    return np.ascontiguousarray([device["peak_gflops"], device["parallel_units"], device["vector_lanes"],
                                 device["cache_bytes"], device["measure_overhead_ms"], device["noise_std"]],
                                dtype=np.float64)


def _task4(task):
    if isinstance(task, dict):
        task = (task["work_gflops"], task["bytes_per_unit"], task["ideal_log2_tiles"], task["ideal_log2_unroll"])
    return np.ascontiguousarray(task, dtype=np.float64)


def _space(knobs):
    dom = np.ascontiguousarray([v for _, d in knobs for v in d], dtype=np.int64)
    sizes = np.ascontiguousarray([len(d) for _, d in knobs], dtype=np.int32)
    roles = np.ascontiguousarray([TEMPLATE_ROLES.get(k, -1) for k, _ in knobs], dtype=np.int32)
    return dom, sizes, roles


def measure_configs(device, task_id, task, knobs, seed, first, n):
    """clean_latency_ms and measure() over configs [first, first+n): (clean, throughput, latency, wall_cost)."""
    dom, sizes, roles = _space(knobs)
    out = [np.zeros(n) for _ in range(4)]
    _check(lib().orc_measure_configs(_p(_dev6(device)), int(device["repeats"]), device["id"].encode(),
                                     task_id.encode(), _p(_task4(task)), _p(dom), _p(sizes), _p(roles), len(knobs),
                                     seed, first, n, *(_p(o) for o in out)))
    return tuple(out)


def true_best(device, task, knobs):
    dom, sizes, roles = _space(knobs)
    v = np.zeros(len(knobs), dtype=np.int64)
    lat = np.zeros(1)
    _check(lib().orc_true_best(_p(_dev6(device)), _p(_task4(task)), _p(dom), _p(sizes), _p(roles), len(knobs),
                               _p(v), _p(lat)))
    return v.tolist(), float(lat[0])


# ---------------------------------------------------------------- training-data pipeline (data.cpp, tuner.cpp)
# Pure-Python restatement (independent of the C++ oracle and of the library): KeyBuilder / RngStream
# (rng.hpp), make_ranking_batches (data.cpp:128-164), sample_replay_features rows (data.cpp:166-183),
# generate_dataset (data.cpp:49-65), pretrain's epoch seed and epoch loop (tuner.cpp:130-156).
_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def key_builder(*parts) -> int:
    """KeyBuilder: FNV-1a over 8 little-endian bytes per integer, UTF-8 bytes + NUL per string."""
    h = 0xCBF29CE484222325
    for p in parts:
        data = (p.encode() + b"\0") if isinstance(p, str) else int(p & _M64).to_bytes(8, "little")
        for b in data:
            h = ((h ^ b) * 0x100000001B3) & _M64
    return h


class RngStream:
    def __init__(self, key: int):
        self.s = key & _M64

    def next_u64(self) -> int:
        self.s = (self.s + _GOLDEN) & _M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def below(self, n: int) -> int:
        t = ((1 << 64) - n) % n
        while True:
            r = self.next_u64()
            if r >= t:
                return r % n

    def uniform01(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53


def _shuffle_with(items, rng):  # data.cpp:16-22
    for i in range(len(items), 1, -1):
        j = rng.below(i)
        items[i - 1], items[j] = items[j], items[i - 1]


def epoch_seed(seed: int, epoch: int) -> int:  # tuner.cpp:136-139
    return key_builder(seed, "epoch", epoch)


def make_ranking_batches(record_task_ids, batch_size: int, seed: int):
    """data.cpp:128-164 over the records' task ids: ([(task_id, [row indices])...], dropped_singletons)."""
    if batch_size < 2:
        raise OracleError(2, "batch size must be at least 2")
    order = list(dict.fromkeys(record_task_ids))
    batches, dropped = [], 0
    for tid in order:
        rows = [i for i, t in enumerate(record_task_ids) if t == tid]
        _shuffle_with(rows, RngStream(key_builder(seed, "shuffle", tid)))
        for s in range(0, len(rows), batch_size):
            chunk = rows[s:s + batch_size]
            if len(chunk) < 2:
                dropped += 1
                continue
            batches.append((tid, chunk))
    _shuffle_with(batches, RngStream(key_builder(seed, "order")))
    return batches, dropped


def replay_rows(n_records: int, size: int, seed: int):  # data.cpp:166-183
    if n_records <= 0:
        raise OracleError(10, "empty record store")
    if size < 1:
        raise OracleError(2, "replay size must be positive")
    rows = list(range(n_records))
    _shuffle_with(rows, RngStream(key_builder(seed, "replay")))
    return rows[:min(n_records, size)]


def sample_config_indices(seed: int, task_id: str, knobs, samples: int):
    """generate_dataset's draws for one task (data.cpp:55-61, sample_config space.cpp:94-100) as
    enumeration indices (last knob fastest)."""
    rng = RngStream(key_builder(seed, "gen", task_id))
    out = []
    for _ in range(samples):
        idx = 0
        for _, dom in knobs:
            idx = idx * len(dom) + rng.below(len(dom))
        out.append(idx)
    return out


def generate_dataset(device, tasks, knobs, samples_per_task: int, seed: int):
    """data.cpp:49-65. tasks = [(task_id, task4)]. Returns a list of record dicts (the reference's
    MeasurementRecord fields) plus a 'features' entry (encode_features)."""
    recs, seq = [], 0
    for tid, task in tasks:
        for idx in sample_config_indices(seed, tid, knobs, samples_per_task):
            f, _, v = encode_configs(task, knobs, idx, 1)
            _, thr, lat, wall = measure_configs(device, tid, task, knobs, seed, idx, 1)
            recs.append({"task_id": tid, "values": [int(x) for x in v[0]], "throughput_gflops": float(thr[0]),
                         "latency_ms": float(lat[0]), "wall_cost_ms": float(wall[0]), "device_id": device["id"],
                         "seq": seq, "features": f[0]})
            seq += 1
    return recs


def pretrain_epoch(dims, w, mom, features, labels, batches, lr, mu=0.9, threads=1):
    """tuner.cpp:146-151: for each planned batch, gradients + momentum update (float64). Returns
    (w, mom, mean batch loss)."""
    losses = [train_step_f64(dims, w, mom, features[rows], labels[rows], lr, mu, threads) for _, rows in batches]
    acc = 0.0
    for x in losses:  # loss_sum += loss (tuner.cpp:148-150); Python's sum() would compensate
        acc += x
    return w, mom, (acc / len(losses) if losses else 0.0)


# ---------------------------------------------------------------- evolve (search.cpp:11-71)
def evolve(knobs, scorer, population=128, generations=4, mutation_count=4, survivors=32, epsilon_random=0.05,
           seed=0):
    """Pure-Python restatement of the GA: scorer(list of value lists) -> list of float scores.
    Returns [(values, score)] sorted by score desc then values asc (search.cpp:32-37)."""
    if population < 1 or mutation_count < 1 or survivors < 1:
        raise OracleError(2, "population, mutation_count and survivors must be positive")
    if generations < 0:
        raise OracleError(2, "generations must be non-negative")
    if survivors > population:
        raise OracleError(2, "survivors cannot exceed the population")
    if not (0.0 <= epsilon_random <= 1.0):
        raise OracleError(2, "epsilon_random must lie in [0,1]")
    rng = RngStream(key_builder(seed, "evolve"))
    doms = [list(d) for _, d in knobs]

    def sample():  # space.cpp:94-100
        return [d[rng.below(len(d))] for d in doms]

    def mutate(cfg):  # space.cpp:102-121
        mut = [k for k, d in enumerate(doms) if len(d) > 1]
        if not mut:
            raise OracleError(4, "every knob domain is a singleton")
        ki = mut[rng.below(len(mut))]
        old = doms[ki].index(cfg[ki])
        pick = rng.below(len(doms[ki]) - 1)
        if pick >= old:
            pick += 1
        out = list(cfg)
        out[ki] = doms[ki][pick]
        return out

    def score_all(cfgs):
        return sorted(zip(cfgs, scorer(cfgs)), key=lambda cs: (-cs[1], cs[0]))

    pop = score_all([sample() for _ in range(population)])
    for _ in range(generations):
        keep = min(survivors, len(pop))
        nxt = [list(pop[s][0]) for s in range(keep)]
        for s in range(keep):
            for _ in range(mutation_count):
                nxt.append(sample() if rng.uniform01() < epsilon_random else mutate(pop[s][0]))
        pop = score_all(nxt)
    return pop


# ---------------------------------------------------------------- online loop (tuner.cpp:158-286, controller.cpp)
def plan_split(total, p, q):  # controller.cpp:10-32
    if q < 2:
        raise OracleError(2, "need at least 2 batches")
    if total < q:
        raise OracleError(2, "total trials below the batch count")
    if not (p > 0.0) or p > 1.0:
        raise OracleError(2, "train fraction must lie in (0,1]")
    measured = int(math.floor(p * float(total) + 1e-9))
    if measured < q:
        raise OracleError(15, "infeasible split")
    base, rem = divmod(measured, q)
    return total - measured, [base + (1 if b < rem else 0) for b in range(q)]


def _seq_sum(values):
    """Left-to-right double accumulation like the reference's loops (Python >= 3.12's sum() of floats is
    compensated, which differs in the last bit)."""
    acc = 0.0
    for v in values:
        acc += v
    return acc


def batch_cv(means):  # controller.cpp:34-45
    mean = _seq_sum(means) / len(means)
    var = _seq_sum((v - mean) * (v - mean) for v in means) / len(means)
    return math.sqrt(var) / mean


def tune_task(strategy, ops, task_id, knobs, budget, seed):
    """Restatement of tune_task (tuner.cpp:158-286) with the model / measurement operations injected:
      ops.evolve(seed) -> [(values, score)] in search order (evolve(params, space, sp), search.cpp:73-80)
      ops.measure([values]) -> [(throughput, latency, wall_cost)] (oracle.cpp:65-88, seq unused by the noise)
      ops.make_adversary(replay_seed) (tuner.cpp:187-201)
      ops.moses_update(values_rows, labels, batch, use_adversary) (tuner.cpp:248-262)
      ops.vanilla_update(values_rows, labels) (tuner.cpp:263-266)
    strategy: 0 raw, 1 random-init, 2 pretrain-only, 3 vanilla-finetune, 4 moses. Returns a dict."""
    nk = len(knobs)
    recs, cvs, predicted = [], [], []
    wall, unspent, term, meas = 0.0, 0, -1, 0
    best_lat, best_cfg = math.inf, None
    means, terminated = [], False
    if strategy == 0:  # tuner.cpp:166-178
        cfg = [d[(len(d) - 1) // 2] for _, d in knobs]
        thr, lat, w = ops.measure([cfg])[0]
        return {"records": [(cfg, thr, lat, w)], "best_values": cfg, "best_latency": lat, "wall": w,
                "batch_means": [], "cvs": [], "termination_batch": -1, "measured": 1, "prediction": 0,
                "unspent": budget.trials_per_task - 1, "predicted": []}
    pred_trials, sizes = plan_split(budget.trials_per_task, budget.train_fraction, budget.num_batches)
    use_adv = strategy == 4 and budget.adversary
    if use_adv:
        ops.make_adversary(key_builder(seed, "replay", task_id))
    measured = set()
    for b in range(budget.num_batches):  # tuner.cpp:209-267
        want = sizes[b]
        if terminated:
            unspent += want
            continue
        pop = ops.evolve(key_builder(seed, "evolve", task_id, b))
        batch, taken = [], set()
        for vals, score in pop:  # select_batch (search.cpp:82-95)
            if len(batch) >= want:
                break
            h = fnv_u64s(vals)
            if h in measured or h in taken:
                continue
            taken.add(h)
            batch.append((list(vals), score))
        unspent += want - len(batch)
        if not batch:
            continue
        first = len(recs)
        out = ops.measure([v for v, _ in batch])
        for (vals, score), (thr, lat, w) in zip(batch, out):
            wall += w
            if lat < best_lat:
                best_lat, best_cfg = lat, vals
            measured.add(fnv_u64s(vals))
            recs.append((vals, thr, lat, w))
        meas += len(batch)
        means.append(_seq_sum(s for _, s in batch) / len(batch))  # should_terminate (controller.cpp:47-56)
        if not terminated and len(means) >= 3 and _seq_sum(means) != 0.0 and abs(batch_cv(means)) < budget.cv_threshold:
            terminated = True
        cvs.append(math.nan if len(means) < 2 or _seq_sum(means) == 0.0 else batch_cv(means))  # tuner.cpp:31-37
        if terminated and term < 0:
            term = len(means)
        if strategy == 2 or len(batch) < 2:
            continue
        rows = [r[0] for r in recs[first:]]
        labels = [r[1] for r in recs[first:]]
        if strategy == 4:
            ops.moses_update(rows, labels, b, use_adv and budget.adversary_beta != 0.0)
        else:
            ops.vanilla_update(rows, labels)
    pop = ops.evolve(key_builder(seed, "predict", task_id))  # tuner.cpp:271-279
    tail, taken = [], set()
    for vals, score in pop:
        if len(tail) >= pred_trials:
            break
        h = fnv_u64s(vals)
        if h in measured or h in taken:
            continue
        taken.add(h)
        tail.append(score)
    unspent += pred_trials - len(tail)
    if not recs:
        raise OracleError(2, "no configuration was measured")
    return {"records": recs, "best_values": best_cfg, "best_latency": best_lat, "wall": wall, "batch_means": means,
            "cvs": cvs, "termination_batch": term, "measured": meas, "prediction": len(tail), "unspent": unspent,
            "predicted": tail}
