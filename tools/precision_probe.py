"""Measure each operand precision's error against the fp64 oracle on the benched shapes.

cfg2: pooled {164,512,512,512,512,1}, 512 programs (synth_offsets, ~2.3K statements):
predictions, loss, gradient and the 3-step momentum-SGD update delta (w_after - w_before).
cfg4: {164,512,512,1} predictions over a 100K-program pool + rank agreement.
Prints one JSON object per (config, precision)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from paper_2201_05752_b200 import moseslab as ml  # noqa: E402
import oracle as orc  # noqa: E402


def nrel(got, ref):
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


def frob(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def pooled_scores_ref(dims, w, x, off):
    _, h = orc.forward(dims, w, x, threads=16)
    hp = orc.segment_sum(h, off)
    H = dims[-2]
    o = ml.param_count(dims) - (H + 1)
    return hp @ w[o:o + H] + w[o + H]


def cfg2(precs, steps=3):
    dims = [164, 512, 512, 512, 512, 1]
    p = ml.init_random(dims, 12345, strict=False)
    off = ml.synth_offsets(1, 512, 8)
    x = np.random.default_rng(1).random((int(off[-1]), 164))
    y = 0.1 + np.random.default_rng(2).random(512)
    s_ref = pooled_scores_ref(dims, p.params, x, off)
    g_ref, loss_ref = orc.gradients_pooled(dims, p.params, x, off, y, threads=16)
    w64, m64 = p.params.copy(), np.zeros_like(p.params)
    for _ in range(steps):
        g, _ = orc.gradients_pooled(dims, w64, x, off, y, threads=16)
        m64 = 0.9 * m64 + g
        w64 = w64 - 0.001 * m64
    dw_ref = w64 - p.params
    for name, prec in precs:
        dm = ml.DeviceModel(p, prec, int(off[-1]) + 128)
        s = ml.predict_pooled(dm, x, off)
        g, loss = ml.gradients_pooled(dm, x, off, y, want_loss=True)
        dm.upload(p)
        for _ in range(steps):
            ml.gradients_pooled(dm, x, off, y)
            ml.apply_update(dm, ml.TrainHyper(learning_rate=0.001, momentum=0.9), None, True)
        dw = dm.download().params - p.params
        print(json.dumps({"cfg": "cfg2", "prec": name, "rows": int(off[-1]), "pred_nrel": nrel(s, s_ref),
                          "loss_rel": abs(loss - loss_ref) / abs(loss_ref), "grad_nrel": nrel(g, g_ref),
                          "grad_frob": frob(g, g_ref), "dw_nrel": nrel(dw, dw_ref), "dw_frob": frob(dw, dw_ref)}),
              flush=True)


def cfg4(precs, n=100_000):
    dims = [164, 512, 512, 1]
    p = ml.init_random(dims, 12345)
    x = np.random.default_rng(3).random((n, 164))
    t = time.time()
    s_ref, _ = orc.forward(dims, p.params, x, threads=16)
    t_ref = time.time() - t
    order = np.argsort(s_ref)
    for name, prec in precs:
        dm = ml.DeviceModel(p, prec, 65536)
        s = ml.predict(dm, x)
        e = nrel(s, s_ref)
        # rank agreement over adjacent pairs of the reference order whose gap exceeds 2 * e * max|ref|
        a, b = order[:-1], order[1:]
        gap = s_ref[b] - s_ref[a]
        tol = 2 * e * np.max(np.abs(s_ref))
        sel = gap > tol
        flips = int(np.sum(s[b][sel] <= s[a][sel]))
        top_ref = orc.topk(s_ref, 1024)
        top = ml.topk(s, 1024)
        print(json.dumps({"cfg": "cfg4", "prec": name, "n": n, "pred_nrel": e, "pred_frob": frob(s, s_ref),
                          "adjacent_pairs_checked": int(sel.sum()), "flips": flips,
                          "top1024_overlap": len(set(top_ref.tolist()) & set(top.tolist())),
                          "oracle_s": t_ref}), flush=True)


if __name__ == "__main__":
    precs = [("bf16", ml.PREC_BF16), ("tf32", ml.PREC_TF32), ("fp32", ml.PREC_FP32), ("bf16x3", ml.PREC_BF16X3)]
    cfg2(precs)
    cfg4(precs)
