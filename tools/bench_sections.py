"""Sub-benchmarks of bench.py (sections of its JSON line beside the cfg2 headline): HBM-roofline
kernels at L2-exceeding sizes, the cfg3 Moses fine-tune step and MMD, the candidate-generation /
simulated-hardware pipeline and the reference's offline pretrain flow (f2).
Imported by bench.py; every function takes the loaded moseslab module `ml`, its library `L` and the
measured peaks."""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIMS = [164, 512, 512, 512, 512, 1]
BATCH = 512
SEED_MODEL = 12345
MAX_STMTS = 8


def bench_hbm_kernels(ml, L, peaks):
    """HBM-roofline kernels of the north star on L2-exceeding sizes (> 126 MB working sets):
    fused lottery step (xi -> partition -> step -> decay), momentum update, segment-sum pooling,
    candidate top-k. achieved = algorithmic bytes / device time."""
    import ctypes as C

    import numpy as np

    import torch

    from paper_2201_05752_b200.distributed import device_gradient_tensor

    hbm = peaks.get("hbm_gbs", 6534.1)
    out = {}

    def timed(fn, stream, reps=5):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps / 1000.0

    # ---- parameter-vector kernels on a 268M-scalar model (1 GB per fp32 array)
    dims = [32768, 8192, 8, 1]
    P = ml.param_count(dims)
    dm = ml.DeviceModel(ml.CostModelParams(dims, np.zeros(P)), ml.PREC_BF16, max_rows=128)
    sp = C.c_void_p()
    L.moses_model_stream(dm.h, C.byref(sp))
    st = torch.cuda.ExternalStream(sp.value)
    wptr = C.POINTER(C.c_float)()
    L.moses_model_device_ptrs(dm.h, C.byref(wptr), None, None)

    class _CAI:
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}

    w = torch.as_tensor(_CAI(C.cast(wptr, C.c_void_p).value, P), device="cuda")
    g = device_gradient_tensor(dm)
    gen = torch.Generator(device="cuda").manual_seed(0)
    w.normal_(0, 0.05, generator=gen)
    g.normal_(0, 1e-2, generator=gen)
    g[torch.rand(P, device="cuda", generator=gen) < 0.4] = 0.0  # zero-gradient ties (README.md:106-113)
    torch.cuda.synchronize()
    pop = C.c_int64()
    for mode, value, name in ((2, 0.5, "lottery_step_ratio0.5"), (1, 0.5, "lottery_step_threshold0.5")):
        t = timed(lambda: ml._ck(L.moses_lottery_step(dm.h, mode, value, 0, 1e-3, 1e-2, None, 0, C.byref(pop))), st)
        algo = 15.0 * P  # read w,g; write w; mask byte; bf16 operand shadow
        out[name] = {"params": P, "ms": t * 1e3, "algorithmic_bytes": algo, "achieved_gbs": algo / t / 1e9,
                     "frac": algo / t / 1e9 / hbm, "bytes_per_param": 15}
    L.moses_set_async(1)
    t = timed(lambda: ml._ck(L.moses_apply_update(dm.h, 1e-3, 0.9, None, 0, 1)), st)
    L.moses_set_async(0)
    algo = 22.0 * P  # read w,v,g; write w,v; bf16 shadow
    out["momentum_update"] = {"params": P, "ms": t * 1e3, "algorithmic_bytes": algo, "achieved_gbs": algo / t / 1e9,
                              "frac": algo / t / 1e9 / hbm, "bytes_per_param": 22}
    del w, g
    dm.close()
    torch.cuda.empty_cache()

    # ---- segment-sum pooling: 4M statement rows x 512 bf16 -> programs x 512 fp32
    programs = 900_000
    off = ml.synth_offsets(11, programs, MAX_STMTS)
    rows = int(off[-1])
    H = torch.empty((rows, 512), dtype=torch.bfloat16, device="cuda").normal_(generator=gen)
    OFF = torch.from_numpy(off).cuda()
    PO = torch.empty((programs, 512), dtype=torch.float32, device="cuda")
    cur = torch.cuda.current_stream()
    t = timed(lambda: ml._ck(L.moses_segment_sum_device(H.data_ptr(), ml.DTYPE_BF16, 512, 512, OFF.data_ptr(),
                                                        programs, PO.data_ptr())), cur)
    algo = rows * 512 * 2 + programs * 512 * 4 + (programs + 1) * 8
    out["segment_sum_pooling"] = {"rows": rows, "programs": programs, "ms": t * 1e3, "algorithmic_bytes": algo,
                                  "achieved_gbs": algo / t / 1e9, "frac": algo / t / 1e9 / hbm}
    del H, PO
    torch.cuda.empty_cache()

    # ---- candidate top-k over 100M fp32 scores (k = 1024)
    n = 100_000_000
    Sc = torch.empty(n, dtype=torch.float32, device="cuda").normal_(generator=gen)
    idx = (C.c_int64 * 1024)()
    ml._ck(L.moses_topk_device(Sc.data_ptr(), n, 1024, idx))
    t0 = time.perf_counter()
    for _ in range(3):
        ml._ck(L.moses_topk_device(Sc.data_ptr(), n, 1024, idx))
    t = (time.perf_counter() - t0) / 3
    out["topk_100M"] = {"n": n, "k": 1024, "ms": t * 1e3, "algorithmic_bytes": 4 * n, "achieved_gbs": 4 * n / t / 1e9,
                        "frac": 4 * n / t / 1e9 / hbm, "note": "wall clock incl. one host sync"}
    del Sc
    torch.cuda.empty_cache()
    out["peak_gbs"] = hbm
    out["peak_source"] = "MEASURED_PEAKS.json hbm_gbs"
    return out


def bench_finetune(ml, L, peaks, reps=20):
    """cfg3: Moses fine-tuning source -> target on the 4x512 model (P = 872,961): one step is the
    tuner.cpp:251-262 Moses branch through the reference-facing C ABI with host buffers
    (gradients with the reversed-BCE adversary over 256 replay rows, beta = 0.01 -> discriminator
    step -> fused lottery step: xi -> ratio 0.5 partition -> transferable step -> variant decay),
    plus the MMD^2 discrepancy between 50k source and 5k target 512-d representations
    (device-resident, tensor-core Gram tiles)."""
    import ctypes as C

    import numpy as np

    import torch

    out = {}
    params = ml.init_random(DIMS, SEED_MODEL, strict=False)
    dm = ml.DeviceModel(params, ml.PREC_BF16X3, max_rows=1024)  # the in-tolerance split-bf16 mode
    rng = np.random.default_rng(3)
    replay = rng.random((256, DIMS[0]))
    adv = ml.AdversaryState(replay, DIMS[-2])
    xt = np.ascontiguousarray(rng.random((BATCH, DIMS[0])))
    yt = np.ascontiguousarray(0.1 + rng.random(BATCH))
    loss = C.c_double()
    dl, cf = C.c_double(), C.c_double()
    pop = C.c_int64()

    def step():
        ml._ck(L.moses_gradients(dm.h, xt.ctypes.data, yt.ctypes.data, BATCH, DIMS[0], adv.h, 0.01, C.byref(loss)))
        ml._ck(L.moses_adversarial_step(adv.h, dm.h, xt.ctypes.data, BATCH, DIMS[0], 0.01, C.byref(dl), C.byref(cf)))
        ml._ck(L.moses_lottery_step(dm.h, 2, 0.5, 0, 1e-3, 1e-2, None, 0, C.byref(pop)))

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out["moses_step"] = {"ms": dt * 1e3, "samples_per_s": BATCH / dt, "batch": BATCH, "replay": 256,
                         "params": len(params.params),
                         "path": "moses_gradients(adv, beta=0.01) + moses_adversarial_step + moses_lottery_step "
                                 "(ratio 0.5), host float64 buffers, wall clock"}

    src = np.ascontiguousarray(rng.random((256, DIMS[0])))

    def mmd_step():  # cfg3 with the MMD^2 domain loss in the discriminator's slot
        ml._ck(L.moses_gradients_mmd(dm.h, xt.ctypes.data, yt.ctypes.data, BATCH, DIMS[0], src.ctypes.data, 256, 0.01,
                                     float(np.sqrt(DIMS[-2] / 6.0)), C.byref(loss)))
        ml._ck(L.moses_lottery_step(dm.h, 2, 0.5, 0, 1e-3, 1e-2, None, 0, C.byref(pop)))

    for _ in range(3):
        mmd_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        mmd_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out["moses_step_mmd"] = {"ms": dt * 1e3, "samples_per_s": BATCH / dt, "source_rows": 256,
                             "path": "moses_gradients_mmd (beta 0.01: rank loss + beta * MMD^2 of the last hidden "
                                     "layer, gradient through every row) + moses_lottery_step (ratio 0.5), host "
                                     "float64 buffers, split-bf16 handle, wall clock"}

    def fused_step():
        ml._ck(L.moses_moses_step(dm.h, adv.h, xt.ctypes.data, yt.ctypes.data, BATCH, DIMS[0], 0.01, 2, 0.5, 0, 1e-3,
                                  1e-2, C.byref(loss), C.byref(dl), C.byref(pop)))

    for _ in range(3):
        fused_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fused_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out["moses_step_fused"] = {"ms": dt * 1e3, "samples_per_s": BATCH / dt,
                               "path": "moses_moses_step: the same three steps in one C-ABI call (the discriminator "
                                       "step reuses the gradients' forward; one host sync), bit-identical"}
    # the lottery step alone at the real parameter count (L2-resident: launch/latency bound)
    sp = C.c_void_p()
    L.moses_model_stream(dm.h, C.byref(sp))
    st = torch.cuda.ExternalStream(sp.value)
    L.moses_set_async(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        ml._ck(L.moses_lottery_step(dm.h, 2, 0.5, 0, 1e-3, 1e-2, None, 0, C.byref(pop)))
    b.record(st)
    torch.cuda.synchronize()
    L.moses_set_async(0)
    out["lottery_step_real_P"] = {"ms": a.elapsed_time(b) / reps, "params": len(params.params),
                                  "note": "device time per fused ratio-0.5 step; w, g L2-resident"}
    del adv
    dm.close()
    # MMD^2 over 50k source / 5k target penultimate representations
    m_s, n_t, w = 50_000, 5_000, DIMS[-2]
    gen = torch.Generator(device="cuda").manual_seed(5)
    H = torch.rand((m_s + n_t, w), device="cuda", generator=gen)
    H[m_s:] += 0.05
    res = C.c_double()
    sig = float(np.sqrt(w / 6.0))

    def mmd():
        ml._ck(L.moses_mmd2_device(C.c_void_p(H.data_ptr()), m_s, C.c_void_p(H[m_s:].data_ptr()), n_t, w, w, sig,
                                   C.byref(res)))

    mmd()
    ml.profile_begin()
    mmd()
    prof = ml.profile_end()
    t0 = time.perf_counter()
    for _ in range(5):
        mmd()
    dt = (time.perf_counter() - t0) / 5
    flops = 2.0 * w * (m_s * (m_s + 1) / 2 + n_t * (n_t + 1) / 2 + m_s * n_t)
    dev_ms = prof.get("other", (None,))[0]
    if peaks.get("tf32_tflops_sustained"):
        peak, peak_src = peaks["tf32_tflops_sustained"], peaks.get("tf32_source", "measured tf32 peak")
    else:
        peak, peak_src = peaks.get("bf16_tflops_sustained", 1408.7) / 2.0, "MEASURED_PEAKS.json bf16 sustained / 2"
    ach = flops / (dev_ms / 1e3) / 1e12 if dev_ms else None
    out["mmd2"] = {"source": m_s, "target": n_t, "width": w, "value": res.value, "ms_wall": dt * 1e3,
                   "ms_device": dev_ms, "flops_unique_pairs": flops,
                   "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                                "frac": ach / peak if ach else None,
                                "peak_source": peak_src,
                                "kernel": "umma_gram_kernel (tcgen05 kind::tf32, exp-sum epilogue)"}}
    del H
    torch.cuda.empty_cache()
    return out


def bench_search(ml, L, peaks):
    """the scorer's input path on the device — enumerate a 10.2M-config knob
    space (6 knobs; space.cpp:168-191 order), encode the 16-d features (space.cpp:140-159) straight
    into packed bf16 model rows plus FNV-1a hashes (space.cpp:193-197), score with the reference's
    {16,512,512,1} model and select the top-1024. No host features, no PCIe."""
    import ctypes as C

    import numpy as np

    import torch

    knobs = [("tile_x", [1 << i for i in range(16)]), ("tile_y", [1 << i for i in range(16)]),
             ("unroll", [0, 1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 128, 256, 512]),
             ("vectorize", [1 << i for i in range(8)]), ("parallel", [1 << i for i in range(13)]),
             ("split", list(range(1, 25)))]
    n = int(np.prod([len(d) for _, d in knobs]))
    task = (2.0, 8.0, 9.0, 5.0)
    dims = [16, 512, 512, 1]
    dm = ml.DeviceModel(ml.init_random(dims, SEED_MODEL), ml.PREC_BF16, max_rows=65536)
    ld = dm.packed_ld
    F = torch.empty((n, ld), dtype=torch.bfloat16, device="cuda")
    Hh = torch.empty(n, dtype=torch.int64, device="cuda")
    S = torch.empty(n, dtype=torch.float32, device="cuda")
    idx = (C.c_int64 * 1024)()

    def encode():
        ml.encode_configs_device(task, knobs, 0, n, ml.DTYPE_BF16, C.c_void_p(F.data_ptr()), ld, dims[0],
                                 C.c_void_p(Hh.data_ptr()))

    def score():
        ml._ck(L.moses_predict_device(dm.h, C.c_void_p(F.data_ptr()), ml.DTYPE_BF16, ld, n, C.c_void_p(S.data_ptr())))
        torch.cuda.synchronize()
        ml._ck(L.moses_topk_device(C.c_void_p(S.data_ptr()), n, 1024, idx))

    encode()
    score()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    encode()
    b.record()
    torch.cuda.synchronize()
    enc_ms = a.elapsed_time(b)
    t0 = time.perf_counter()
    encode()
    score()
    total = time.perf_counter() - t0
    wbytes = n * (ld * 2 + 8)
    hbm = peaks.get("hbm_gbs", 6534.1)
    # f3: simulated-hardware labels (oracle.cpp:65-88) for the whole space, and its exhaustive optimum
    server = {"id": "server", "peak_gflops": 8000.0, "parallel_units": 16.0, "vector_lanes": 8.0,
              "cache_bytes": 2000000.0, "measure_overhead_ms": 2.0, "noise_std": 0.05, "repeats": 3}
    lab = torch.empty(n, dtype=torch.float32, device="cuda")
    ml.measure_configs_device(server, "conv3x3_64", task, knobs, 1, 0, n, label_ptr=C.c_void_p(lab.data_ptr()))
    a.record()
    ml.measure_configs_device(server, "conv3x3_64", task, knobs, 1, 0, n, label_ptr=C.c_void_p(lab.data_ptr()))
    b.record()
    torch.cuda.synchronize()
    label_ms = a.elapsed_time(b)
    t0 = time.perf_counter()
    best, best_lat = ml.true_best(server, task, knobs)
    tb_ms = (time.perf_counter() - t0) * 1e3
    del lab
    # evolve (search.cpp:41-71) with the reference SearchParams (128 / 4 generations / 32 survivors x
    # 4 mutants) on the default knob template, scored by the {16,512,512,1} model on the device
    dknobs = [("tile_x", [1, 2, 4, 8, 16, 32, 64]), ("tile_y", [1, 2, 4, 8, 16, 32, 64]), ("unroll", [0, 16, 64, 512]),
              ("vectorize", [1, 2, 4, 8, 16]), ("parallel", [1, 2, 4, 8, 16, 32, 64, 128, 256])]
    em = ml.DeviceModel(ml.init_random(dims, SEED_MODEL), ml.PREC_BF16, 1024)
    ml.evolve(em, task, dknobs, seed=1)
    t0 = time.perf_counter()
    for r in range(10):
        ml.evolve(em, task, dknobs, seed=r)
    evolve_ms = (time.perf_counter() - t0) / 10 * 1e3
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc

    wts = orc.init_random(dims, SEED_MODEL)
    sizes = [len(d) for _, d in dknobs]

    def cpu_scorer(cfgs):
        rows = []
        for c in cfgs:
            i = 0
            for k, x in enumerate(c):
                i = i * sizes[k] + dknobs[k][1].index(x)
            rows.append(orc.encode_configs(task, dknobs, i, 1)[0][0])
        return list(orc.forward(dims, wts, np.stack(rows))[0])

    t0 = time.perf_counter()
    orc.evolve(dknobs, cpu_scorer, seed=1)
    evolve_cpu_ms = (time.perf_counter() - t0) * 1e3
    em.close()
    out = {"configs": n, "knobs": len(knobs), "model": dims, "encode_ms": enc_ms,
           "encode_roofline": {"bound": "hbm", "achieved": wbytes / (enc_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                               "frac": wbytes / (enc_ms / 1e3) / 1e9 / hbm,
                               "algorithmic_bytes": wbytes, "note": "packed bf16 rows + u64 hashes written"},
           "pipeline_ms": total * 1e3, "configs_per_s": n / total,
           "labels_ms": label_ms, "labels_per_s": n / (label_ms / 1e3),
           "true_best": {"values": best, "latency_ms": best_lat, "ms": tb_ms,
                         "note": "exhaustive noise-free optimum over the 10.2M-config space (oracle.cpp:90-105)"},
           "pipeline": "encode_configs (device) -> predict (tcgen05) -> top-1024, wall clock",
           "evolve": {"ms": evolve_ms, "cpu_oracle_ms": evolve_cpu_ms,
                      "params": "population 128, 4 generations, 32 survivors x 4 mutants, eps 0.05 (SearchParams)",
                      "path": "moses_evolve: device encode from enumeration indices + tcgen05 scoring per "
                              "generation; host RngStream walk and sort; CPU: fp64 oracle forward, 1 thread"}}
    del F, Hh, S
    torch.cuda.empty_cache()
    return out


def bench_pretrain(ml, L, peaks, epochs: int = 30, per_task: int = 6000):
    """the reference's own offline flow — `moseslab gen-dataset --samples 6000`
    on the 8 default tasks / server device (data.cpp:49-65, cli.cpp:344) then `pretrain` with the
    default TrainHyper (30 epochs, batch 512, lr 0.001, momentum 0.9; tuner.cpp:130-156) on
    {16,512,512,1}: dataset generated on the device, per-epoch keyed shuffles / single-task chunking
    on the host overlapped with the device epochs, batches gathered on the device."""
    import ctypes as C

    import numpy as np

    import torch

    lab = json.load(open(os.path.join(ROOT, "paper_2201_05752_b200", "configs", "lab.json")))
    device = lab["devices"]["server"]
    tasks = [(t["id"], (t["work_gflops"], t["bytes_per_unit"], t["ideal_log2_tiles"], t["ideal_log2_unroll"]))
             for t in lab["tasks"]]
    knobs = [("tile_x", [1, 2, 4, 8, 16, 32, 64]), ("tile_y", [1, 2, 4, 8, 16, 32, 64]), ("unroll", [0, 16, 64, 512]),
             ("vectorize", [1, 2, 4, 8, 16]), ("parallel", [1, 2, 4, 8, 16, 32, 64, 128, 256])]
    dims = [16, 512, 512, 1]
    seed = 0
    dm = ml.DeviceModel(ml.init_random(dims, seed), ml.PREC_BF16, 512)
    ld = dm.packed_ld
    n = per_task * len(tasks)
    X = torch.zeros((n, ld), dtype=torch.bfloat16, device="cuda")
    Y = torch.zeros(n, dtype=torch.float32, device="cuda")

    def generate():
        for t, (tid, task) in enumerate(tasks):
            r0 = t * per_task
            ml.generate_dataset_device(device, tid, task, knobs, per_task, 1, ml.DTYPE_BF16,
                                       C.c_void_p(X.data_ptr() + r0 * ld * 2), ld, 16, None, None, None, None,
                                       C.c_void_p(Y.data_ptr() + r0 * 4))

    generate()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    generate()
    torch.cuda.synchronize()
    gen_ms = (time.perf_counter() - t0) * 1e3
    task_of = [i // per_task for i in range(n)]
    ids = [tid for tid, _ in tasks]
    t0 = time.perf_counter()
    plan = ml.make_ranking_batches(task_of, ids, 512, ml.epoch_seed(seed, 0))
    plan_ms = (time.perf_counter() - t0) * 1e3
    ml.pretrain_device(dm, C.c_void_p(X.data_ptr()), ld, C.c_void_p(Y.data_ptr()), task_of, ids, 512, seed, 1)  # warm
    dm.upload(ml.init_random(dims, seed))
    torch.cuda.synchronize()
    k0 = L.moses_kernel_launches()
    t0 = time.perf_counter()
    losses, dropped = ml.pretrain_device(dm, C.c_void_p(X.data_ptr()), ld, C.c_void_p(Y.data_ptr()), task_of, ids,
                                         512, seed, epochs, 0.001, 0.9)
    total = time.perf_counter() - t0
    launches = L.moses_kernel_launches() - k0
    # SURVEY.md §8(f) f4 shape: a (seed) job grid of independent pretrain runs on the native worker
    # pool, one handle (and stream set) per job, sharing the device-resident store
    # (f4 across GPUs: jobs round-robin over every GPU of the process, each over its device's copy)
    n_gpu = torch.cuda.device_count()
    n_jobs = 8 * n_gpu
    home = torch.cuda.current_device()
    copies = {home: (X, Y)}
    jobs = []
    for j in range(n_jobs):
        dev = j % n_gpu
        torch.cuda.set_device(dev)
        if dev not in copies:
            copies[dev] = (X.to(f"cuda:{dev}"), Y.to(f"cuda:{dev}"))
        jobs.append(ml.DeviceModel(ml.init_random(dims, j), ml.PREC_BF16, 512))
    torch.cuda.set_device(home)
    torch.cuda.synchronize()
    xs = [C.c_void_p(copies[j % n_gpu][0].data_ptr()) for j in range(n_jobs)]
    ys = [C.c_void_p(copies[j % n_gpu][1].data_ptr()) for j in range(n_jobs)]
    ml.pretrain_jobs_mapped(jobs, list(range(n_jobs)), xs, ld, ys, task_of, ids, 512, 1, 0.001, 0.9,
                            n_jobs)  # warm (graph capture per handle)
    for j, jm in enumerate(jobs):
        jm.upload(ml.init_random(dims, j))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    job_losses, _ = ml.pretrain_jobs_mapped(jobs, list(range(n_jobs)), xs, ld, ys, task_of, ids, 512, epochs, 0.001,
                                            0.9, n_jobs)
    jobs_s = time.perf_counter() - t0
    for jm in jobs:
        jm.close()
    del copies
    # the same loop on the fp64 CPU oracle: a bounded sample of epoch 0's batches
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc

    threads = os.cpu_count() or 1
    feats = X[:, :16].float().double().cpu().numpy()
    labels = Y.double().cpu().numpy()
    w = orc.init_random(dims, seed)
    mom = np.zeros_like(w)
    nb = min(len(plan), 24)
    t0 = time.perf_counter()
    for b in range(nb):
        _, rows = plan.batch(b)
        orc.train_step_f64(dims, w, mom, feats[rows], labels[rows], 0.001, 0.9, threads)
    cpu_dt = time.perf_counter() - t0
    cpu_rows = int(plan.off[nb])
    del X, Y
    torch.cuda.empty_cache()
    return {"workload": f"gen-dataset --samples {per_task} (8 default tasks, server) + pretrain {epochs} epochs, "
                        f"batch 512, {dims}, bf16",
            "records": n, "batches_per_epoch": len(plan), "dropped_singletons": dropped,
            "generate_ms": gen_ms, "plan_ms_host": plan_ms,
            "pretrain_s": total, "samples_per_s": epochs * n / total, "ms_per_epoch": total / epochs * 1e3,
            "epoch_mean_loss_first_last": [losses[0], losses[-1]], "gpu_launches": int(launches),
            "job_grid": {"jobs": n_jobs, "gpus": n_gpu, "workers": n_jobs, "wall_s": jobs_s,
                         "samples_per_s": n_jobs * epochs * n / jobs_s,
                         "speedup_vs_sequential": n_jobs * total / jobs_s,
                         "path": "moses_pretrain_jobs_mapped: 8 seeds per GPU x 30 epochs, jobs round-robin over "
                                 "the process's GPUs, one handle/stream set per job, each over its GPU's store copy"},
            "cpu_oracle": {"samples_per_s": cpu_rows / cpu_dt, "cores": threads, "kind": "port",
                           "sample": f"{nb} batches ({cpu_rows} rows) of epoch 0, fp64"},
            "path": "moses_generate_dataset_device x8 -> moses_pretrain_device (host plan of epoch e+1 overlapped "
                    "with device epoch e; full batches replay one CUDA graph), wall clock"}
