"""Benchmark of the B200 Moses cost-model hot path (driver contract: one JSON line on rank 0).

Headline workload (BASELINE.json configs[1], cfg2): source-device pre-training of the cost model
{164, 512, 512, 512, 512, 1} ("4x512 hidden") on 200k synthetic TenSet-shaped programs (1-8
statements each, segment-sum pooled), batch 512 programs per GPU, momentum SGD — the tuner.cpp:130-156
loop body (gradients + apply_update). A step = one batch: fused forward chain, pairwise ranking loss,
fused dZ chain, grouped weight gradients with the momentum update in their epilogue. Precision: split
bf16 (MOSES_PREC_BF16X3: every operand hi + lo, 3 bf16 tensor-core MMAs per product; ~1e-5 from the
fp64 reference, tests/test_gpu_bf16x3.py). Metric: train samples/s (whole job). N > 1: data parallel,
one process per GPU, gradient all-reduce between gradients and update (weak scaling, each rank its own
512-program batch of its own shard).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 without a torchrun environment re-launches itself under torch.distributed.run with N
ranks. --impl reference times the reference's CPU path (the fp64 C++ oracle restating model.cpp; the
reference itself cannot be built here) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

METRIC = "cost-model programs/sec (infer) & train samples/sec, 1–8 B200 vs CPU"
DIMS = [164, 512, 512, 512, 512, 1]
PROGRAMS = 200_000
BATCH = 512
SEED_DATA, SEED_MODEL = 1, 12345
LR, MU = 0.001, 0.9
MAX_STMTS = 8  # statements per program: 1 + below(8), mean 4.5
MIN_WINDOW_S = 0.3  # timed K-step windows are repeated until at least this much device time is covered
E2E_MIN_STEPS = 200


def workload_config(world: int) -> dict:
    """The `config` object of both arms (ours and --impl reference): identical by construction."""
    return {"workload": f"cfg2: pretrain {DIMS} (4x512 hidden) on {PROGRAMS} TenSet-shaped programs "
                        f"(segment-sum pooling over 1-{MAX_STMTS} statements per program), batch {BATCH} "
                        f"programs per GPU, momentum SGD lr={LR} mu={MU}",
            "model": "moses-mlp-4x512", "programs": PROGRAMS, "global_batch": BATCH * world,
            "seq_len": None, "parallelism": f"dp{world}",
            "l2": "inputs larger than L2: every step gathers a different batch of the 605 MB device-resident "
                  "fp32 dataset"}


def train_flops_per_sample(dims):
    """Algorithmic FLOPs per training row: forward + weight-grad + data-grad (levels >= 1)."""
    L = len(dims) - 1
    fwd = sum(2 * dims[l] * dims[l + 1] for l in range(L))
    wgrad = sum(2 * dims[l] * dims[l + 1] for l in range(L))
    dgrad = sum(2 * dims[l] * dims[l + 1] for l in range(1, L - 1))
    return fwd, wgrad, dgrad


def hidden_flops_per_step(dims, n):
    """(forward, data-gradient, weight-gradient) FLOPs of the hidden-layer GEMMs of one step over n rows."""
    L = len(dims) - 1
    fwd = sum(2 * n * dims[l] * dims[l + 1] for l in range(L - 1))
    dgrad = sum(2 * n * dims[l] * dims[l + 1] for l in range(1, L - 1))
    return fwd, dgrad, fwd


def gemm_flops_per_step(dims, n):
    """Hidden-layer GEMM FLOPs of one training step over n rows (the head GEMV is not a GEMM)."""
    L = len(dims) - 1
    fwd = sum(2 * n * dims[l] * dims[l + 1] for l in range(L - 1))
    wgrad = sum(2 * n * dims[l] * dims[l + 1] for l in range(L - 1))
    dgrad = sum(2 * n * dims[l] * dims[l + 1] for l in range(1, L - 1))
    return fwd + wgrad + dgrad


class ClockSampler:
    """SM clocks and throttle reasons sampled every 20 ms during the timed region (NVML)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self._stop.is_set():
                self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                bits = int(get_reasons(h))
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
                self._stop.wait(0.02)
        except Exception as e:  # noqa: BLE001 — sampling must never break the bench
            self.error = repr(e)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=5)

    def summary(self):
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s), "sampler": "NVML every 20 ms over all timed windows"}


def cpu_baseline(budget_s: float, threads: int):
    """Reference CPU path (fp64 oracle, reference formulas) on a bounded sample of the cfg2 workload."""
    import numpy as np

    import oracle as orc

    w = orc.init_random(DIMS, SEED_MODEL, strict=False)
    mom = np.zeros_like(w)
    off = orc.synth_offsets(SEED_DATA, BATCH, MAX_STMTS)
    x = orc.synth_features(SEED_DATA, 0, int(off[-1]), DIMS[0])
    y = orc.synth_labels(SEED_DATA, 0, BATCH)

    def step():  # tuner.cpp:146-147 with segment-sum pooling over each program's statements
        nonlocal w, mom
        g, _ = orc.gradients_pooled(DIMS, w, x, off, y, threads)
        w, mom = orc.apply_update(w, mom, g, LR, MU, None, True)

    step()  # warm
    t0 = time.perf_counter()
    n = 0
    while True:
        step()
        n += 1
        if time.perf_counter() - t0 > budget_s or n >= 2000:
            break
    dt = time.perf_counter() - t0
    return {"value": n * BATCH / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{n} fp64 training steps of {BATCH} TenSet-shaped programs ({int(off[-1])} statements) on "
                      f"{DIMS} ({dt:.1f} s), oracle/moses_oracle.hpp restating model.cpp:192-296 + pooling"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (fp64 oracle port), all host threads, rank 0 only."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    budget = max(5.0, min(30.0, 0.05 * (args.steps + args.warmup)))
    base = cpu_baseline(budget, os.cpu_count() or 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": base["value"], "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * BATCH / base["value"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (keyed SplitMix64 TenSet-shaped features, labels 0.1+U; random-init model)",
        "config": workload_config(world),
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def self_launch(args) -> int:
    """--gpus N > 1 outside torchrun: re-run this command under torch.distributed.run with N ranks."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def timed_windows(run_k, K, stream, world, dist):
    """Device time of K back-to-back steps (CUDA events on the launch stream, barrier + synchronize on
    both sides, max over ranks), repeated until MIN_WINDOW_S is covered (>= 3 windows)."""
    import torch

    windows = []
    while len(windows) < 3 or (sum(windows) < MIN_WINDOW_S * 1e3 and len(windows) < 200):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_k(K)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        windows.append(ms)
    return windows


def median(v):
    s = sorted(v)
    return s[len(s) // 2] if len(s) % 2 else 0.5 * (s[len(s) // 2 - 1] + s[len(s) // 2])


_COMM = None


def library_comm(world):
    """The library's NCCL communicator of this rank (N > 1): every collective of the data path runs inside
    libmoses_gpu.so (captured into the step graphs); torch.distributed only distributes the NCCL id."""
    global _COMM
    if world > 1 and _COMM is None:
        from paper_2201_05752_b200.distributed import Comm

        _COMM = Comm.from_torch()
    return _COMM


def bench_cfg2(ml, L, args, rank, world, dist, peaks):
    """The headline: cfg2 training steps on split-bf16 handles, device-resident dataset, graph replay."""
    import ctypes as C

    import numpy as np

    import torch

    from paper_2201_05752_b200.distributed import shard_range

    params = ml.init_random(DIMS, SEED_MODEL, strict=False)
    off_all = ml.synth_offsets(SEED_DATA, PROGRAMS, MAX_STMTS)
    p_lo, p_hi = shard_range(PROGRAMS, rank, world)
    nb = (p_hi - p_lo) // BATCH
    p_hi = p_lo + nb * BATCH
    off = off_all[p_lo:p_hi + 1] - off_all[p_lo]
    row0, n_rows = int(off_all[p_lo]), int(off[-1])
    batch_rows = np.diff(off[::BATCH])
    rows_pad = int((batch_rows.max() + 127) // 128 * 128)
    dm = ml.DeviceModel(params, ml.PREC_BF16X3, max_rows=rows_pad)
    ld = dm.packed_ld
    X = torch.empty((n_rows, ld), dtype=torch.float32, device="cuda")
    Y = torch.empty(nb * BATCH, dtype=torch.float32, device="cuda")
    OFF = torch.from_numpy(off).cuda()
    assert L.moses_synth_features_device(SEED_DATA, row0, n_rows, DIMS[0], ml.DTYPE_F32, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(SEED_DATA, p_lo, nb * BATCH, Y.data_ptr()) == 0
    torch.cuda.synchronize()
    sp = C.c_void_p()
    L.moses_model_stream(dm.h, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    if world > 1:  # throughput-mode DP: NCCL average of the gradients + update inside the step graph
        from paper_2201_05752_b200.distributed import DP_AVERAGE, set_data_parallel

        set_data_parallel(dm, library_comm(world), DP_AVERAGE)
    L.moses_set_async(1)
    # one CUDA graph per step: device gather of the batch's programs -> pooled gradients [-> all-reduce]
    # -> update
    ml._ck(L.moses_train_graph_create_pooled(dm.h, X.data_ptr(), ld, Y.data_ptr(), OFF.data_ptr(), nb, BATCH,
                                             rows_pad, LR, MU, 1))

    def run_k(k):
        ml._ck(L.moses_train_graph_launch(dm.h, k))

    out = {}
    with torch.cuda.stream(stream):
        run_k(args.warmup)
        torch.cuda.synchronize()
        launches0 = ml.kernel_launches()
        with ClockSampler(torch.cuda.current_device()) as clk:
            windows = timed_windows(run_k, args.steps, stream, world, dist)
        launches = (ml.kernel_launches() - launches0) // len(windows)
        ms_step = median(windows) / args.steps
        out["value"] = world * BATCH / (ms_step / 1e3)
        out["ms_per_step"] = ms_step
        out["windows_ms"] = windows
        out["gpu_launches"] = int(launches)
        out["clocks"] = clk.summary()

        # the same step with a 256 MiB L2 flush before each one (reported, not the headline)
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
        nfl = 100
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nfl)]
        for k in range(nfl):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            run_k(1)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        out["ms_per_step_l2_flushed"] = sum(a.elapsed_time(b) for a, b in evs) / nfl
        del flush

        # device-time attribution: the same step through the eager C-ABI calls with CUDA events
        # around every kernel class on its launch stream (a separate pass: events perturb timing)
        xb = np.ascontiguousarray(X[: int(batch_rows[0]), : DIMS[0]].double().cpu().numpy())
        ob = np.ascontiguousarray(off[: BATCH + 1])
        yb = np.ascontiguousarray(Y[:BATCH].double().cpu().numpy())
        for _ in range(3):
            ml._ck(L.moses_gradients_pooled(dm.h, xb.ctypes.data, xb.shape[0], DIMS[0], ob.ctypes.data, BATCH,
                                            yb.ctypes.data, None))
        ml.profile_begin()
        for _ in range(args.profile_steps):
            ml._ck(L.moses_gradients_pooled(dm.h, xb.ctypes.data, xb.shape[0], DIMS[0], ob.ctypes.data, BATCH,
                                            yb.ctypes.data, None))
            ml._ck(L.moses_apply_update(dm.h, LR, MU, None, 0, 1))
        torch.cuda.synchronize()
        out["prof"] = ml.profile_end()
        out["rows_per_step"] = n_rows / nb
        out["rows_pad"] = rows_pad

        # end to end through the reference-facing C ABI with host buffers: every step uploads its
        # batch's float64 statement rows, CSR offsets and labels from pinned host memory and reads its
        # loss back. N = 1: moses_train_step_pooled_async (upload of step k+1 overlapping step k);
        # N > 1: moses_gradients_pooled + all-reduce + moses_apply_update.
        L.moses_set_async(0)
        nhb = 4
        host = []
        for hb in range(nhb):
            lo, hi = int(off[hb * BATCH]), int(off[(hb + 1) * BATCH])
            host.append((torch.from_numpy(np.ascontiguousarray(X[lo:hi, : DIMS[0]].double().cpu().numpy())).pin_memory(),
                         torch.from_numpy(np.ascontiguousarray(off[hb * BATCH:(hb + 1) * BATCH + 1] - lo)).pin_memory(),
                         torch.from_numpy(np.ascontiguousarray(Y[hb * BATCH:(hb + 1) * BATCH].double().cpu().numpy()))
                         .pin_memory()))
        e2e_steps = max(E2E_MIN_STEPS, args.steps)
        losses = torch.zeros(e2e_steps + 64, dtype=torch.float64).pin_memory()
        loss = C.c_double()
        step_args = [(xh.data_ptr(), xh.shape[0], oh.data_ptr(), yh.data_ptr()) for xh, oh, yh in host]
        loss_ptrs = [losses[k:k + 1].data_ptr() for k in range(e2e_steps + 64)]
        async_step = L.moses_train_step_pooled_async
        rcs = []

        def e2e_step(k):
            xp, ns, op, yp = step_args[k % nhb]
            if world == 1:
                rcs.append(async_step(dm.h, xp, ns, DIMS[0], op, BATCH, yp, LR, MU, loss_ptrs[k]))
                return
            ml._ck(L.moses_gradients_pooled(dm.h, xp, ns, DIMS[0], op, BATCH, yp, C.byref(loss)))
            ml._ck(L.moses_dp_allreduce_gradients(dm.h, 1))
            ml._ck(L.moses_apply_update(dm.h, LR, MU, None, 0, 1))

        for k in range(max(args.warmup, 300)):  # slot graphs captured, copy pipeline in steady state
            e2e_step(e2e_steps + (k % 64))
        ml._ck(L.moses_model_synchronize(dm.h))
        torch.cuda.synchronize()
        import gc

        e2e_windows = []
        for _ in range(3):
            if world > 1:
                dist.barrier()
            gc.disable()
            t0 = time.perf_counter()
            for k in range(e2e_steps):
                e2e_step(k)
            ml._ck(L.moses_model_synchronize(dm.h))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            gc.enable()
            if world > 1:
                t = torch.tensor([dt], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = float(t.item())
            e2e_windows.append(dt)
        if any(rcs):
            ml._ck(next(r for r in rcs if r))
        assert world > 1 or (bool(torch.isfinite(losses[:e2e_steps]).all()) and float(losses[e2e_steps - 1]) > 0)
        h2d = int(np.mean([sum(t.numel() * t.element_size() for t in hb) for hb in host]))
        # this box's pinned host -> device copy rate for one step's rows (the e2e floor is h2d / rate)
        # (on a torch-owned stream: the pinned block's use is recorded on it, and the handle's stream
        # this section runs on is destroyed with the handle)
        xh = host[0][0]
        with torch.cuda.stream(torch.cuda.Stream()):
            dst = torch.empty(xh.numel(), dtype=torch.float64, device="cuda")
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(3):
                dst.copy_(xh.view(-1), non_blocking=True)
            ev0.record()
            for _ in range(20):
                dst.copy_(xh.view(-1), non_blocking=True)
            ev1.record()
            torch.cuda.synchronize()
            h2d_gbs = 20 * xh.numel() * 8 / (ev0.elapsed_time(ev1) / 1e3) / 1e9
            del dst
        out["e2e"] = {"value": world * BATCH * e2e_steps / median(e2e_windows), "unit": "samples/s",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8, "steps_per_window": e2e_steps,
                      "h2d_gbs_measured": h2d_gbs,
                      "h2d_floor_us_per_step": h2d / (h2d_gbs * 1e3),
                      "windows_samples_per_s": [world * BATCH * e2e_steps / w for w in e2e_windows],
                      "path": ("moses_train_step_pooled_async (C ABI: pinned host float64 rows/offsets/labels "
                               "uploaded every step, upload of step k+1 overlapping step k, per-step loss read "
                               "back; 4 distinct host batches)") if world == 1 else
                              "moses_gradients_pooled + moses_dp_allreduce_gradients (NCCL) + moses_apply_update "
                              "(C ABI, pinned host buffers)"}
    out["dataset_bytes"] = int(X.numel() * X.element_size())
    dm.close()
    del X, Y
    torch.cuda.empty_cache()
    return out


def bench_cfg5(ml, L, args, rank, world, dist, peaks):
    """cfg5: TenSet-scale training of {164,512,512,1} on 2M single-statement programs with a GLOBAL batch
    of 4096 (exact-batch data parallel at N > 1: each rank holds 4096/N rows of every batch, scores are
    all-gathered so the pair loss couples the whole batch, gradients summed over NCCL inside the step
    graph), split bf16, graph replay. At N = 1 the GEMM roofline of the step at a batch where the chains
    are throughput- rather than latency-bound."""
    import ctypes as C

    import torch

    from paper_2201_05752_b200.distributed import shard_range

    dims, programs, gbatch = [164, 512, 512, 1], 2_000_000, 4096
    batch = gbatch // world  # this rank's rows of every global batch
    lo, hi = shard_range(programs, rank, world)
    nb = (hi - lo) // batch
    dm = ml.DeviceModel(ml.init_random(dims, SEED_MODEL), ml.PREC_BF16X3, max_rows=batch)
    ld = dm.packed_ld
    X = torch.empty((nb * batch, ld), dtype=torch.float32, device="cuda")
    Y = torch.empty(nb * batch, dtype=torch.float32, device="cuda")
    assert L.moses_synth_features_device(SEED_DATA + 5, lo, nb * batch, dims[0], ml.DTYPE_F32, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(SEED_DATA + 5, lo, nb * batch, Y.data_ptr()) == 0
    torch.cuda.synchronize()
    sp = C.c_void_p()
    L.moses_model_stream(dm.h, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    if world > 1:
        from paper_2201_05752_b200.distributed import DP_EXACT, set_data_parallel

        set_data_parallel(dm, library_comm(world), DP_EXACT)
    L.moses_set_async(1)
    ml._ck(L.moses_train_graph_create(dm.h, X.data_ptr(), ld, Y.data_ptr(), nb, batch, LR, MU, 1))

    def run_k(k):
        ml._ck(L.moses_train_graph_launch(dm.h, k))

    with torch.cuda.stream(stream):
        run_k(5)
        windows = timed_windows(run_k, 20, stream, world, dist)
        ms = median(windows) / 20
        xs = X[:batch]
        step_fn = L.moses_dp_train_step if world > 1 else L.moses_train_step_device
        ml.profile_begin()
        for _ in range(10):
            ml._ck(step_fn(dm.h, xs.data_ptr(), ld, Y.data_ptr(), batch, LR, MU, None))
        torch.cuda.synchronize()
        prof = ml.profile_end()
    L.moses_set_async(0)
    gemm_ms = sum(prof[c][0] for c in ("gemm_fwd", "gemm_dgrad", "gemm_wgrad")) / 10
    flops = gemm_flops_per_step(dims, batch)  # this GPU's rows
    peak = peaks.get("bf16_tflops_sustained", 1395.6)
    ach = flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else None
    dm.close()
    del X, Y
    torch.cuda.empty_cache()
    return {"workload": f"cfg5: train {dims} on {programs} single-statement programs, global batch {gbatch} "
                        f"({batch} rows per GPU), split bf16, {world} GPU(s)"
                        + (" (exact-batch DP: score all-gather + gradient all-reduce over NCCL in the step graph)"
                           if world > 1 else ""),
            "value": gbatch / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms,
            "timed_windows": len(windows), "steps_per_window": 20,
            "scaling": "strong",
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                         "frac": ach / peak if ach else None, "mma_per_product": 3,
                         "tensor_pipe_frac": 3 * ach / peak if ach else None, "flops_per_step": flops,
                         "gemm_ms_per_step": gemm_ms,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                         "note": "achieved = algorithmic FLOPs / GEMM device time; split bf16 issues 3 bf16 MMAs "
                                 "per product (tensor_pipe_frac)"},
            "step_breakdown_ms": {k: v[0] / 10 for k, v in prof.items() if v[1]}}


def bench_infer(ml, L, programs, peaks, rank, world, dist, precision, reps=3):
    """cfg4: score a pool of `programs` synthetic programs with the 4x512 model and select the global
    top-1024 (score desc, index asc). N > 1: contiguous program ranges per rank (strong scaling); each
    rank scores and top-k's its shard, the (score, global index) winners are all-gathered and merged
    (distributed.py) — the only exchange. Features generated on the device."""
    import ctypes as C

    import numpy as np

    import torch

    from paper_2201_05752_b200.distributed import shard_range, topk_sharded

    chunk = 131072  # rows per predict call (tools/score_chunk_probe.py: larger chunks amortise the per-layer launch tails)
    k = 1024
    lo, hi = shard_range(programs, rank, world)
    n_local = hi - lo
    dm = ml.DeviceModel(ml.init_random(DIMS, SEED_MODEL, strict=False), precision, max_rows=chunk)
    ld = dm.packed_ld
    dt_in = ml.input_dtype(precision)
    X = torch.empty((n_local, ld), dtype=torch.bfloat16 if dt_in == ml.DTYPE_BF16 else torch.float32, device="cuda")
    S = torch.empty(n_local, dtype=torch.float32, device="cuda")
    assert L.moses_synth_features_device(SEED_DATA + 100, lo, n_local, DIMS[0], dt_in, X.data_ptr(), ld) == 0
    torch.cuda.synchronize()
    idx = (C.c_int64 * k)()
    sp = C.c_void_p()
    L.moses_model_stream(dm.h, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)

    def one_pass():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            a.record(stream)
            ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), dt_in, ld, n_local, S.data_ptr()))
            b.record(stream)
        torch.cuda.synchronize()
        if world > 1:  # local top-k + NCCL all-gather of the winners + comparator merge (library)
            win = topk_sharded(library_comm(world), S.data_ptr(), n_local, lo, k)
        else:
            kk = min(k, n_local)
            ml._ck(L.moses_topk_device(S.data_ptr(), n_local, kk, idx))
            win = np.array(idx[:kk], dtype=np.int64)
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        return dt, a.elapsed_time(b), win

    one_pass()
    times, fwd_ms = [], []
    for _ in range(reps):
        dt, fm, win = one_pass()
        times.append(dt)
        fwd_ms.append(fm)
    best = min(times)
    gemm_flops = n_local * sum(2 * DIMS[l] * DIMS[l + 1] for l in range(len(DIMS) - 2))
    peak = peaks.get("bf16_tflops_sustained", 1395.6)
    ach = gemm_flops / (min(fwd_ms) / 1e3) / 1e12
    split = precision == ml.PREC_BF16X3
    dm.close()
    del X
    torch.cuda.empty_cache()
    return {"metric": "cost-model programs/sec (infer)", "value": programs / best, "unit": "programs/s",
            "precision": "bf16x3 (split bf16, in tolerance)" if split else "bf16 (throughput mode)",
            "workload": f"cfg4: score {programs} synthetic programs with {DIMS}, global top-{k}, {world} GPU(s), "
                        f"contiguous program shards",
            "scaling": "strong", "programs_per_gpu": n_local, "first_winners": [int(v) for v in win[:4]],
            "ms_per_pass": best * 1000.0, "forward_ms": min(fwd_ms),
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                         "mma_per_product": 3 if split else 1,
                         "kernel": "umma_fwd_pair_split (tcgen05 cta_group::2, split-bf16 weight slices resident, "
                                   "layer by layer above 16K rows)" if split else
                                   "umma_fwd_pair (tcgen05 cta_group::2, weight-resident)",
                         "forward_device_ms": min(fwd_ms)},
            "inputs": f"device-resident {'fp32' if dt_in == ml.DTYPE_F32 else 'bf16'} packed features (> L2)",
            "timing": "wall clock per pass (device forward + local top-k + NCCL all-gather merge in the library), "
                      "max over ranks"}


def roofline_dominant(prof, K, fwd, dg, wg, peak, traffic, flops, gemm_ms, gemm_launches):
    """Roofline of the step's dominant kernel — the fused forward chain (mlp_chain_split_stream_kernel<FWD>):
    its algorithmic FLOPs per launch over its average launch duration (CUDA events on its stream); the dZ
    chain and the split-K weight-gradient launches alongside, each against its own FLOPs."""
    def ach(f, cat):
        ms = prof[cat][0] / K
        return (f / (ms / 1e3) / 1e12 if ms > 0 else None), ms

    a_f, ms_f = ach(fwd, "gemm_fwd")
    a_d, ms_d = ach(dg, "gemm_dgrad")
    a_w, ms_w = ach(wg, "gemm_wgrad")
    kernels = {
        "fwd_chain": {"kernel": "mlp_chain_split_stream_kernel<FWD>", "flops": fwd, "ms": ms_f, "achieved": a_f},
        "dz_chain": {"kernel": "mlp_chain_split_stream_kernel<DGRAD>", "flops": dg, "ms": ms_d, "achieved": a_d},
        "wgrad": {"kernel": "wgrad_sk_kernel (last hidden level beside the dZ chain + the others after it)",
                  "flops": wg, "ms": ms_w, "achieved": a_w},
    }
    for v in kernels.values():
        v["frac"] = v["achieved"] / peak if v["achieved"] else None
        v["tensor_pipe_frac"] = 3 * v["achieved"] / peak if v["achieved"] else None
    return {"bound": "tensor", "achieved": a_f, "peak": peak, "unit": "TFLOP/s",
            "frac": a_f / peak if a_f else None, "traffic": traffic,
            "traffic_unit": "DRAM bytes per forward-chain launch, cold-cache ncu replay (profiles/ncu_traffic.json)",
            "mma_per_product": 3, "tensor_pipe_frac": 3 * a_f / peak if a_f else None,
            "kernel": "mlp_chain_split_stream_kernel<FWD>: the fused split-bf16 forward chain, the step's "
                      "longest launch",
            "kernels": kernels,
            "all_gemms": {"flops_per_step": flops, "gemm_ms_per_step": gemm_ms,
                          "gemm_launches_per_step": gemm_launches,
                          "achieved": flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None,
                          "note": "sum of GEMM launch durations (the early weight-gradient launch overlaps the dZ "
                                  "chain, so this undercounts the overlap)"},
            "timing": f"CUDA events on the launch streams around each GEMM launch, eager profiling pass of {K} steps "
                      "beside the timed windows",
            "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained"}


def bench_cfg1(ml, L):
    """cfg1: the reference's CPU-runnable case — {164,256,256,1} (2x256 hidden) scoring 4,096 programs,
    fp32 parity mode (3xTF32, <= 1e-5 of fp64), through moses_predict with host float64 rows."""
    import numpy as np

    import oracle as orc

    dims, n = [164, 256, 256, 1], 4096
    p = ml.init_random(dims, SEED_MODEL, strict=False)
    x = orc.synth_features(SEED_DATA, 0, n, dims[0])
    dm = ml.DeviceModel(p, ml.PREC_FP32, n)
    s = ml.predict(dm, x)
    t0 = time.perf_counter()
    reps = 50
    for _ in range(reps):
        s = ml.predict(dm, x)
    dt = (time.perf_counter() - t0) / reps
    ref, _ = orc.forward(dims, p.params, x, threads=os.cpu_count() or 1)
    t1 = time.perf_counter()
    orc.forward(dims, p.params, x, threads=1)
    cpu1 = time.perf_counter() - t1
    err = float(np.max(np.abs(s - ref)) / np.max(np.abs(ref)))
    dm.close()
    return {"workload": f"cfg1: score {n} programs with {dims}, fp32 parity mode (3xTF32)", "ms": dt * 1e3,
            "programs_per_s": n / dt, "normwise_err_vs_fp64": err,
            "path": "moses_predict (host float64 rows in, scores out; H2D + 2 split GEMMs + head + D2H)",
            "cpu_oracle_1thread": {"ms": cpu1 * 1e3, "programs_per_s": n / cpu1}}


_FULL_AFFINITY = set()


def restore_affinity():
    """All host cores again (the CPU baselines time the reference path on every core)."""
    if _FULL_AFFINITY:
        os.sched_setaffinity(0, _FULL_AFFINITY)


def gpu_local_affinity(local):
    """Run this rank on the CPUs of its GPU's NUMA node (as numactl --cpunodebind would), so the pinned
    host buffers of the end-to-end leg are allocated node-local to the GPU's PCIe root; a far node
    halves the H2D rate of the float64 rows on some boxes. No-op when the topology is unavailable."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local)
        bus = pynvml.nvmlDeviceGetPciInfo(h).busId
        bus = (bus.decode() if isinstance(bus, bytes) else bus).lower()
        dom, rest = bus.split(":", 1)
        path = f"/sys/bus/pci/devices/{dom[-4:]}:{rest}/local_cpulist"
        cpus = set()
        for part in open(path).read().strip().split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            _FULL_AFFINITY.update(os.sched_getaffinity(0))
            os.sched_setaffinity(0, cpus)
    except Exception:  # noqa: BLE001
        pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=20)
    ap.add_argument("--no-infer", action="store_true")
    ap.add_argument("--no-hbm", action="store_true")
    ap.add_argument("--no-finetune", action="store_true")
    ap.add_argument("--no-pretrain", action="store_true")
    ap.add_argument("--no-search", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true")
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--infer-programs", type=int, default=10_000_000)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.steps = max(args.steps, 1)
    if args.headline_only:
        args.no_infer = args.no_hbm = args.no_finetune = args.no_pretrain = args.no_search = args.no_cfg5 = True

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)
    gpu_local_affinity(local)

    import torch
    import torch.distributed as dist

    from paper_2201_05752_b200 import moseslab as ml

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = ml.lib()
    if L.moses_device_check() != 0:
        raise SystemExit("moses: " + L.moses_last_error().decode())
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        pass
    try:
        tp = json.load(open(os.path.join(ROOT, "profiles", "measured_tf32_peak.json")))
        peaks["tf32_tflops_sustained"] = tp["tf32_tflops_sustained"]
        peaks["tf32_source"] = "profiles/measured_tf32_peak.json (tools/measure_tf32_peak.py, this pool's B200)"
    except Exception:  # noqa: BLE001
        pass

    head = bench_cfg2(ml, L, args, rank, world, dist, peaks)
    restore_affinity()  # the node-local binding only matters for the e2e leg's pinned buffers
    cfg5 = None if args.no_cfg5 else bench_cfg5(ml, L, args, rank, world, dist, peaks)
    infer = infer_bf16 = None
    if not args.no_infer:  # every rank: the candidate pool is sharded across the GPUs
        infer = bench_infer(ml, L, args.infer_programs, peaks, rank, world, dist, ml.PREC_BF16X3)
        infer_bf16 = bench_infer(ml, L, args.infer_programs, peaks, rank, world, dist, ml.PREC_BF16)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    prof, K = head["prof"], args.profile_steps
    gemm_ms = sum(prof[c][0] for c in ("gemm_fwd", "gemm_dgrad", "gemm_wgrad")) / K
    gemm_launches = sum(prof[c][1] for c in ("gemm_fwd", "gemm_dgrad", "gemm_wgrad")) / K
    flops = gemm_flops_per_step(DIMS, head["rows_per_step"])  # real statement rows, not the padding
    peak = peaks.get("bf16_tflops_sustained", 1395.6)
    traffic = None
    try:  # DRAM bytes per launch of the forward chain from one ncu --set full capture (tools/ncu_train_split.sh)
        per = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get("per_kernel_bytes", {})
        fw = [v for k, v in per.items() if "chain" in k and ("<true>" in k or "<1>" in k)]
        traffic = fw[0] if fw else None
    except Exception:  # noqa: BLE001
        pass
    fwd, wg, dg = (v * head["rows_per_step"] / BATCH for v in train_flops_per_sample(DIMS))
    line = {
        "metric": METRIC, "value": head["value"], "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16x3",
        "dtype_note": "split bf16: every GEMM operand is hi + lo (bf16 each), products hi*hi + hi*lo + lo*hi on the "
                      "bf16 tensor cores with fp32 accumulation; ~1e-5 normwise from the fp64 reference "
                      "(tests/test_gpu_bf16x3.py; north-star bound 1e-3)",
        "data": "synthetic (keyed SplitMix64 TenSet-shaped features 164-d, labels 0.1+U; random-init model)",
        "config": workload_config(world),
        "timed_windows": len(head["windows_ms"]), "windows_ms": head["windows_ms"],
        "ms_per_step_l2_flushed": head["ms_per_step_l2_flushed"],
        "e2e": head["e2e"],
        "roofline": roofline_dominant(prof, K, *hidden_flops_per_step(DIMS, head["rows_per_step"]), peak, traffic, flops,
                                      gemm_ms, gemm_launches),
        "step_breakdown_ms": {k: v[0] / K for k, v in prof.items() if v[1]},
        "algorithmic_flops_per_sample": {"fwd": fwd, "wgrad": wg, "dgrad": dg},
        "rows_per_step": head["rows_per_step"], "rows_per_step_padded": head["rows_pad"],
        "gpu_launches": head["gpu_launches"],
        "clocks": head["clocks"],
    }
    if cfg5 is not None:
        line["cfg5"] = cfg5
    if infer is not None:
        line["infer"] = infer
        line["infer_bf16_throughput_mode"] = infer_bf16
    import bench_sections as bs

    if not args.no_hbm:
        line["hbm_kernels"] = bs.bench_hbm_kernels(ml, L, peaks)
    if not args.no_finetune:
        line["finetune"] = bs.bench_finetune(ml, L, peaks)
    if not args.no_search:
        line["search"] = bs.bench_search(ml, L, peaks)
    if not args.no_pretrain:
        line["pretrain"] = bs.bench_pretrain(ml, L, peaks)
    if world == 1 and not args.headline_only:
        line["cfg1"] = bench_cfg1(ml, L)
    if not args.no_cpu_baseline and world == 1:
        restore_affinity()
        allc = cpu_baseline(10.0, os.cpu_count() or 1)
        one = cpu_baseline(8.0, 1)
        line["cpu_baseline"] = allc
        line["cpu_baseline_1thread"] = one
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
