"""Host-side staging costs on the GPU box: numpy copy into pinned memory vs pageable and pinned H2D copies."""
import time, numpy as np, torch
x = np.random.default_rng(0).random((512, 164))
for sz_rows in (512, 2048):
    src = np.ascontiguousarray(np.random.default_rng(1).random((sz_rows, 164)))
    pin = torch.empty(src.shape, dtype=torch.float64, pin_memory=True)
    pn = pin.numpy()
    for _ in range(5): np.copyto(pn, src)
    t0 = time.perf_counter()
    for _ in range(50): np.copyto(pn, src)
    dt = (time.perf_counter() - t0) / 50
    print(f"{src.nbytes/1e3:.0f} KB numpy copy into pinned: {dt*1e6:.1f} us = {src.nbytes/dt/1e9:.1f} GB/s")
    d = torch.empty(src.shape, dtype=torch.float64, device="cuda")
    s = torch.from_numpy(src)
    for _ in range(5): d.copy_(s); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50): d.copy_(s); torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 50
    print(f"  pageable H2D copy_: {dt*1e6:.1f} us")
    for _ in range(5): d.copy_(pin, non_blocking=True); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50): d.copy_(pin, non_blocking=True); torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 50
    print(f"  pinned H2D copy_: {dt*1e6:.1f} us")
