import sys, time, torch
sys.path.insert(0, ".")
from paper_2201_05752_b200 import moseslab as ml
DIMS = [164, 512, 512, 512, 512, 1]
L = ml.lib()
n = 2_000_000
for prec in ("BF16X3", "BF16"):
    P = getattr(ml, "PREC_" + prec)
    DT = ml.input_dtype(P)
    for cap in (16384, 32768, 65536, 131072):
        dm = ml.DeviceModel(ml.init_random(DIMS, 1, strict=False), P, max_rows=cap)
        ld = dm.packed_ld
        X = torch.empty((n, ld), dtype=torch.bfloat16 if DT == ml.DTYPE_BF16 else torch.float32, device="cuda")
        S = torch.empty(n, dtype=torch.float32, device="cuda")
        assert L.moses_synth_features_device(3, 0, n, DIMS[0], DT, X.data_ptr(), ld) == 0
        ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), DT, ld, n, S.data_ptr()))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            ml._ck(L.moses_predict_device(dm.h, X.data_ptr(), DT, ld, n, S.data_ptr()))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 3
        print(prec, cap, f"{n / dt / 1e6:.1f} M programs/s")
        dm.close(); del X, S; torch.cuda.empty_cache()
