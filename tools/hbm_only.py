import json, os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from paper_2201_05752_b200 import moseslab as ml
import bench_sections as bs
peaks = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
out = bs.bench_hbm_kernels(ml, ml.lib(), peaks)
print(json.dumps({k: (round(v["frac"], 3) if isinstance(v, dict) and "frac" in v else v) for k, v in out.items()}))
