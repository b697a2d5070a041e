cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "lottery or threshold" > gpurun_out/pytest_lot.log 2>&1; echo pytest rc=$?
grep -E "^(FAILED|ERROR)|passed|failed|Error|assert" gpurun_out/pytest_lot.log | tail -20
timeout 300 python bench.py --headline-only --no-cpu-baseline --steps 20 --warmup 5 > /dev/null 2>&1
timeout 600 python -c "
import sys, json; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
from paper_2201_05752_b200 import moseslab as ml
import bench_sections as bs
peaks=json.load(open('MEASURED_PEAKS.json'))
r=bs.bench_hbm_kernels(ml, ml.lib(), peaks)
print(json.dumps({k:(v if not isinstance(v,dict) else {a:b for a,b in v.items() if a in ('ms','frac','achieved_gbs')}) for k,v in r.items()}))
"
