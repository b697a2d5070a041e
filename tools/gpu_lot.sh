set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -k "lottery or ratio or threshold or rho1" > gpurun_out/pytest_lot.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_lot.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lot_launches.csv python tools/lot_prof.py ratio 2 > gpurun_out/lot_prof.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 50 --warmup 5 --no-infer --no-cpu-baseline > gpurun_out/bench_lot.json 2> gpurun_out/bench_lot.err; echo bench rc=$?
tail -3 gpurun_out/bench_lot.err; python -c "
import json; d=json.load(open('gpurun_out/bench_lot.json'))
print(json.dumps({k: (v['ms'], v['frac']) for k, v in d['hbm_kernels'].items() if isinstance(v, dict)}))"
