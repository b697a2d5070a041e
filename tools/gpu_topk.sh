set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -k "topk" > gpurun_out/pytest_topk.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_topk.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_tk.json 2> gpurun_out/bench_tk.err; echo bench rc=$?
tail -3 gpurun_out/bench_tk.err; python -c "
import json; d=json.load(open('gpurun_out/bench_tk.json'))
print(json.dumps({k: (v['ms'], v['frac']) for k, v in d['hbm_kernels'].items() if isinstance(v, dict)}))
print(d['value'], d['infer']['value'], d['infer']['roofline']['frac'])"
