cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -k "lottery or ratio or threshold or rho1" > gpurun_out/pytest16a.log 2>&1; echo lot rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest16a.log | tail -10
timeout 900 python bench.py --no-infer --no-cpu-baseline > gpurun_out/bench11.json 2> gpurun_out/bench11.err; echo bench rc=$?
tail -3 gpurun_out/bench11.err; python -c "
import json; d=json.load(open('gpurun_out/bench11.json'))
print(d['value'], d['ms_per_step']); print(json.dumps({k: (v['ms'], v['frac']) for k, v in d['hbm_kernels'].items() if isinstance(v, dict)}))"
