cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 > gpurun_out/pytest11.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest11.log | tail -30
timeout 900 python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo bench rc=$?
tail -3 gpurun_out/bench6.err; python -c "
import json; d=json.load(open('gpurun_out/bench6.json'))
print(d['value'], d['ms_per_step']); print(d['step_breakdown_ms']); print(d['e2e']); print(d['infer']['value'], d['infer']['roofline']); print(d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
