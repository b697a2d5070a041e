cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 -x > gpurun_out/pytest13.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest13.log | tail -30
timeout 900 python bench.py > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo bench rc=$?
tail -3 gpurun_out/bench8.err; python -c "
import json; d=json.load(open('gpurun_out/bench8.json'))
print(d['value'], d['ms_per_step']); print(d['step_breakdown_ms']); print(d['e2e']['value']); print(d['roofline']['frac']); print(d['infer']['value'], d['infer']['roofline']); print(d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
