# One GPU session: smoke, full gpu test suite, bench, ncu launch list, ncu full capture.
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -5 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -30
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-infer --no-hbm --profile-steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain -s 20 -c 2 -o gpurun_out/prof_chain python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-infer --no-hbm --profile-steps 1 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu2.log
ls -la gpurun_out
