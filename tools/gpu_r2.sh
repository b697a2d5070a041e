# One GPU session: smoke, full gpu test suite, default bench line, ncu launch list of the headline step.
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -q -m gpu --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -30
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -3 gpurun_out/bench.err; head -c 3000 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --headline-only --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
ls -la gpurun_out
