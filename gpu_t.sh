cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cpp_api.py -q -m gpu --timeout 300 > gpurun_out/pytest8.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest8.log | tail -30
timeout 900 python bench.py --steps 100 --warmup 10 --no-infer > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench rc=$?
tail -3 gpurun_out/bench4.err; cat gpurun_out/bench4.json
