cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 300 python -m pytest "tests/test_gpu_parity.py::test_gradients_vs_precision_model" -q -m gpu 2>&1 | tail -3; done
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 > gpurun_out/pytest10.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest10.log | tail -30
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo bench rc=$?
tail -3 gpurun_out/bench5.err; cat gpurun_out/bench5.json
