cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_tune.py tests/test_gpu_evolve.py -q --timeout 300 > gpurun_out/pytest_tune.log 2>&1; echo pytest rc=$?
grep -E "^(FAILED|ERROR)|passed|failed|Error|assert|error" gpurun_out/pytest_tune.log | head -30
