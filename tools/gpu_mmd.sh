set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -k "mmd" > gpurun_out/pytest_mmd.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_mmd.log
timeout 300 python tools/mmd_bench.py > gpurun_out/mmd_bench.log 2>&1; echo mmd rc=$?
cat gpurun_out/mmd_bench.log | tail -5
