set -x
cd $GRAFT_REPO_ROOT
timeout 300 python tools/gemm_sweep.py > gpurun_out/sweep.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep.log
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -m gpu -x --timeout 120 > gpurun_out/pytest_gemm.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gemm.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 120 -k "predict or golden or topk or pooled" > gpurun_out/pytest_pred.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_pred.log
