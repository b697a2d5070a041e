set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -m gpu -x --timeout 300 > gpurun_out/pytest_gemm.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gemm.log
timeout 300 python tools/gemm_sweep.py > gpurun_out/sweep.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep.log
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_persistent -s 4 -c 2 -o gpurun_out/prof_fwd python tools/gemm_sweep.py fwd > gpurun_out/ncu_p.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_p.log
