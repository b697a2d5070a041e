cd $GRAFT_REPO_ROOT
timeout 600 python tools/gemm_sweep.py 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -m gpu --timeout 120 -k cluster 2>&1 | tail -2
