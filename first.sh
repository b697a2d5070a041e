set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd $GRAFT_REPO_ROOT
timeout 240 python -c "
import __graft_entry__ as g
g.smoke()
" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -20 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 > gpurun_out/pytest1.log 2>&1; echo pytest rc=$?
tail -40 gpurun_out/pytest1.log
