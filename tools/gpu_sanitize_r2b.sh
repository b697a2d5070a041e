# compute-sanitizer over this session's kernels: the one-launch top-k (topk.cu), the resident lottery
# step with the split operand pairs, and the early-wgrad / fused-update ordering (capi.cu backward_rows)
cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
M='tests/test_gpu_parity.py tests/test_gpu_bf16x3.py tests/test_gpu_wgrad_sk.py::test_fused_update_with_early_level_equals_single_launch'
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest $M -q -x -p no:cacheprovider -k "topk or lottery or moses_step or early_level" > gpurun_out/sanitize_memcheck_r2b.log 2>&1; echo memcheck rc=$?
tail -3 gpurun_out/sanitize_memcheck_r2b.log
K='tests/test_gpu_parity.py'
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest $K -q -x -p no:cacheprovider -k "test_topk_one_launch_pools and 1048577 or test_resident_lottery_step_bit_exact" > gpurun_out/sanitize_racecheck_r2b.log 2>&1; echo racecheck rc=$?
tail -3 gpurun_out/sanitize_racecheck_r2b.log
timeout 1500 $CS --tool synccheck --print-limit 20 python -m pytest $K -q -x -p no:cacheprovider -k "test_topk_one_launch_pools and 1048577 or test_resident_lottery_step_bit_exact" > gpurun_out/sanitize_synccheck_r2b.log 2>&1; echo synccheck rc=$?
tail -3 gpurun_out/sanitize_synccheck_r2b.log
