cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
K='tests/test_gpu_parity.py'
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest $K -q -x -p no:cacheprovider -k "test_topk_one_launch_pools and 1048577 or test_resident_lottery_step_bit_exact or test_fused_lottery_step_compaction_path_bit_exact" > gpurun_out/sanitize_racecheck_r2b.log 2>&1; echo racecheck rc=$?
tail -3 gpurun_out/sanitize_racecheck_r2b.log
