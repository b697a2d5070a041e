# compute-sanitizer over the round-2 kernels' GPU tests (memcheck over the files, racecheck and
# synccheck on one representative case each: they serialise every shared-memory access)
cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_wgrad_sk.py tests/test_gpu_rank_sym.py tests/test_gpu_chain_pair.py"
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest $T -q -x -p no:cacheprovider > gpurun_out/sanitize_memcheck.log 2>&1; echo memcheck rc=$?
tail -3 gpurun_out/sanitize_memcheck.log
K='tests/test_gpu_wgrad_sk.py::test_splits_agree_and_are_deterministic tests/test_gpu_rank_sym.py::test_symmetric_all_ties_and_tiny'
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest $K -q -x -p no:cacheprovider -k "dims1 or ties" > gpurun_out/sanitize_racecheck.log 2>&1; echo racecheck rc=$?
tail -3 gpurun_out/sanitize_racecheck.log
timeout 1500 $CS --tool synccheck --print-limit 20 python -m pytest $K -q -x -p no:cacheprovider -k "dims1 or ties" > gpurun_out/sanitize_synccheck.log 2>&1; echo synccheck rc=$?
tail -3 gpurun_out/sanitize_synccheck.log
