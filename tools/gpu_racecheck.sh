cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
K='tests/test_gpu_wgrad_sk.py::test_splits_agree_and_are_deterministic tests/test_gpu_rank_sym.py::test_symmetric_all_ties_and_tiny tests/test_gpu_chain_pair.py::test_pair_chain_bit_identical'
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest $K -q -x -p no:cacheprovider -k "dims1 or ties or (dims0 and 300)" > gpurun_out/sanitize_racecheck.log 2>&1; echo racecheck rc=$?
tail -3 gpurun_out/sanitize_racecheck.log
grep -A3 "Race reported" gpurun_out/sanitize_racecheck.log | head -20
