# Iteration session: targeted GPU tests ($TESTS), then the CUPTI step timelines of cfg2 and cfg5.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_wgrad_sk.py} -q -x --timeout 600 > gpurun_out/iter_tests.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/iter_tests.log
CFG=2 timeout 300 python tools/step_prof.py 2>&1 | grep -v -i warn > gpurun_out/timeline_cfg2.txt; echo t2 rc=$?
CFG=5 timeout 300 python tools/step_prof.py 2>&1 | grep -v -i warn > gpurun_out/timeline_cfg5.txt; echo t5 rc=$?
cat gpurun_out/timeline_cfg2.txt gpurun_out/timeline_cfg5.txt
