# Diagnostics session: TMA ingest vs producer warps, CUPTI step timelines of cfg2 and cfg5.
cd $GRAFT_REPO_ROOT
timeout 300 ./tools/tma_bench.bin > gpurun_out/tma_bench.json 2>&1; echo tma rc=$?
CFG=2 timeout 300 python tools/step_prof.py > gpurun_out/timeline_cfg2.txt 2>&1; echo t2 rc=$?
CFG=5 timeout 300 python tools/step_prof.py > gpurun_out/timeline_cfg5.txt 2>&1; echo t5 rc=$?
tail -40 gpurun_out/timeline_cfg5.txt
