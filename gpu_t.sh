cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 100 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 40 --warmup 20 --no-cpu-baseline --no-infer --profile-steps 1 > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_summary.py list gpurun_out/launches2.csv gpurun_out/launches2_summary.csv; cat gpurun_out/launches2_summary.csv
