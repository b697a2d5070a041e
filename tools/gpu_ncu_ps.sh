cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_split -s 2 -c 2 -o gpurun_out/ps_full python tools/prof_infer.py > gpurun_out/ncu_ps.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_ps.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ps_launches.csv python tools/prof_infer.py > /dev/null 2>&1; echo ncu2 rc=$?
