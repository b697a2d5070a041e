cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 > gpurun_out/pytest5.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest5.log | tail -30
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 30 -c 4 -o gpurun_out/prof_gemm python bench.py --steps 3 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu2.log
ls -la gpurun_out
