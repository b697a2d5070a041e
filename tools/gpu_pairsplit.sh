cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_bf16x3.py -q --timeout 300 -k "scoring_pair or cfg4 or predict_and_pen" > gpurun_out/pytest_ps.log 2>&1; echo pytest rc=$?
grep -E "^(FAILED|ERROR)|passed|failed|^E " gpurun_out/pytest_ps.log | head -20
timeout 600 python bench.py --no-cpu-baseline --no-hbm --no-finetune --no-search --no-pretrain --no-cfg5 --steps 20 --warmup 5 > gpurun_out/bench_ps.json 2> gpurun_out/bench_ps.err; echo bench rc=$?
tail -2 gpurun_out/bench_ps.err
python -c "
import json; d=json.load(open('gpurun_out/bench_ps.json')); i=d['infer']; print(i['value'], i['forward_ms'], i['roofline']['frac'], i['first_winners'])"
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ps_launches.csv python tools/prof_infer.py > /dev/null 2>&1; echo ncu2 rc=$?
grep pair_split gpurun_out/ps_launches.csv | head -8 | cut -c1-300
