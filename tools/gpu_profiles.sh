# Round-end evidence: full GPU tests, smoke, bench, ncu launch list + --set full captures.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/prof/gpu.txt
nproc >> gpurun_out/prof/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/prof/smoke.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/prof/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/prof/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/prof/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err; echo bench rc=$?
tail -3 gpurun_out/prof/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/prof/bench_ref.json 2> gpurun_out/prof/bench_ref.err; echo ref rc=$?
N="ncu --clock-control none"
timeout 600 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 400 --csv --log-file gpurun_out/prof/launches_train.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-infer --no-hbm --no-finetune --no-search --no-pretrain --profile-steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 $N --set full --import-source on -k regex:"mlp_chain|wgrad_group|rank_cluster|head_backward" -s 16 -c 5 -o gpurun_out/prof/train_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-infer --no-hbm --no-finetune --no-search --no-pretrain --profile-steps 1 > /dev/null 2>&1; echo ncu2 rc=$?
timeout 600 $N --set full --import-source on -k regex:umma_fwd_pair -s 4 -c 2 -o gpurun_out/prof/score_full python tools/gemm_sweep.py pair > /dev/null 2>&1; echo ncu3 rc=$?
timeout 600 $N --set full --import-source on -k regex:"lot_pass1c|lot_apply|lot_max" -c 3 -o gpurun_out/prof/lottery_full python tools/lot_prof.py ratio 1 > /dev/null 2>&1; echo ncu4 rc=$?
timeout 600 $N --set full --import-source on -k regex:"lot_max|lot_apply" -c 2 -o gpurun_out/prof/lottery_thr_full python tools/lot_prof.py threshold 1 > /dev/null 2>&1; echo ncu4b rc=$?
timeout 600 $N --set full --import-source on -k regex:"umma_gram" -c 1 -o gpurun_out/prof/mmd_full python tools/mmd_bench.py > /dev/null 2>&1; echo ncu5 rc=$?
timeout 600 $N --set full --import-source on -k regex:"sgd_kernel|segment_sum" -c 2 -o gpurun_out/prof/hbm_full python tools/hbm_prof.py > /dev/null 2>&1; echo ncu6 rc=$?
timeout 600 $N --set full --import-source on -k regex:"tk_pass" -c 1 -o gpurun_out/prof/topk_full python tools/topk_prof.py > /dev/null 2>&1; echo ncu7 rc=$?
timeout 600 $N --set full --import-source on -k regex:"lot_resident" -c 1 -o gpurun_out/prof/lottery_resident_full python -c "
import sys; sys.path.insert(0,'.'); import numpy as np
from paper_2201_05752_b200 import moseslab as ml
dims=[164,512,512,512,512,1]; p=ml.init_random(dims,1,strict=False); dm=ml.DeviceModel(p, ml.PREC_BF16, 16)
dm.set_gradients(np.random.default_rng(0).normal(0,1e-2,dm.P)); ml.lottery_step(dm, ml.RATIO, 0.5, 0, 1e-3, 1e-2)" > /dev/null 2>&1; echo ncu8 rc=$?
timeout 600 $N --set full --import-source on -k regex:"encode_configs|measure_configs" -c 2 -o gpurun_out/prof/space_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-infer --no-hbm --no-finetune --no-pretrain > /dev/null 2>&1; echo ncu9 rc=$?
# summaries on the box (the .ncu-rep files would exceed gpurun's 64 MiB copy-back limit)
P=gpurun_out/prof
python tools/ncu_summary.py list $P/launches_train.csv $P/r_launches_train_summary.csv
python tools/ncu_summary.py full $P/r_full_summary.csv $P/train_full.ncu-rep $P/score_full.ncu-rep $P/lottery_full.ncu-rep $P/lottery_thr_full.ncu-rep $P/mmd_full.ncu-rep $P/hbm_full.ncu-rep $P/topk_full.ncu-rep $P/lottery_resident_full.ncu-rep $P/space_full.ncu-rep
python tools/ncu_summary.py train-traffic $P/train_full.ncu-rep $P/ncu_traffic.json
mkdir -p $P/keep && mv $P/score_full.ncu-rep $P/keep/ 2>/dev/null
rm -f $P/*.ncu-rep
ls -la $P
