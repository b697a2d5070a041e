# ncu --set full of the split-bf16 training step's GEMM kernels (fwd chain, dZ chain, grouped wgrad) +
# a per-kernel metric dump read back here. Usage (under gpurun): bash tools/ncu_train_split.sh <tag>
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r2}
P=gpurun_out/prof_$TAG
mkdir -p $P
N="ncu --clock-control none"
timeout 900 $N --set full --import-source on -k regex:"mlp_chain_split|wgrad_sk|rank_cluster|head_backward" -s 12 -c 5 -o $P/train_full python bench.py --steps 3 --warmup 3 --headline-only --profile-steps 1 > $P/ncu_full.log 2>&1; echo ncu rc=$?
timeout 300 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $P/launches_train.csv python bench.py --steps 3 --warmup 3 --headline-only --profile-steps 1 > /dev/null 2>&1; echo ncu list rc=$?
CFG=5 timeout 600 $N --set full --import-source on -k regex:"rank_sym|wgrad_sk" -s 4 -c 2 -o $P/cfg5_full python tools/step_prof.py > $P/ncu_cfg5.log 2>&1; echo ncu cfg5 rc=$?
python tools/ncu_summary.py full $P/full_summary.csv $P/train_full.ncu-rep $P/cfg5_full.ncu-rep
python tools/ncu_summary.py train-traffic $P/train_full.ncu-rep $P/ncu_traffic.json
python tools/ncu_summary.py list $P/launches_train.csv $P/launches_summary.csv
ncu -i $P/train_full.ncu-rep --page details --csv > $P/details.csv 2>/dev/null
rm -f $P/*.ncu-rep
ls -la $P
