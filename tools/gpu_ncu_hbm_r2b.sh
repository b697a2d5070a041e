# ncu --set full of this session's HBM / latency kernels: the one-launch top-k (100M scores) and the
# resident lottery step (P = 873K, split pairs)
cd $GRAFT_REPO_ROOT
KREGEX=tk_fused TAG=ncu_topk_fused SKIP=5 bash tools/gpu_ncu_one.sh python tools/topk_prof.py
KREGEX=lot_resident TAG=ncu_lot_resident SKIP=5 bash tools/gpu_ncu_one.sh python tools/lot_res_prof.py
