cd $GRAFT_REPO_ROOT
for mode in fast fast fast; do
  f=0
  for i in $(seq 1 8); do
    if [ $mode = slow ]; then export MOSES_HB_SLOW=1; else unset MOSES_HB_SLOW; fi
    timeout 120 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py -q -m gpu --timeout 120 -x -k "fused_train_step or pooled_train_graph or train_graph_matches or chain_pooled" > /tmp/o.log 2>&1 || { f=$((f+1)); grep FAILED /tmp/o.log | head -2; }
  done
  echo "$mode failures: $f / 8"
done
