# ncu --set full of one kernel ($KREGEX) launched by the command "$@"; report to gpurun_out/$TAG.ncu-rep
cd $GRAFT_REPO_ROOT
timeout 600 ncu --clock-control none --set full --import-source on -k regex:"$KREGEX" -s ${SKIP:-3} -c 1 -o gpurun_out/$TAG "$@" > gpurun_out/$TAG.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/$TAG.log
