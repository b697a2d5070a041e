cd $GRAFT_REPO_ROOT
timeout 600 python tools/debug_fwd.py 2>&1 | tail -20
