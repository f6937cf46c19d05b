cd $GRAFT_REPO_ROOT
timeout 300 python tools/dev/launch_cost.py 1 2>&1 | tail -4
