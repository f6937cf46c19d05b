cd $GRAFT_REPO_ROOT
timeout 300 python tools/dev/e2e_profile.py 1 2>&1 | head -60
