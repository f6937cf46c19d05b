cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 2>&1 | grep -v "^\.\|passed" | tail -40
