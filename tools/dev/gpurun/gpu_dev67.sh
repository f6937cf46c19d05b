cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_small_fused.py -x -q --timeout 120 -k back_to_back 2>&1 | grep -E "^E |FAILED|passed|failed" | head -20
