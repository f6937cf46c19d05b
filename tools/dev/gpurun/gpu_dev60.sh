cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_small_fused.py -x -q -k back_to_back 2>&1 | tail -15
