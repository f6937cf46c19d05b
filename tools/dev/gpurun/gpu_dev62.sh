cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_guards.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
