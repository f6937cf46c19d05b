cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_small_fused.py -x -q --timeout 120 2>&1 | tail -12
timeout 300 python -m pytest tests/test_gpu_guards.py tests/test_gpu_configs.py -x -q --timeout 120 2>&1 | tail -3
for c in 1 2; do timeout 60 python tools/dev/small_rot.py $c 64 2>&1 | tail -1; done
