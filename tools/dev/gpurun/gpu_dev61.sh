cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_guards.py -x -q 2>&1 | tail -2
for c in 2 1; do timeout 120 python tools/dev/small_rot.py $c 64 2>&1 | tail -1; done
