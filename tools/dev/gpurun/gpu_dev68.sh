cd $GRAFT_REPO_ROOT
for i in 1 2 3 4 5 6 7 8; do timeout 300 python -m pytest tests/test_gpu_small_fused.py -x -q --timeout 120 -k "back_to_back or streamed or reset" 2>&1 | tail -1; done
for c in 1 2; do for r in 1 2; do timeout 60 python tools/dev/small_rot.py $c 64 2>&1 | tail -1; done; done
