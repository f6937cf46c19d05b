cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_guards.py -x -q 2>&1 | tail -2
timeout 120 python tools/dev/small_rot.py 1 200 32 2>&1 | tail -1
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 1 --trace 2>&1 | tail -14
