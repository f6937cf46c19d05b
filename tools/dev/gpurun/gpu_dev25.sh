cd $GRAFT_REPO_ROOT
./tools/microbench/tilestore_bulk
timeout 600 python -m pytest tests/test_gpu_small_fused.py -x -q 2>&1 | tail -3
for skip in 0 1 2 3; do echo "skip $skip"; CORR2D_DEBUG_SKIP=$skip CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 2 2>&1 | tail -2; done
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 2 --trace 2>&1 | tail -16
