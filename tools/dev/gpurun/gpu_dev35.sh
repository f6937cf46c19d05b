cd $GRAFT_REPO_ROOT
for skip in 0 1; do CORR2D_DEBUG_SKIP=$skip CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 2 --trace 2>&1 | tail -9; done
