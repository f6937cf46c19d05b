cd $GRAFT_REPO_ROOT
for skip in 4 3; do echo "skip $skip"; CORR2D_DEBUG_SKIP=$skip CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/dev/small_rot.py 2 2>&1 | tail -1; done
for skip in 4 3 0; do echo "cfg1 skip $skip"; CORR2D_DEBUG_SKIP=$skip CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/dev/small_rot.py 1 2>&1 | tail -1; done
./tools/microbench/floor 2>&1 | tail -12
