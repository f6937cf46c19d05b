cd $GRAFT_REPO_ROOT
for skip in 3 11 19 0 16; do echo "skip $skip"; CORR2D_DEBUG_SKIP=$skip CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/dev/small_rot.py 2 64 2>&1 | tail -1; done
