cd $GRAFT_REPO_ROOT
for skip in 0 1 2 3; do echo "skip $skip"; CORR2D_DEBUG_SKIP=$skip CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/dev/small_rot.py 2 2>&1 | tail -1; done
for skip in 0 1 2 3; do echo "nb2 skip $skip"; CORR2D_SMALL_STREAM_NB=2 CORR2D_DEBUG_SKIP=$skip CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/dev/small_rot.py 2 2>&1 | tail -1; done
