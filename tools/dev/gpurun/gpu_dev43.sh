cd $GRAFT_REPO_ROOT
timeout 120 python tools/dev/small_rot.py 1 2>&1 | tail -1
CORR2D_LIB=_variants/libcorr2d_two.so timeout 120 python tools/dev/small_rot.py 1 2>&1 | tail -1
CORR2D_LIB=_variants/libcorr2d_two.so CORR2D_SMALL_STREAM_NB=2 timeout 120 python tools/dev/small_rot.py 1 2>&1 | tail -1
