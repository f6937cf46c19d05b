cd $GRAFT_REPO_ROOT
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/dev/small_trace.py 2>&1 | grep -v "^  K\|small path trace" | head -80
