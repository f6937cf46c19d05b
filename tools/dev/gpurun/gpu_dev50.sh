cd $GRAFT_REPO_ROOT
for R in 8 12 16 32; do timeout 120 python tools/dev/small_rot.py 1 64 $R 2>&1 | tail -1; done
for R in 6 11; do timeout 120 python tools/dev/small_rot.py 2 64 $R 2>&1 | tail -1; done
