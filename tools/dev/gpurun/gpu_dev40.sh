cd $GRAFT_REPO_ROOT
for st in 0 800 1500 2500; do echo "stagger $st"; CORR2D_SMALL_STAGGER=$st timeout 120 python tools/dev/small_rot.py 2 2>&1 | tail -1; done
