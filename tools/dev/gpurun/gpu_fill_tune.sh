cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for c in 5 3; do
    for f in 15 20 30; do
      CORR2D_FETCH_FILL_PCT=$f timeout 300 python tools/dev/e2e_calls.py $c 8
    done
  done
done 2>&1 | grep -v Warning | tee gpurun_out/fill_tune.txt
