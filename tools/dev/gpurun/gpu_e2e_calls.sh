cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for c in 3 4 5; do
    CORR2D_FETCH_FILL_PCT=0 timeout 300 python tools/dev/e2e_calls.py $c 8
    CORR2D_FETCH_FILL_PCT=30 timeout 300 python tools/dev/e2e_calls.py $c 8
    CORR2D_FETCH_FILL_PCT=30 CORR2D_FETCH_THREADS=12 timeout 300 python tools/dev/e2e_calls.py $c 8
    CORR2D_FETCH_FILL_PCT=20 CORR2D_FETCH_THREADS=12 timeout 300 python tools/dev/e2e_calls.py $c 8
  done
done 2>&1 | grep -v Warning | tee gpurun_out/e2e_calls.txt
