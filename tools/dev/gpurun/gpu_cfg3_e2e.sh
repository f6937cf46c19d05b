cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab3
python -c "import numpy; numpy.show_config()" 2>&1 | grep -i -A3 "blas" | head -8
for f in 0 30; do
  for ob in default 1; do
    if [ $ob = 1 ]; then export OPENBLAS_NUM_THREADS=1 OMP_NUM_THREADS=1; else unset OPENBLAS_NUM_THREADS OMP_NUM_THREADS; fi
    CORR2D_FETCH_FILL_PCT=$f timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 6 > gpurun_out/ab3/f${f}_ob$ob.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab3/f${f}_ob$ob.json'));print('fill $f blas $ob e2e', d['e2e']['ms_per_step'])"
  done
done
unset OPENBLAS_NUM_THREADS OMP_NUM_THREADS
CORR2D_FETCH_FILL_PCT=30 timeout 300 python tools/dev/e2e_calls.py 3 8
