cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_guards.py -x -q 2>&1 | tail -2
for t in 0 1; do
CORR2D_SMALL_TMA_OPS=$t timeout 300 python bench.py --config 2 --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('tma_ops $t cfg2', d['ms_per_step']*1e3, 'us', d['clocks']['sm_mhz'])"
done
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 2 --trace 2>&1 | tail -9
