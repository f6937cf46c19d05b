cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_guards.py -x -q 2>&1 | tail -3
for nb in 0 2; do for skip in 0 1 2 3; do echo "nb $nb skip $skip"; CORR2D_SMALL_STREAM_NB=$nb CORR2D_DEBUG_SKIP=$skip CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 2 2>&1 | tail -1; done; done
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 2 --trace 2>&1 | tail -10
timeout 300 python bench.py --config 2 --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg2', d['ms_per_step']*1e3, 'us', d['value'], d['gpu_launches'], d['e2e']['value'], d['clocks']['sm_mhz'])"
