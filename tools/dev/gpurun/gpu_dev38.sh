cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_guards.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 120 python tools/dev/small_rot.py 2 2>&1 | tail -1
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 2 --trace 2>&1 | tail -16
timeout 300 python bench.py --config 2 --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg2', d['ms_per_step']*1e3, 'us', d['value'], d['gpu_launches'], d['e2e']['value'], d['clocks']['sm_mhz'])"
