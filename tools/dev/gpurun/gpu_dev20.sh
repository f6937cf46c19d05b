cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_prep_paths.py tests/test_gpu_guards.py tests/test_gpu_dropin.py -x -q 2>&1 | tail -5
for lib in main _variants/libcorr2d_twok.so _variants/libcorr2d_fused.so; do
  if [ $lib = main ]; then unset CORR2D_LIB; else export CORR2D_LIB=$lib; fi
  for c in 1 2; do
    timeout 300 python bench.py --config $c --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib cfg$c', d['ms_per_step']*1e3, 'us', d['value'], d['gpu_launches'], d['e2e']['value'], d['clocks'])"
  done
done
