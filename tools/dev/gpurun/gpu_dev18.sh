cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_prep_paths.py tests/test_gpu_guards.py -x -q 2>&1 | tail -15
for lib in main _variants/libcorr2d_twok.so; do
  if [ $lib = main ]; then unset CORR2D_LIB; else export CORR2D_LIB=$lib; fi
  for c in 1 2; do echo "$lib $(timeout 120 python tools/one_small.py $c 2>&1 | tail -1)"; done
done
unset CORR2D_LIB
for c in 1 2; do echo "flush $(timeout 120 python tools/one_small.py $c --flush 2>&1 | tail -1)"; done
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 1 --trace 2>&1 | tail -12
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 2 --trace 2>&1 | tail -12
