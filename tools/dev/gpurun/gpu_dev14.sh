mkdir -p gpurun_out/d14
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_guards.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for lib in main _variants/libcorr2d_c2.so _variants/libcorr2d_c2n6.so _variants/libcorr2d_ws1.so _variants/libcorr2d_ws2.so; do
  if [ $lib = main ]; then unset CORR2D_LIB; else export CORR2D_LIB=$lib; fi
  for c in 3 4; do echo "$lib $(timeout 120 python tools/time_contract.py $c 30)"; done
done
unset CORR2D_LIB
CORR2D_F64_WS=0 timeout 120 python tools/time_contract.py 3 30
