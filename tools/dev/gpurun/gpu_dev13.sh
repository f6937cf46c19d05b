mkdir -p gpurun_out/d13
cd $GRAFT_REPO_ROOT
for lib in main _variants/libcorr2d_ws1.so _variants/libcorr2d_ws2.so; do
  if [ $lib = main ]; then unset CORR2D_LIB; else export CORR2D_LIB=$lib; fi
  for r in 1 2; do echo "$lib $(timeout 120 python tools/time_contract.py 3 30)"; done
done
