cd $GRAFT_REPO_ROOT
for lib in main _variants/libcorr2d_mt1b2.so _variants/libcorr2d_mt1b3.so _variants/libcorr2d_kc16.so main; do
  if [ $lib = main ]; then unset CORR2D_LIB; else export CORR2D_LIB=$lib; fi
  for c in 3 4; do echo "$lib $(timeout 120 python tools/time_contract.py $c 30)"; done
done
