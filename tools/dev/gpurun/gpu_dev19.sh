cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_prep_paths.py tests/test_gpu_guards.py -x -q 2>&1 | tail -15
for c in 1 2; do echo "$(timeout 120 python tools/one_small.py $c 2>&1 | tail -1)"; done
for c in 1 2; do echo "flush $(timeout 120 python tools/one_small.py $c --flush 2>&1 | tail -1)"; done
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 1 --trace 2>&1 | tail -10
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 120 python tools/one_small.py 2 --trace 2>&1 | tail -10
for c in 1 2; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:small_fused --launch-skip 20 --launch-count 1 -o gpurun_out/fused_cfg$c -f python tools/one_small.py $c > gpurun_out/ncu_fused_$c.log 2>&1
done
ls -la gpurun_out
