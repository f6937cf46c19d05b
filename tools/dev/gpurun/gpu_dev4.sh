#!/bin/bash
python tools/dev/small_debug.py > gpurun_out/small_debug.log 2>&1
python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_configs.py -q -x 2>&1 | tail -15 > gpurun_out/tests4.log
python tools/dev/e2e_phases.py > gpurun_out/e2e_phases.log 2>&1
for cfg in 1 2; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err
done
# cfg3 bound decomposition of the Gauss contraction (profiling build)
for skip in 0 1 2 3; do
  CORR2D_LIB=_variants/libcorr2d_prof.so CORR2D_DEBUG_SKIP=$skip python tools/time_contract.py 3 > gpurun_out/t3_skip$skip.json 2>&1
done
