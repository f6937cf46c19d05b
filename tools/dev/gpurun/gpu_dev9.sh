#!/bin/bash
CORR2D_LIB=_variants/libcorr2d_prof.so python tools/dev/small_trace.py > gpurun_out/small_trace.log 2>&1
python tools/dev/small_debug.py > gpurun_out/small_debug.log 2>&1
python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_configs.py -q -x 2>&1 | tail -3 > gpurun_out/tests9.log
for cfg in 1 2; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err
done
