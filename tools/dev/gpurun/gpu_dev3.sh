#!/bin/bash
python tools/dev/small_debug.py > gpurun_out/small_debug.log 2>&1
python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_parity.py -q -x 2>&1 | tail -15 > gpurun_out/tests3.log
for cfg in 3 4; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err
done
