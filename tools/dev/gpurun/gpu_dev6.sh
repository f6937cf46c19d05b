#!/bin/bash
python tools/dev/small_debug.py > gpurun_out/small_debug.log 2>&1
python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_configs.py tests/test_gpu_dropin.py tests/test_gpu_hilbert_big.py -q -x 2>&1 | tail -15 > gpurun_out/tests6.log
python tools/dev/e2e_phases.py > gpurun_out/e2e_phases.log 2>&1
for cfg in 1 2; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err
done
CMD1="python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"small_" -c 2 -o gpurun_out/prof/full_cfg1c $CMD1 > gpurun_out/prof/ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches_cfg1.csv $CMD1 > gpurun_out/prof/ncu_l1.log 2>&1
