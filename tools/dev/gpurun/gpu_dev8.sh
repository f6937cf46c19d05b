#!/bin/bash
mkdir -p gpurun_out/prof
python tools/dev/small_debug.py > gpurun_out/small_debug.log 2>&1
python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_configs.py -q -x 2>&1 | tail -5 > gpurun_out/tests8.log
for cfg in 1 2; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err
done
CMD1="python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches_cfg1d.csv $CMD1 > gpurun_out/prof/ncu_l1.log 2>&1
CMD2="python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches_cfg2d.csv $CMD2 > gpurun_out/prof/ncu_l2.log 2>&1
