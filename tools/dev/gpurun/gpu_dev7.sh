#!/bin/bash
mkdir -p gpurun_out/prof
python -m pytest tests/test_gpu_hilbert_big.py tests/test_gpu_hilbert.py -q -x 2>&1 | tail -5 > gpurun_out/tests7.log
./tools/microbench/floor > gpurun_out/floor.json 2>&1
./tools/microbench/peaks > gpurun_out/peaks.json 2>&1
CMD1="python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"small_" -c 2 -o gpurun_out/prof/full_cfg1c $CMD1 > gpurun_out/prof/ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches_cfg1c.csv $CMD1 > gpurun_out/prof/ncu_l1.log 2>&1
CMD2="python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"small_" -c 2 -o gpurun_out/prof/full_cfg2c $CMD2 > gpurun_out/prof/ncu2.log 2>&1
