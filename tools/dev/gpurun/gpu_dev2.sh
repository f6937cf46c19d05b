#!/bin/bash
# dev batch: gpu tests, cfg1/cfg2 bench, ncu full capture of the cfg3 Gauss contraction and the small kernel
mkdir -p gpurun_out/prof
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_wholemap.py 2>&1 | tail -25 > gpurun_out/tests.log
for cfg in 1 2; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err
done
CMD3="python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"contract_f64" -c 1 -o gpurun_out/prof/full_cfg3g $CMD3 > gpurun_out/prof/ncu3.log 2>&1
CMD1="python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"small_block" -c 1 -o gpurun_out/prof/full_cfg1 $CMD1 > gpurun_out/prof/ncu1.log 2>&1
CMD2="python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"small_block" -c 1 -o gpurun_out/prof/full_cfg2 $CMD2 > gpurun_out/prof/ncu2.log 2>&1
