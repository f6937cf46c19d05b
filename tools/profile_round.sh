#!/bin/bash
# Round evidence: bench lines (both arms), launch list and one full ncu capture
# of each hot kernel.  Run under gpurun from the repo root.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $OUT/gpu.csv 2>&1
# 1. headline bench (cfg5) with cpu_baseline, then the other configs
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_cfg5.json 2> $OUT/bench_reference.err
timeout 600 python tools/bench_extras.py > $OUT/extras.json 2> $OUT/extras.err
# 2. launch list of the headline command (per-launch device time, cold / serialised)
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_cfg5.csv $CMD > $OUT/ncu_launch.log 2>&1
# 3. full captures: contraction + K1 on cfg5 and cfg3, the peak scan on cfg5
ncu --set full --clock-control none --import-source on -k regex:"contract_tc_2sm|prep_fast" -c 2 -o $OUT/full_cfg5 $CMD > $OUT/ncu_full5.log 2>&1
CMD3="python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD3 > $OUT/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"contract_f64|prep_fast" -c 2 -o $OUT/full_cfg3 $CMD3 > $OUT/ncu_full3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"peaks_vec" -c 1 -o $OUT/full_peaks5 python tools/bench_extras.py > $OUT/ncu_peaks.log 2>&1
# the one-launch small-m kernel (cfg1 / cfg2) and its launch lists
for c in 1 2; do
  CMDS="python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
  ncu --set full --clock-control none --import-source on -k regex:"small_fused" -c 1 -o $OUT/full_cfg$c $CMDS > $OUT/ncu_full$c.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_cfg$c.csv $CMDS > $OUT/ncu_launch$c.log 2>&1
done
ls -la $OUT
