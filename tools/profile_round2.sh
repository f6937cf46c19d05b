#!/bin/bash
# Round-2 evidence under gpurun, from the repo root: bench lines (both arms),
# microbenchmarks (peaks, launch / store floors), whole-map parity evidence,
# guard-band (out-of-bounds) tests, the fp64 bound decomposition and the small-path
# trace (profiling build), ncu launch lists and full captures.
# Summarised into profiles/ by tools/summarize_round2.py.
set -u
OUT=gpurun_out/prof2
mkdir -p $OUT/evidence
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $OUT/gpu.csv 2>&1
# 1. microbenchmarks
./tools/microbench/peaks > $OUT/peaks.json 2> $OUT/peaks.err
./tools/microbench/floor > $OUT/floor.json 2> $OUT/floor.err
# 2. bench lines: headline (cfg5, with cpu_baseline), the other configs, the reference arm
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_cfg5.json 2> $OUT/bench_reference.err
timeout 600 python tools/bench_extras.py > $OUT/extras.json 2> $OUT/extras.err
# 3. whole-map parity + adversarial evidence (slow tests) and the full GPU suite
CORR2D_EVIDENCE_DIR=$OUT/evidence timeout 1800 python -m pytest tests/test_gpu_wholemap.py -q > $OUT/wholemap_tests.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1
# 4. fp64 bound decomposition and the small-path trace (profiling build)
for c in 3 4; do
  for skip in 0 1 2 3; do
    CORR2D_LIB=_variants/libcorr2d_prof.so CORR2D_DEBUG_SKIP=$skip timeout 300 python tools/time_contract.py $c > $OUT/decomp_cfg${c}_skip$skip.json 2>&1
  done
done
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 300 python tools/dev/small_trace.py > $OUT/small_trace.txt 2>&1
# small-m step decomposition in the bench's rotation graph (profiling build switches)
{ for c in 1 2; do
    timeout 120 python tools/dev/small_rot.py $c 64 2>&1 | tail -1 | sed "s/^/release: /"
    for skip in 0 1 2 3 4; do
      CORR2D_LIB=_variants/libcorr2d_prof.so CORR2D_DEBUG_SKIP=$skip timeout 120 python tools/dev/small_rot.py $c 64 2>&1 | tail -1 | sed "s/^/skip $skip: /"
    done
    CORR2D_SMALL_ONEKERNEL=1 timeout 120 python tools/dev/small_rot.py $c 64 2>&1 | tail -1 | sed "s/^/one-kernel variant: /"
  done
  echo "skip 1 = no plane stores, 2 = no DMMAs, 3 = neither, 4 = K1 + an empty contraction grid"; } > $OUT/small_decomp.txt
# cfg5 power decomposition (sustained, clocks / power sampled): full, no stores,
# MMA only, stores only (profiling build)
CORR2D_LIB=_variants/libcorr2d_prof.so timeout 600 python tools/ab_power.py 0 1 5 6 > $OUT/power_cfg5.txt 2>&1
# 5. memory-safety: guard-band tests (compute-sanitizer is closed on this pool)
timeout 900 python -m pytest tests/test_gpu_guards.py -q -rA > $OUT/guards.log 2>&1
# 6. ncu: launch lists of the bench commands, full captures of the hot kernels
for c in 5 1 2 3; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_cfg$c.csv $CMD > $OUT/ncu_launch$c.log 2>&1
done
CMD5="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"contract_tc_2sm|prep_fast" -c 2 -o $OUT/full_cfg5 $CMD5 > $OUT/ncu_full5.log 2>&1
CMD3="python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"contract_f64|prep_fast" -c 2 -o $OUT/full_cfg3 $CMD3 > $OUT/ncu_full3.log 2>&1
# small-m path: both kernels of one step late in a rotation (--cache-control none: L2
# already holds other steps' dirty planes, so DRAM traffic is the steady state's, not
# an L2-resident capture's)
for c in 1 2; do
  CMDS="python tools/dev/small_rot.py $c 16"
  ncu --set full --clock-control none --cache-control none --import-source on -k regex:"small_" -s 300 -c 2 -o $OUT/full_cfg$c $CMDS > $OUT/ncu_full$c.log 2>&1
done
# small-m path: single-pass DRAM counters (no replay) of the step's kernels late in a rotation
for c in 1 2; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none \
    -k regex:"small_" -s 400 -c 4 --csv python tools/dev/small_rot.py $c 16 > $OUT/traffic_cfg$c.csv 2> $OUT/traffic_cfg$c.err
done
ncu --set full --clock-control none --import-source on -k regex:"peaks_vec" -c 1 -o $OUT/full_peaks5 python tools/bench_extras.py > $OUT/ncu_peaks.log 2>&1
ls -la $OUT
