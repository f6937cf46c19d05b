# Round-2 closing evidence at HEAD (kernels unchanged since the last full
# tools/profile_round2.sh run): bench lines of all configs, the reference arm,
# the full GPU suite, guard-band tests and the ncu launch lists.  Summarised by
# tools/summarize_round2.py (partial runs keep the other committed files).
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/prof2
rm -rf $OUT; mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $OUT/gpu.csv 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err; echo cfg5=$?
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo cfg$c=$?
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_cfg5.json 2> $OUT/bench_reference.err; echo ref=$?
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/gpu_tests.log 2>&1; echo tests=$?; tail -2 $OUT/gpu_tests.log
timeout 900 python -m pytest tests/test_gpu_guards.py -q -rA > $OUT/guards.log 2>&1; echo guards=$?
for c in 5 1 2 3; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_cfg$c.csv $CMD > $OUT/ncu_launch$c.log 2>&1; echo launches$c=$?
done
ls -la $OUT
