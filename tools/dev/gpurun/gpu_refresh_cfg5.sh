# cfg5 / cfg3 / cfg4 bench lines and the GPU suite after the e2e hand-off change
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/prof2
rm -rf $OUT; mkdir -p $OUT
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err; echo cfg5=$?
for c in 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo cfg$c=$?
done
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/gpu_tests.log 2>&1; echo tests=$?; tail -2 $OUT/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
