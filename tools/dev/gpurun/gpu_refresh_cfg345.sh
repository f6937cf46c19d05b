cd $GRAFT_REPO_ROOT
OUT=gpurun_out/prof2
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_fetch.py tests/test_gpu_wholemap.py -q --timeout 600 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err; echo cfg5=$?
for c in 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 6 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo cfg$c=$?
done
for c in 5 3 4; do python -c "import json;d=json.load(open('$OUT/bench_cfg$c.json'));print($c, d['value'], d['e2e']['ms_per_step'])"; done
