cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/tests.log
for c in 1 2 3 5; do
 timeout 400 python bench.py --config $c --steps 50 --warmup 10 --no-cpu-baseline --e2e-steps 10 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
 tail -1 gpurun_out/b_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c', d['ms_per_step']*1e3, 'us', d['value'], d['roofline']['frac'], d['gpu_launches'], d['e2e']['value'], d['clocks']['sm_mhz'])"
done
cat gpurun_out/tests.log
