cd $GRAFT_REPO_ROOT
for c in 1 2; do
timeout 300 python bench.py --config $c --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg$c', d['ms_per_step']*1e3, 'us', d['value'], d['roofline']['frac'], d['e2e']['value'])"
done
timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg3', d['ms_per_step']*1e3, 'us', d['value'], d['roofline']['frac'], d['e2e']['value'])"
