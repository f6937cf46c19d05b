cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 1 2; do
timeout 300 python bench.py --config $c --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg$c', d['ms_per_step']*1e3, 'us', d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'])"
done
