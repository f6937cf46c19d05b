cd $GRAFT_REPO_ROOT
timeout 120 python tools/dev/small_rot.py 1 200 32 2>&1 | tail -1
timeout 300 python bench.py --config 1 --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg1', d['ms_per_step']*1e3, 'us', d['timing'], d['clocks'])"
timeout 300 python bench.py --config 1 --steps 64 --warmup 20 --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg1', d['ms_per_step']*1e3, 'us', d['timing'], d['clocks'])"
