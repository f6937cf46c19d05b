cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_small_fused.py tests/test_gpu_guards.py -q -x 2>&1 | tail -2
for v in prof; do echo "== $v"; CORR2D_LIB=_variants/libcorr2d_$v.so timeout 300 python tools/dev/small_trace.py 2>&1 | grep -E "cfg|K1|K2 after|K2 end"; done
for c in 1 2; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 | python -c "
import json,sys;d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]);print($c,'ms/step',d['ms_per_step']*1e3,'us')"; done
