mkdir -p gpurun_out/d12
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_guards.py tests/test_gpu_parity.py -q -x > gpurun_out/d12/t1.log 2>&1
tail -3 gpurun_out/d12/t1.log
for cfg in 3 4; do for ws in 1 0; do
  CORR2D_F64_WS=$ws timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/d12/b${cfg}_$ws.json 2> gpurun_out/d12/b${cfg}_$ws.err
  python -c "
import json;d=json.loads([l for l in open('gpurun_out/d12/b${cfg}_$ws.json') if l.startswith('{')][-1]);r=d['roofline']
print($cfg,$ws,'ms/step %.4f K2 %.4f MHz %s'%(d['ms_per_step'],r['kernel_ms'],d['clocks']['sm_mhz']))"
done; done
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_wholemap.py -q -k "cfg3 or cfg4" > gpurun_out/d12/t2.log 2>&1
tail -3 gpurun_out/d12/t2.log
