set -x
mkdir -p gpurun_out/d10
cd $GRAFT_REPO_ROOT
for v in 0 1; do
  CORR2D_PAIR_SPLITB=$v timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_wholemap.py -x -q -k "cfg5 or fp32 or f16 or bf16 or tc" > gpurun_out/d10/t_$v.log 2>&1
  for r in 1 2 3; do CORR2D_PAIR_SPLITB=$v timeout 120 python tools/time_contract.py 5 30 >> gpurun_out/d10/k2_$v.json 2>>gpurun_out/d10/k2_$v.err; done
  CORR2D_PAIR_SPLITB=$v timeout 300 python bench.py --config 5 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/d10/b5_$v.json 2>gpurun_out/d10/b5_$v.err
done
tail -3 gpurun_out/d10/t_*.log
cat gpurun_out/d10/k2_*.json
