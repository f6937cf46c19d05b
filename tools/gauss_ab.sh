set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_sharded.py tests/test_gpu_dropin.py tests/test_gpu_streaming.py -x -q 2>&1 | tail -15 > gpurun_out/t3.log
for cfg in 3 4; do
  for fmt in four gauss; do
    CORR2D_F64_FORMAT=$fmt python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${cfg}_${fmt}.json 2>gpurun_out/b_${cfg}_${fmt}.err
  done
done
