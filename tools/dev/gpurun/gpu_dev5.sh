#!/bin/bash
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_wholemap.py 2>&1 | tail -15 > gpurun_out/tests5.log
python tools/dev/e2e_phases.py > gpurun_out/e2e_phases.log 2>&1
python -c "import torch,time; torch.cuda.init(); t=time.perf_counter(); [torch.cuda.mem_get_info() for _ in range(100)]; print('mem_get_info us', (time.perf_counter()-t)*1e4)" >> gpurun_out/e2e_phases.log 2>&1
for cfg in 1 2; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err
done
for skip in 0 1 2 3; do
  CORR2D_LIB=_variants/libcorr2d_prof.so CORR2D_DEBUG_SKIP=$skip python tools/time_contract.py 3 > gpurun_out/t3_skip$skip.json 2>&1
done
CMD1="python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"small_block" -c 1 -o gpurun_out/prof/full_cfg1b $CMD1 > gpurun_out/prof/ncu1.log 2>&1
CMD2="python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"small_block" -c 1 -o gpurun_out/prof/full_cfg2b $CMD2 > gpurun_out/prof/ncu2.log 2>&1
