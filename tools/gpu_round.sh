#!/bin/bash
# GPU batch used during development: full -m gpu suite, then bench lines for the
# configs given as arguments (default 1 2 3 4).  Outputs under gpurun_out/.
cfgs=${@:-1 2 3 4}
python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/tests.log
for cfg in $cfgs; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err
done
