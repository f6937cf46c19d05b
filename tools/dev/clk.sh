cd $GRAFT_REPO_ROOT
(for i in $(seq 1 30); do nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw --format=csv,noheader; sleep 0.1; done) > gpurun_out/clk.txt &
python - <<'PY'
import sys, time, torch
sys.path.insert(0,'.')
import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import api, configs
case = configs.make(1)
s1 = case.set1
ds1 = P.SpectralDataset(s1.spectral_axis, s1.perturbation_axis, s1.intensities)
plan = api.build_plan(ds1, None, P.PreprocessSpec())[0]
t=time.time()
while time.time()-t < 3:
    for _ in range(50): plan.launch()
    torch.cuda.synchronize()
PY
wait
cat gpurun_out/clk.txt | sort | uniq -c
