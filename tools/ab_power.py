"""Sustained timing of the cfg5 contraction with nvidia-smi clocks / power
sampled during the loop, for the CORR2D_DEBUG_SKIP variants (experiments)."""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402  (ClockSampler)
import paper_1808_00685_b200 as P  # noqa: E402
from paper_1808_00685_b200 import api, configs  # noqa: E402

case = configs.make(5)
ds = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities, dtype=np.float32)
plan, _ = api.build_plan(ds, None, P.PreprocessSpec(), dtype='float32')
plan.launch_prep_only()
torch.cuda.synchronize()
for dbg in sys.argv[1:] or ["0"]:
    os.environ["CORR2D_DEBUG_SKIP"] = dbg
    for _ in range(20):
        plan.launch_contract()
    torch.cuda.synchronize()
    q = "clocks.sm,power.draw"
    proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "50"],
                            stdout=subprocess.PIPE, text=True)
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(300):
        plan.launch_contract()
    e1.record()
    torch.cuda.synchronize()
    proc.terminate()
    rows = [l.split(",") for l in proc.stdout.read().strip().splitlines() if l.strip()]
    clk = [float(r[0]) for r in rows if len(r) == 2]
    pw = [float(r[1]) for r in rows if len(r) == 2]
    print(f"dbg {dbg}: {e0.elapsed_time(e1) / 300:.4f} ms  sm MHz median {np.median(clk):.0f}  power W median {np.median(pw):.0f}",
          flush=True)
