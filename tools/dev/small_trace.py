"""Per-phase timeline of the small-m path (profiling build, CORR2D_SMALL_TRACE=1)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import api, configs

for cfg in (1, 2):
    case = configs.make(cfg)
    s1 = case.set1
    ds1 = P.SpectralDataset(s1.spectral_axis, s1.perturbation_axis, s1.intensities)
    ds2 = None if case.set2 is None else P.SpectralDataset(case.set2.spectral_axis, case.set2.perturbation_axis,
                                                          case.set2.intensities)
    plans = [api.build_plan(ds1, ds2, P.PreprocessSpec())[0] for _ in range(8)]
    for q in plans:
        q.launch()
    torch.cuda.synchronize()
    # a cold-ish step: other plans' outputs in between
    for q in plans[:-1]:
        q.launch()
    print(f"cfg{cfg}:", file=sys.stderr, flush=True)
    import os
    os.environ["CORR2D_SMALL_TRACE"] = "1"
    plans[-1].launch()
    torch.cuda.synchronize()
    os.environ["CORR2D_SMALL_TRACE"] = "0"

# the same plan back to back (its operand rows and code warm in L2), then one
# traced step after an idle gap (the previous step's output drain finished)
import time
for cfg in (1, 2):
    case = configs.make(cfg)
    s1 = case.set1
    ds1 = P.SpectralDataset(s1.spectral_axis, s1.perturbation_axis, s1.intensities)
    ds2 = None if case.set2 is None else P.SpectralDataset(case.set2.spectral_axis, case.set2.perturbation_axis,
                                                          case.set2.intensities)
    plan = api.build_plan(ds1, ds2, P.PreprocessSpec())[0]
    for _ in range(5):
        plan.launch()
    torch.cuda.synchronize()
    for label, gap in (("warm, back to back", False), ("warm, after idle", True)):
        for _ in range(3):
            plan.launch()
        if gap:
            torch.cuda.synchronize()
            time.sleep(0.01)
        print(f"cfg{cfg} {label}:", file=sys.stderr, flush=True)
        os.environ["CORR2D_SMALL_TRACE"] = "1"
        plan.launch()
        torch.cuda.synchronize()
        os.environ["CORR2D_SMALL_TRACE"] = "0"
