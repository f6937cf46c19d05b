"""Event-timed back-to-back contraction launches of one config (K2 alone, after
one K1): the tool behind the bound decompositions in profiles/ (run with a
profiling build, CORR2D_LIB=_variants/libcorr2d_prof.so CORR2D_DEBUG_SKIP=1|2,
to drop the stores or the MMAs).  Not part of the product."""
import json
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1808_00685_b200 import api, configs
import paper_1808_00685_b200 as P

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
case = configs.make(cfg)
dt = np.float32 if case.dtype == "float32" else np.float64
ds = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities, dtype=dt)
spec = P.PreprocessSpec(resample=None if case.resample is None else P.ResampleSpec(
    case.resample, P.InterpolantKind.from_name(case.interpolant)), scaling_exponent=case.alpha)
plan, _ = api.build_plan(ds, None, spec, dtype=case.dtype)
plan.launch_prep_only()
for _ in range(5):
    plan.launch_contract()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    plan.launch_contract()
b.record()
torch.cuda.synchronize()
print(json.dumps({"config": cfg, "kernel_ms": a.elapsed_time(b) / reps, "reps": reps}))
