"""One cfg5 contraction launch (profiling target for ncu; not part of the product)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1808_00685_b200 import api, configs
import paper_1808_00685_b200 as P

case = configs.make(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
ds = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities,
                       dtype=np.float32 if case.dtype == "float32" else np.float64)
plan, _ = api.build_plan(ds, None, P.PreprocessSpec(), dtype=case.dtype)
plan.launch_prep_only()
plan.launch_contract()
plan.launch_contract()
torch.cuda.synchronize()
print("ok")
