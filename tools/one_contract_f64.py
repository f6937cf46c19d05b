"""One cfg3 fp64 contraction launch (profiling target for ncu; not part of the product)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1808_00685_b200 import api, configs
import paper_1808_00685_b200 as P

case = configs.make(3)
ds = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities)
plan, _ = api.build_plan(ds, None, P.PreprocessSpec())
plan.launch_prep_only()
plan.launch_contract()
plan.launch_contract()
torch.cuda.synchronize()
print("ok")
