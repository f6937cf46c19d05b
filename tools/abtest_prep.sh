#!/bin/bash
# prep-kernel timing on cfg5 for several channels-per-CTA settings (experiments)
for C in ${CS:-2 4 8 16}; do CORR2D_PREP_C=$C timeout 300 python -c "
import sys, torch, numpy as np
sys.path.insert(0,'.')
from paper_1808_00685_b200 import api, configs
import paper_1808_00685_b200 as P
case=configs.make(${CFG:-5})
ds=P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities, dtype=np.float32 if case.dtype=='float32' else np.float64)
spec=P.PreprocessSpec(resample=None if case.resample is None else P.ResampleSpec(case.resample, P.InterpolantKind.from_name(case.interpolant)), scaling_exponent=case.alpha)
plan,_=api.build_plan(ds,None,spec,dtype=case.dtype)
for i in range(3): plan.launch_prep_only()
torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20): plan.launch_prep_only()
e1.record(); torch.cuda.synchronize()
print('C', $C, 'prep ms', round(e0.elapsed_time(e1)/20, 4))
"; done
