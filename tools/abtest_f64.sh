#!/bin/bash
# A/B timing of the fp64 contraction on cfg3 for library variants (experiments)
for lib in ${LIBS:-paper_1808_00685_b200/libcorr2d.so}; do CORR2D_LIB=$lib timeout 300 python -c "
import sys, torch, numpy as np
sys.path.insert(0,'.')
from paper_1808_00685_b200 import api, configs
import paper_1808_00685_b200 as P
case=configs.make(${CFG:-3})
ds=P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities)
spec=P.PreprocessSpec(resample=None if case.resample is None else P.ResampleSpec(case.resample, P.InterpolantKind.from_name(case.interpolant)), scaling_exponent=case.alpha)
plan,_=api.build_plan(ds,None,spec)
plan.launch_prep_only(); torch.cuda.synchronize()
for i in range(3): plan.launch_contract()
torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20): plan.launch_contract()
e1.record(); torch.cuda.synchronize()
s=float(plan.phi[::997].double().abs().sum()); a=float(plan.psi[::991].double().abs().sum())
print('$lib'.split('/')[-1], 'cfg${CFG:-3} contract ms', round(e0.elapsed_time(e1)/20, 4), 'chk %.12e %.12e' % (s, a))
"; done
