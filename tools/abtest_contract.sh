#!/bin/bash
# A/B timing of the bf16x3 contraction on cfg5 (experiments; not part of the product)
for lib in ${LIBS:-paper_1808_00685_b200/libcorr2d.so}; do
for dbg in ${DBGS:-0 1 2 3}; do CORR2D_LIB=$lib CORR2D_DEBUG_SKIP=$dbg timeout 300 python -c "
import sys, torch, numpy as np
sys.path.insert(0,'.')
from paper_1808_00685_b200 import api, configs
import paper_1808_00685_b200 as P
case=configs.make(5)
ds=P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities, dtype=np.float32)
plan,_=api.build_plan(ds,None,P.PreprocessSpec(),dtype='float32')
plan.launch_prep_only(); torch.cuda.synchronize()
for i in range(3): plan.launch_contract()
torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(10): plan.launch_contract()
e1.record(); torch.cuda.synchronize()
print('lib', '$lib'.split('/')[-1], 'dbg', $dbg, 'contract ms', round(e0.elapsed_time(e1)/10, 4))
"; done; done
