#!/bin/bash
# A/B timing of the bf16x3 contraction on cfg5 (experiments; not part of the product).
# VARIANTS: '|'-separated env settings, e.g. VARIANTS="CORR2D_MIRROR_REG=0|CORR2D_MIRROR_REG=1"
# Each variant also checks a few rows against the default kernel's output.
IFS='|' read -ra VS <<< "${VARIANTS:-CORR2D_DEBUG_SKIP=0}"
for rep in $(seq ${ROUNDS:-1}); do for v in "${VS[@]}"; do env $v timeout 300 python -c "
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
for i in range(${REPS:-10}): plan.launch_contract()
e1.record(); torch.cuda.synchronize()
s, a = plan.phi, plan.psi
rows = [0, 1, 127, 128, 5000, 32767]
cs = float(s[rows].double().abs().sum()); ca = float(a[rows].double().abs().sum())
cols = float(s[:, 4097].double().abs().sum() + a[:, 30001].double().abs().sum())
print('$v', 'contract ms', round(e0.elapsed_time(e1)/${REPS:-10}, 4), 'chk', '%.9e %.9e %.9e' % (cs, ca, cols))
"; done; done
