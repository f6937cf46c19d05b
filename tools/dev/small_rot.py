"""Device time per step of the small-m path the way bench.py times it: an
event-free CUDA graph of K steps rotating over R independent plans (inputs and
planes > 4 x L2), events only around the whole replay.  A/B harness for the
profiling build's switches (CORR2D_DEBUG_SKIP, ...).
usage: python tools/dev/small_rot.py CFG [K]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import api, configs as C

cfg = int(sys.argv[1])
K = int(sys.argv[2]) if len(sys.argv) > 2 else 64
case = C.make(cfg)
ds1 = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities)
ds2 = None if case.set2 is None else P.SpectralDataset(case.set2.spectral_axis, case.set2.perturbation_axis,
                                                        case.set2.intensities)
R = int(sys.argv[3]) if len(sys.argv) > 3 else (12 if cfg == 1 else 8)
plans = [api.build_plan(ds1, ds2, P.PreprocessSpec(), dtype="float64")[0] for _ in range(R)]
for q in plans:
    q.launch()
torch.cuda.synchronize()
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for k in range(K):
            plans[k % R].launch()
torch.cuda.synchronize()
t0 = time.time()
while time.time() - t0 < 0.5:
    g.replay()
    torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
a.record()
for _ in range(reps):
    g.replay()
b.record()
torch.cuda.synchronize()
print(f"cfg{cfg} rotation R={R} K={K}: {a.elapsed_time(b) * 1e3 / (reps * K):.2f} us/step")
