"""Time one configuration's device step (plan.launch) back to back with CUDA
events after 0.5 s of the same load (steady clocks), no L2 flush -- A/B
experiments on the small-m paths (cfg1 / cfg2).  With --trace, one more launch
runs with CORR2D_SMALL_TRACE=1 right after the loaded period (per-phase
globaltimer stamps of the fused kernel, printed by the library).
usage: python tools/one_small.py CFG [--trace]"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import api, configs as C

cfg = int(sys.argv[1])
trace = "--trace" in sys.argv
flush = "--flush" in sys.argv      # bench.py's L2 condition: a 256 MB write before every step
case = C.make(cfg)
dev = torch.device("cuda", 0)
ds1 = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities)
ds2 = None if case.set2 is None else P.SpectralDataset(case.set2.spectral_axis, case.set2.perturbation_axis,
                                                        case.set2.intensities)
plan, _ = api.build_plan(ds1, ds2, P.PreprocessSpec(), dtype="float64", device=dev)
for _ in range(10):
    plan.launch()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(40)]
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for k in range(20):
            if flush:
                buf.fill_(1)
            ev[2 * k].record(s)
            plan.launch()
            ev[2 * k + 1].record(s)
torch.cuda.synchronize()
t0 = time.time()
while time.time() - t0 < 0.5:          # steady clocks before anything is timed
    for _ in range(50):
        g.replay()
    torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 50
a.record()
for _ in range(reps):
    g.replay()
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) * 1e3 / (reps * 20)
if flush:   # per-step events of the last replay (the flush is outside them)
    us = sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(20)) * 1e3 / 20
if trace:
    for _ in range(50):
        g.replay()
    if flush:
        buf.fill_(1)
    os.environ["CORR2D_SMALL_TRACE"] = "1"
    plan.launch()
    os.environ.pop("CORR2D_SMALL_TRACE")
print(f"cfg{cfg} small={getattr(plan, 'small', False)} flush={flush} graph {us:.2f} us/step")
