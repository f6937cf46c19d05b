"""Host cost of one small-path launch: plan._launch_small() vs the bare C call
with pre-marshalled arguments (no sync; median of 2000)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import api, configs as C, engine

case = C.make(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
ds1 = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities)
plan, _ = api.build_plan(ds1, None, P.PreprocessSpec(), dtype="float64")
for _ in range(10):
    plan.launch()
torch.cuda.synchronize()


def bench(fn, n=2000):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if len(ts) % 200 == 0:
            torch.cuda.synchronize()
    ts.sort()
    return ts[len(ts) // 2] * 1e6


print(f"plan.launch(): {bench(plan.launch):.1f} us")
print(f"engine.stream_handle(): {bench(engine.stream_handle):.1f} us")
print(f"ptr(phi): {bench(lambda: engine.ptr(plan.phi)):.1f} us")
