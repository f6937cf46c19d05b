"""Host-side profile of the public corr2d() call on a small map (cfg1 shape):
per-call wall time, and cProfile's top entries (where the non-PCIe time goes)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch

import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import configs as C

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
case = C.make(cfg)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
ds1 = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, pin(case.set1.intensities))
ds2 = None if case.set2 is None else P.SpectralDataset(case.set2.spectral_axis, case.set2.perturbation_axis,
                                                        pin(case.set2.intensities))
hs = torch.empty((case.n1, case.n2), dtype=torch.float64, pin_memory=True)
ha = torch.empty((case.n1, case.n2), dtype=torch.float64, pin_memory=True)
kw = dict(out=(hs, ha))
for _ in range(5):
    P.corr2d(ds1, ds2, **kw)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    P.corr2d(ds1, ds2, **kw)
dt = (time.perf_counter() - t0) / n
print(f"cfg{cfg} corr2d(): {dt * 1e3:.3f} ms per call; planes {2 * hs.numel() * 8 / 1e6:.1f} MB")
# the D2H alone (the same two planes, pinned, as corr2d queues them)
dev_s = torch.empty_like(hs, device="cuda")
dev_a = torch.empty_like(ha, device="cuda")
from paper_1808_00685_b200 import engine
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    engine.copy_d2h([(hs, dev_s), (ha, dev_a)])
print(f"D2H of both planes alone: {(time.perf_counter() - t0) / n * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    P.corr2d(ds1, ds2, **kw)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
