"""Per-call wall time of the public corr2d() call on a BASELINE config with
pinned host inputs / outputs (bench.py's e2e leg, call by call):
python tools/dev/e2e_calls.py CONFIG CALLS"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1808_00685_b200 as P  # noqa: E402
from paper_1808_00685_b200 import configs, engine  # noqa: E402


def main():
    c, calls = int(sys.argv[1]), int(sys.argv[2])
    case = configs.make(c)
    dt = np.float32 if case.dtype == "float32" else np.float64
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    s1 = case.set1
    ds = P.SpectralDataset(s1.spectral_axis, s1.perturbation_axis, pin(s1.intensities.astype(dt)), dtype=dt)
    odt = torch.float32 if case.dtype == "float32" else torch.float64
    hs = torch.empty((case.n1, case.n2), dtype=odt, pin_memory=True)
    ha = torch.empty((case.n1, case.n2), dtype=odt, pin_memory=True)
    kw = dict(resample=case.resample, interpolant=case.interpolant, alpha=case.alpha, dtype=case.dtype, out=(hs, ha))
    ts = []
    for _ in range(calls):
        t0 = time.perf_counter()
        P.corr2d(ds, **kw)
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"cfg{c} fill {engine.MIRROR_FILL_PCT} threads {engine.MIRROR_THREADS or 'all'}: "
          f"median {np.median(ts[1:]):.2f} ms, calls " + " ".join(f"{t:.1f}" for t in ts), flush=True)


if __name__ == "__main__":
    main()
