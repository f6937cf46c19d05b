"""Where the host time of a small-map corr2d() call goes (cfg1 / cfg2 shapes)."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import api, configs, engine

for cfg in (1, 2):
    case = configs.make(cfg)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    s1 = case.set1
    ds1 = P.SpectralDataset(s1.spectral_axis, s1.perturbation_axis, pin(s1.intensities))
    ds2 = None if case.set2 is None else P.SpectralDataset(case.set2.spectral_axis, case.set2.perturbation_axis,
                                                          pin(case.set2.intensities))
    hs = torch.empty((case.n1, case.n2), dtype=torch.float64, pin_memory=True)
    ha = torch.empty((case.n1, case.n2), dtype=torch.float64, pin_memory=True)
    for _ in range(3):
        P.corr2d(ds1, ds2, out=(hs, ha))
    torch.cuda.synchronize()
    N = 20
    t0 = time.perf_counter()
    for _ in range(N):
        P.corr2d(ds1, ds2, out=(hs, ha))
    full = (time.perf_counter() - t0) / N
    spec = P.PreprocessSpec()
    t = {}
    for name in ("plan", "launch", "sync", "check", "fetch"):
        t[name] = 0.0
    for _ in range(N):
        a = time.perf_counter()
        plan, homo = api._cached_plan(ds1, ds2, spec, norm=None, on_zero_variance="error", dtype="float64",
                                      device=None, engine_name="fourier")
        b = time.perf_counter()
        plan.launch()
        c = time.perf_counter()
        engine.sync()
        d = time.perf_counter()
        plan.check(axes=(ds1.spectral_axis, (ds2 or ds1).spectral_axis))
        e = time.perf_counter()
        plan.fetch((hs, ha))
        f = time.perf_counter()
        for k, v in zip(t, (b - a, c - b, d - c, e - d, f - e)):
            t[k] += v / N
    print(cfg, "corr2d ms", round(full * 1e3, 3), {k: round(v * 1e3, 3) for k, v in t.items()},
          "cache", len(api._PLAN_CACHE))
