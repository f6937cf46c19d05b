#!/usr/bin/env python
"""Timings of the SURVEY 8f rows beside the headline bench (one JSON line each):
Hilbert route (cfg3 map), find_peaks scan (cfg5 device map), serialization
(native formatter vs the reference's per-value repr).  Not part of bench.py's
contract; results go to profiles/<round>_extras.json."""

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def ev():
    import torch
    return torch.cuda.Event(enable_timing=True)


def hilbert_cfg3(steps=10):
    import torch
    import paper_1808_00685_b200 as P
    from paper_1808_00685_b200 import api, configs
    case = configs.make(3)
    ds = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities)
    out = {}
    for eng in ("fourier", "hilbert"):
        plan, _ = api.build_plan(ds, None, P.PreprocessSpec(), engine_name=eng)
        for _ in range(3):
            plan.launch()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        for _ in range(steps):
            plan.launch()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        out[eng] = {"ms_per_call": ms, "GElem_s": case.n1 * case.n2 / ms / 1e6}
    return {"what": "Hilbert route vs Fourier route, cfg3 16384^2 homo fp64, device-resident, K1 + contraction(s)",
            **out}


def peaks_cfg5():
    import torch
    import paper_1808_00685_b200 as P
    from paper_1808_00685_b200 import configs
    case = configs.make(5)
    ds = P.SpectralDataset(case.set1.spectral_axis, case.set1.perturbation_axis, case.set1.intensities,
                           dtype=np.float32)
    dev = P.corr2d(ds, dtype="float32", return_device=True)
    P.find_peaks(dev, 0.1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = P.find_peaks(dev, 0.1)
    t1 = time.perf_counter()
    # the K3 scan alone, CUDA events on the current stream
    from paper_1808_00685_b200 import _abi, engine
    lib = _abi.load()
    idx = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    n = dev.sync.shape[0]
    thr_s = 0.1 * dev.meta["stats"]["max_abs_sync"]
    thr_a = 0.1 * dev.meta["stats"]["max_abs_async"]
    a, b = ev(), ev()
    a.record()
    reps = 5
    for _ in range(reps):
        lib.corr2d_find_peaks(_abi.F32, engine.ptr(dev.sync), engine.ptr(dev.asyn), n, n, n, 1, thr_s, thr_a,
                              engine.ptr(idx), idx.numel(), engine.ptr(cnt), engine.stream_handle())
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    read_bytes = n * n * 8 / 2           # upper-triangle tiles of both fp32 planes
    return {"what": "find_peaks on the cfg5 32768^2 device map (threshold 0.1)",
            "call_s": t1 - t0, "scan_ms": ms, "scan_GBs_upper_triangle": read_bytes / ms / 1e6,
            "cross_peaks": len(rep.cross_peaks), "auto_peaks": len(rep.auto_peaks)}


def serialize_rate():
    import paper_1808_00685_b200 as P
    from paper_1808_00685_b200.serialize import _threads, write_correlation
    rng = np.random.default_rng(0)
    n = 4096
    s = rng.standard_normal((n, n))
    res = P.CorrelationSpectra(axis1=np.arange(n, dtype=float), axis2=np.arange(n, dtype=float), sync=s,
                               asyn=-s.T.copy() * 0 + rng.standard_normal((n, n)), ref1=np.zeros(n),
                               ref2=np.zeros(n), normalization=1.0, engine="fourier", is_homo=False)
    t0 = time.perf_counter()
    pay = write_correlation(res)
    t1 = time.perf_counter()
    vals = 2 * n * n
    sample = s.reshape(-1)[:200000]
    t2 = time.perf_counter()
    ",".join(repr(float(v)) for v in sample)
    t3 = time.perf_counter()
    return {"what": "write_correlation matrix-pair, 4096^2 fp64 (2 planes)", "threads": _threads(),
            "values_per_s": vals / (t1 - t0), "bytes": sum(len(v) for v in pay.values()),
            "python_repr_values_per_s": sample.size / (t3 - t2),
            "speedup_vs_per_value_repr": (vals / (t1 - t0)) / (sample.size / (t3 - t2))}


if __name__ == "__main__":
    for f in (hilbert_cfg3, peaks_cfg5, serialize_rate):
        try:
            print(json.dumps(f()), flush=True)
        except Exception as exc:  # keep the other measurements
            print(json.dumps({"what": f.__name__, "error": repr(exc)}), flush=True)
