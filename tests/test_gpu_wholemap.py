"""Whole-map parity at the BASELINE.json sizes (parity beyond
sampled rows).

* cfg5 (32768^2, fp32 planes): every element of the tensor-core map -- both
  operand formats, F16F8 (default) and bf16x3 -- against the fp64 DMMA map of
  the same fp32 inputs, which is itself pinned to the reference's rows
  (tests/golden/config5.npz) at 1e-10.  Tolerance 1e-4 of max|sync|
  (north_star).
* cfg3 / cfg4 (fp64): every element against the streamed row-block oracle
  (oracle/corr2d_oracle.py) at 1e-10 of max|sync|.
* F16F8 on adversarial inputs: neighbouring channels (one K1 FFT pair) whose
  magnitudes differ by up to 10^8, and coherent band-limited dynamics (the
  energy of each channel in one or two DFT bins).

Measured worst-case errors are written to $CORR2D_EVIDENCE_DIR (when set) as
JSON; the committed copies live in profiles/."""

import json
import os
from pathlib import Path

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import corr2d_oracle as O
import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import configs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _evidence(name, d):
    out = os.environ.get("CORR2D_EVIDENCE_DIR")
    if out:
        Path(out).mkdir(parents=True, exist_ok=True)
        (Path(out) / f"{name}.json").write_text(json.dumps(d, indent=1))


def _datasets(case, dtype):
    dt = np.float32 if dtype == "float32" else np.float64
    s1 = case.set1
    ds1 = P.SpectralDataset(s1.spectral_axis, s1.perturbation_axis, s1.intensities, dtype=dt)
    ds2 = None
    if case.set2 is not None:
        ds2 = P.SpectralDataset(case.set2.spectral_axis, case.set2.perturbation_axis, case.set2.intensities, dtype=dt)
    return ds1, ds2


def _maxdiff(x, y, rows=2048):
    import torch
    d = 0.0
    for r0 in range(0, x.shape[0], rows):
        d = max(d, float(torch.abs(x[r0:r0 + rows].double() - y[r0:r0 + rows].double()).max()))
    return d


def test_cfg5_whole_map_both_formats_against_fp64(monkeypatch):
    import torch
    case = configs.make(5)
    ds, _ = _datasets(case, "float32")
    ref = P.corr2d(ds, dtype="float64", return_device=True)            # fp64 DMMA from the fp32 inputs
    g = golden("config5")
    rows = g["rows"]
    scale = ref.meta["stats"]["max_abs_sync"]
    assert rel_err(ref.sync[rows].cpu().numpy(), g["sync_rows"], scale) <= 1e-10
    assert rel_err(ref.asyn[rows].cpu().numpy(), g["asyn_rows"], scale) <= 1e-10
    report = {"config": case.name, "scale_max_abs_sync": scale, "reference_rows_rel_err_fp64": max(
        rel_err(ref.sync[rows].cpu().numpy(), g["sync_rows"], scale),
        rel_err(ref.asyn[rows].cpu().numpy(), g["asyn_rows"], scale))}
    for fmt in ("f16f8", "bf16x3"):
        monkeypatch.setenv("CORR2D_FP32_FORMAT", fmt)
        res = P.corr2d(ds, dtype="float32", return_device=True)
        es = _maxdiff(res.sync, ref.sync) / scale
        ea = _maxdiff(res.asyn, ref.asyn) / scale
        report[fmt] = {"sync_rel_err": es, "asyn_rel_err": ea}
        assert es <= 1e-4 and ea <= 1e-4, (fmt, es, ea)
        del res
        torch.cuda.empty_cache()
    _evidence("r2_wholemap_cfg5", report)


@pytest.mark.parametrize("k", [3, 4])
def test_fp64_whole_map_against_streamed_oracle(k):
    case = configs.make(k)
    ds1, ds2 = _datasets(case, "float64")
    res = P.corr2d(ds1, ds2, resample=case.resample, interpolant=case.interpolant, alpha=case.alpha,
                   return_device=True)
    _, v, _, _ = O.preprocess(case.set1.perturbation_axis, case.set1.intensities, resample=case.resample,
                              kind=case.interpolant, alpha=case.alpha)
    n = v.shape[1]
    threads = O.host_threads()
    worst = [0.0, 0.0]
    scale = 0.0
    for r0 in range(0, n, 2048):
        r1 = min(n, r0 + 2048)
        s, a, _ = O.correlate_ft(v[:, r0:r1], v, workers=threads)
        gs = res.sync[r0:r1].cpu().numpy()
        ga = res.asyn[r0:r1].cpu().numpy()
        worst[0] = max(worst[0], float(np.abs(gs - s).max()))
        worst[1] = max(worst[1], float(np.abs(ga - a).max()))
        scale = max(scale, float(np.abs(s).max()), float(np.abs(a).max()))
    err = max(worst) / scale
    _evidence(f"r2_wholemap_cfg{k}", {"config": case.name, "rows": n, "block_rows": 2048,
                                       "sync_max_abs_err": worst[0], "asyn_max_abs_err": worst[1],
                                       "scale": scale, "rel_err": err})
    assert err <= 1e-10


def _adversarial(m, n, seed):
    """Band-limited, coherent dynamics with wildly unequal neighbours."""
    rng = np.random.default_rng(seed)
    t = np.arange(m)
    v = np.empty((m, n))
    for i in range(n):
        f = rng.integers(1, m // 2)                       # one dominant bin per channel
        ph = rng.uniform(0, 2 * np.pi)
        v[:, i] = np.cos(2 * np.pi * f * t / m + ph) + 1e-3 * rng.normal(size=m)
    # K1 transforms channels (2k, 2k + 1) as one complex FFT: make the partners
    # differ by up to 10^8 (and the pairs differ among themselves by 10^6)
    mag = np.empty(n)
    mag[0::2] = 10.0 ** rng.uniform(-3, 3, size=(n + 1) // 2)
    mag[1::2] = mag[0::2][: n // 2] * 10.0 ** rng.uniform(-8, -4, size=n // 2)
    return v * mag


@pytest.mark.parametrize("fmt", ["f16f8", "bf16x3"])
@pytest.mark.parametrize("m", [64, 512, 1024])
def test_fp32_formats_adversarial_unequal_pairs_and_coherent_bands(m, fmt, monkeypatch):
    """m = 64 / 512 run K1's fp32 paired transform (fast kernel), m = 1024 the
    generic fp64 one.  Errors are held to each element's OWN scale: K1 brings
    both channels of a pair to max|x| in [1, 2) before the paired fp32 FFT, so a
    channel 10^8 below its partner keeps its own ~2^-24 transform error."""
    monkeypatch.setenv("CORR2D_FP32_FORMAT", fmt)
    v = _adversarial(m, 640, m)
    dyn = P.DynamicSpectra(np.arange(640.0), np.arange(float(m)), v, np.zeros(640))
    res = P.correlate_ft(dyn, dtype="float32")
    s, a, _ = O.correlate_ft(v)
    sc = max(float(np.abs(s).max()), float(np.abs(a).max()))
    err = max(rel_err(res.sync, s, sc), rel_err(res.asyn, a, sc))
    # own-scale error: each element against the product of its two channels'
    # own magnitudes (sqrt of the diagonal of sync)
    own = np.sqrt(np.abs(np.diag(s)))
    denom = np.outer(own, own)
    own_err = max(float(np.max(np.abs(res.sync - s) / denom)), float(np.max(np.abs(res.asyn - a) / denom)))
    _evidence(f"r2_{fmt}_adversarial_m{m}", {"m": m, "n": 640, "rel_err_vs_max": err,
                                             "own_scale_rel_err": own_err})
    assert err <= 1e-4
    assert own_err <= 1e-4
