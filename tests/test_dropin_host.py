"""Host-side drop-in surface against the reference's own messages (no GPU):
SpectralDataset validation (dataset.py:77-100) and the argument checks of the
preprocessing functions (preprocess.py:155-259), compared with the exception
classes and texts the reference raised on the same inputs
(tests/golden/dropin_messages.json, made by make_golden_dropin.py).  Plus
CorrelationSpectra.to_reference() when the reference is importable."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1808_00685_b200 as P
from conftest import GOLDEN, golden

MSG = json.loads((GOLDEN / "dropin_messages.json").read_text())


def _g():
    return golden("dropin_functions")


def _expect(name, fn):
    cls, text = MSG[name]
    with pytest.raises(getattr(P, cls)) as e:
        fn()
    assert str(e.value) == text


def test_spectral_dataset_messages_match_reference():
    g = _g()
    nu, t, raw = g["nu"], g["t"], g["raw"]
    _expect("m_lt_2", lambda: P.SpectralDataset(nu, t[:1], raw[:1]))
    _expect("n_lt_2", lambda: P.SpectralDataset(nu[:1], t, raw[:, :1]))
    _expect("shape", lambda: P.SpectralDataset(nu, t, raw[:, :40]))
    _expect("nonfinite_axis", lambda: P.SpectralDataset(np.where(np.arange(41) == 3, np.nan, nu), t, raw))
    _expect("nonfinite_pert", lambda: P.SpectralDataset(nu, np.where(np.arange(13) == 2, np.inf, t), raw))
    _expect("nonfinite_intensity", lambda: P.SpectralDataset(nu, t, np.where(
        (np.arange(13)[:, None] == 4) & (np.arange(41)[None, :] == 6), np.nan, raw)))
    _expect("duplicate_spectral", lambda: P.SpectralDataset(np.concatenate([nu[:5], nu[4:40]]), t, raw))
    _expect("nonmonotonic_spectral",
            lambda: P.SpectralDataset(np.concatenate([nu[:10], nu[10:][::-1]]), t, raw))
    _expect("pert_not_increasing",
            lambda: P.SpectralDataset(nu, np.concatenate([t[:6], [t[5] - 1.0], t[7:]]), raw))


def test_preprocess_argument_messages_match_reference():
    g = _g()
    nu, t, raw = g["nu"], g["t"], g["raw"]
    ds = P.SpectralDataset(nu, t, raw)
    dyn = P.DynamicSpectra(nu, t, raw - raw.mean(axis=0), raw.mean(axis=0))
    scaled = P.DynamicSpectra(nu, t, raw, raw.mean(axis=0), scaling_exponent=0.5)
    _expect("target_count", lambda: P.resample_equidistant(ds, 3))
    _expect("alpha_range", lambda: P.apply_scaling(dyn, g["sigma_mean"], 1.5))
    _expect("already_scaled", lambda: P.apply_scaling(scaled, g["sigma_mean"], 0.5))
    _expect("sigma_length", lambda: P.apply_scaling(dyn, g["sigma_mean"][:40], 0.5))
    _expect("provided_length", lambda: P.ReferenceSpec.provided(g["provided_ref"][:40]).resolve(ds))


def test_to_reference_round_trip():
    ref_src = Path("/root/reference/pkg/src")
    if ref_src.exists() and str(ref_src) not in sys.path:
        sys.path.append(str(ref_src))
    corrtwo = pytest.importorskip("corrtwo")
    rng = np.random.default_rng(5)
    x = rng.normal(size=(6, 6))
    sync = x + x.T
    asyn = x - x.T
    res = P.CorrelationSpectra(np.arange(6.0), np.arange(6.0), sync, asyn, np.zeros(6), np.zeros(6),
                               0.25, "fourier", True, 0.5)
    r = res.to_reference()
    assert isinstance(r, corrtwo.CorrelationSpectra)
    assert np.array_equal(r.sync, sync) and np.array_equal(r.asyn, asyn)
    assert (r.normalization, r.engine, r.is_homo, r.scaling_exponent) == (0.25, "fourier", True, 0.5)
    f32 = P.CorrelationSpectra._trusted(np.arange(6.0), np.arange(6.0), sync.astype(np.float32),
                                        asyn.astype(np.float32), np.zeros(6), np.zeros(6), 0.25, "fourier",
                                        True, 0.0)
    r32 = f32.to_reference()
    assert r32.sync.dtype == np.float64 and np.array_equal(r32.sync, sync.astype(np.float32).astype(np.float64))
