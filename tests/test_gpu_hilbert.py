"""Hilbert route on the GPU: correlate_ht against the
reference's own outputs (tests/golden/hilbert_*.npz), the cross-engine
identity FT sync = (m/pi) HT sync, exact homo symmetry, hilbert_transform."""

import numpy as np
import pytest

from conftest import golden, golden_names, rel_err
from oracle import corr2d_oracle as O
import paper_1808_00685_b200 as P

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _dyn(values, t, nu):
    return P.DynamicSpectra(nu, t, values, np.zeros(values.shape[1]))


@pytest.mark.parametrize("name", golden_names("hilbert_"))
def test_correlate_ht_matches_reference(name):
    g = golden(name)
    d1 = _dyn(g["values1"], g["t"], g["nu1"])
    homo = g["values1"].shape == g["values2"].shape and np.array_equal(g["values1"], g["values2"])
    d2 = None if homo else _dyn(g["values2"], g["t"], g["nu2"])
    res = P.correlate_ht(d1, d2)
    assert res.engine == "hilbert" and res.is_homo == homo
    assert res.normalization == float(g["norm"])
    scale = float(np.abs(g["sync"]).max())
    assert rel_err(res.sync, g["sync"], scale) <= TOL
    assert rel_err(res.asyn, g["asyn"], scale) <= TOL
    if homo:
        assert np.array_equal(res.sync, res.sync.T)
        assert np.array_equal(res.asyn, -res.asyn.T)
        assert not np.any(np.diag(res.asyn))


@pytest.mark.parametrize("m,n", [(2, 7), (11, 40), (64, 300), (100, 77), (512, 130)])
def test_cross_engine_sync_identity(m, n):
    """FT sync = (m / pi) * HT sync (test_cross_engine.py:26-43), both on the GPU."""
    rng = np.random.default_rng(m * 1000 + n)
    t = np.linspace(0.0, 3.0, m)
    ds = P.SpectralDataset(np.arange(n, dtype=float), t, rng.normal(size=(m, n)))
    dyn = P.preprocess_dataset(ds)
    ft = P.correlate_ft(dyn)
    ht = P.correlate_ht(dyn)
    scale = float(np.abs(ft.sync).max())
    assert rel_err(ft.sync, (m / np.pi) * ht.sync, scale) <= TOL
    s, a, _ = O.correlate_ht(dyn.values)
    assert rel_err(ht.sync, s, float(np.abs(s).max())) <= TOL
    assert rel_err(ht.asyn, a, float(np.abs(s).max())) <= TOL


def test_hilbert_transform_and_sync_direct():
    rng = np.random.default_rng(7)
    m, n = 37, 53
    dyn = _dyn(rng.normal(size=(m, n)), np.arange(m, dtype=float), np.arange(n, dtype=float))
    z = P.hilbert_transform(dyn)
    want = O.hilbert_noda_matrix(m) @ dyn.values
    assert z.shape == (m, n)
    assert rel_err(z, want, float(np.abs(want).max())) <= 1e-13
    s = P.sync_direct(dyn)
    ws, _, _ = O.correlate_ht(dyn.values)
    assert rel_err(s, ws, float(np.abs(ws).max())) <= TOL
    assert np.array_equal(P.hilbert_noda_matrix(m), O.hilbert_noda_matrix(m))


def test_corr2d_engine_hilbert_and_errors():
    rng = np.random.default_rng(3)
    m, n = 21, 60
    ds = P.SpectralDataset(np.arange(n, dtype=float), np.linspace(0, 1, m), rng.normal(size=(m, n)))
    res = P.corr2d(ds, engine="hilbert")
    assert res.engine == "hilbert" and res.normalization == 1.0 / (m - 1)
    _, values, _, _ = O.preprocess(ds.perturbation_axis, ds.intensities)
    s, a, _ = O.correlate_ht(values)
    assert rel_err(res.sync, s, float(np.abs(s).max())) <= TOL
    assert rel_err(res.asyn, a, float(np.abs(s).max())) <= TOL
    with pytest.raises(P.DataError):
        P.corr2d(ds, engine="hilbert", dtype="float32")
    with pytest.raises(P.DataError):
        P.corr2d(ds, engine="laplace")
