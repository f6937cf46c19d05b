"""Maps whose output planes exceed the device budget are computed in row
blocks and streamed to the host (engine.stream_blocks / run_streamed): the
result is bit-identical to the one-launch map.  The budget is forced small
with CORR2D_DEVICE_BUDGET."""

import numpy as np
import pytest

import paper_1808_00685_b200 as P

pytestmark = pytest.mark.gpu


def _dyn(v, shift=0.0):
    m, n = v.shape
    return P.DynamicSpectra(np.arange(n, dtype=float) + shift, np.arange(m, dtype=float), v, np.zeros(n))


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("homo", [True, False])
def test_correlate_ft_streamed_is_bit_identical(monkeypatch, dtype, homo):
    rng = np.random.default_rng(5)
    v1 = rng.normal(size=(64, 700))
    v2 = rng.normal(size=(64, 333))
    d1, d2 = _dyn(v1), (None if homo else _dyn(v2, 0.5))
    if dtype == "float32":
        # row shards run the 1-SM tcgen05 kernel (the whole map, the CTA-pair
        # one): bit-identity holds against the 1-SM whole map
        monkeypatch.setenv("CORR2D_BF16_1SM", "1")
    whole = P.correlate_ft(d1, d2, dtype=dtype)
    monkeypatch.delenv("CORR2D_BF16_1SM", raising=False)
    pair = P.correlate_ft(d1, d2, dtype=dtype)
    n2 = 700 if homo else 333
    elem = 4 if dtype == "float32" else 8
    monkeypatch.setenv("CORR2D_DEVICE_BUDGET", str(2 * elem * n2 * 200))   # ~200 rows -> 128-row blocks
    from paper_1808_00685_b200 import engine
    assert engine.stream_blocks(700, n2, elem, int(engine.device_budget(None))) is not None
    part = P.correlate_ft(d1, d2, dtype=dtype)
    assert np.array_equal(part.sync, whole.sync) and np.array_equal(part.asyn, whole.asyn)
    assert part.is_homo == homo
    scale = float(np.abs(pair.sync).max())
    assert float(np.abs(part.sync - pair.sync).max()) <= 1e-5 * scale
    assert float(np.abs(part.asyn - pair.asyn).max()) <= 1e-5 * scale


def test_corr2d_and_hilbert_streamed(monkeypatch):
    rng = np.random.default_rng(6)
    ds = P.SpectralDataset(np.arange(500.0), np.sort(rng.uniform(0, 10, 37)), rng.normal(size=(37, 500)) + 1.0)
    whole = P.corr2d(ds, resample=64, interpolant="linear", alpha=0.5)
    dyn = P.preprocess_dataset(ds)
    ht = P.correlate_ht(dyn)
    monkeypatch.setenv("CORR2D_DEVICE_BUDGET", str(2 * 8 * 500 * 150))
    part = P.corr2d(ds, resample=64, interpolant="linear", alpha=0.5)
    assert np.array_equal(part.sync, whole.sync) and np.array_equal(part.asyn, whole.asyn)
    assert np.array_equal(part.ref1, whole.ref1) and part.normalization == whole.normalization
    htp = P.correlate_ht(dyn)
    assert np.array_equal(htp.sync, ht.sync) and np.array_equal(htp.asyn, ht.asyn)
