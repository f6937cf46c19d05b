"""The Hilbert route above the reference's DENSE_LIMIT (hilbert.py:38, :52-61):
for m > 4096 the reference applies the Hilbert-Noda matrix through its
Toeplitz structure (scipy matmul_toeplitz); here the same matrix is applied by
the FP64 tensor-core contraction against its rows, for any m.  Pinned to the
reference's own outputs at m = 4200 (tests/golden/ht_beyond_dense_m4200.npz,
make_golden_hilbert_big.py)."""

import numpy as np
import pytest

from conftest import golden, rel_err
import paper_1808_00685_b200 as P

pytestmark = pytest.mark.gpu


def test_hilbert_route_above_dense_limit_matches_reference():
    g = golden("ht_beyond_dense_m4200")
    v = g["values"]
    m, n = v.shape
    dyn = P.DynamicSpectra(np.arange(n, dtype=float), np.arange(m, dtype=float), v, np.zeros(n))
    res = P.correlate_ht(dyn)
    sc = max(float(np.abs(g["sync"]).max()), float(np.abs(g["asyn"]).max()))
    assert rel_err(res.sync, g["sync"], sc) <= 1e-10
    assert rel_err(res.asyn, g["asyn"], sc) <= 1e-10
    assert res.normalization == float(g["norm"]) and res.engine == "hilbert"
    assert np.array_equal(res.sync, res.sync.T) and np.array_equal(res.asyn, -res.asyn.T)
    ht = P.hilbert_transform(dyn)
    assert rel_err(ht, g["transformed"]) <= 1e-10
