"""Locate disagreements of the one-kernel small-m path against the oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1808_00685_b200 as P
from oracle import corr2d_oracle as O


def dyn(v, shift=0.0):
    m, n = v.shape
    return P.DynamicSpectra(np.arange(n, dtype=float) + shift, np.arange(m, dtype=float), v, np.zeros(n))


for (m, n1, n2) in [(21, 130, 70), (21, 200, 130), (11, 130, 70), (21, 2000, 1500), (5, 64, 64), (21, 64, 64)]:
    rng = np.random.default_rng(m + n1)
    v1 = rng.normal(size=(m, n1))
    v2 = rng.normal(size=(m, n2))
    res = P.correlate_ft(dyn(v1), dyn(v2, 0.5))
    s, a, _ = O.correlate_ft(v1, v2)
    sc = max(np.abs(s).max(), np.abs(a).max())
    ds = np.abs(res.sync - s) / sc
    da = np.abs(res.asyn - a) / sc
    bad = np.argwhere((ds > 1e-10) | (da > 1e-10))
    print(m, n1, n2, "max", ds.max(), da.max(), "bad", len(bad), bad[:5].tolist(),
          "rows", np.unique(bad[:, 0] // 64)[:10].tolist() if len(bad) else [],
          "cols", np.unique(bad[:, 1] // 64)[:10].tolist() if len(bad) else [])
