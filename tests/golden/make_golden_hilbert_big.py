"""Golden fixture for the Hilbert route above the reference's DENSE_LIMIT
(hilbert.py:38, :52-61: m > 4096 applies the Hilbert-Noda matrix through its
Toeplitz structure, scipy.linalg.matmul_toeplitz).  Made by running the
REFERENCE (build container):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_hilbert_big.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
import corrtwo as R  # noqa: E402
from corrtwo import hilbert  # noqa: E402

rng = np.random.default_rng(4097)
m, n = 4200, 12
assert m > hilbert.DENSE_LIMIT
t = np.arange(m, dtype=float)
values = rng.normal(size=(m, n)) * np.linspace(0.5, 2.0, n)
dyn = R.DynamicSpectra(np.arange(n, dtype=float), t, values, np.zeros(n))
res = R.correlate_ht(dyn)
ht = hilbert.hilbert_transform(dyn)
np.savez_compressed(HERE / "ht_beyond_dense_m4200.npz", values=values, sync=res.sync, asyn=res.asyn,
                    transformed=ht, norm=np.float64(res.normalization))
print("wrote ht_beyond_dense_m4200.npz")
