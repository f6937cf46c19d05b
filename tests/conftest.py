import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libcorr2d.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def golden_names(prefix):
    return sorted(p.stem for p in GOLDEN.glob(f"{prefix}*.npz"))


def rel_err(got, want, scale=None):
    got = np.asarray(got)
    want = np.asarray(want)
    if not (np.iscomplexobj(got) or np.iscomplexobj(want)):
        got = got.astype(np.float64)
        want = want.astype(np.float64)
    if scale is None:
        scale = max(float(np.abs(want).max()), 1e-300)
    return float(np.abs(got - want).max()) / scale
