"""K1 execution paths (csrc/prep.cu) give the same planes: the persistent fast
kernel with TMA-loaded raw blocks and a TMA-stored row image (default), the
same kernel with the register copy-out (CORR2D_PREP_TMA_STORE=0) and with
register-staged loads, one block per CTA (CORR2D_PREP_TMA=0) are bit-identical;
the generic Stockham kernel (CORR2D_PREP_FAST=0) agrees within the tolerance.
Ragged channel counts exercise the TMA zero fill of the last block; a row pitch
that is not a multiple of 16 bytes falls back to the register loads."""

import numpy as np
import pytest

from conftest import rel_err
import paper_1808_00685_b200 as P

pytestmark = pytest.mark.gpu

CASES = [
    # m, n1, n2 (None = homo), compute dtype, fp32 operand format
    (64, 1000, None, "float64", None),
    (128, 333, 250, "float64", None),
    (512, 1000, None, "float32", "f16f8"),
    (256, 517, 300, "float32", "bf16x3"),
    (64, 1001, None, "float32", "f16f8"),   # 1001 x 4 B rows: not 16-byte pitched -> register loads
]


def _ds(m, n, seed, dtype):
    rng = np.random.default_rng(seed)
    t = np.arange(m, dtype=float)
    nu = np.arange(n, dtype=float) * 2.0 + 100.0
    x = rng.normal(size=(m, n)) + np.sin(np.outer(t / m * 7.0, np.ones(n))) * rng.uniform(0.5, 2.0, size=n)
    x = x.astype(np.float32 if dtype == "float32" else np.float64)
    return P.SpectralDataset(nu, t, x, dtype=x.dtype)


def _run(monkeypatch, env, m, n1, n2, dtype, fmt):
    for k in ("CORR2D_PREP_FAST", "CORR2D_PREP_TMA", "CORR2D_PREP_TMA_STORE"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    if fmt:
        monkeypatch.setenv("CORR2D_FP32_FORMAT", fmt)
    d1 = _ds(m, n1, 1 + m, dtype)
    d2 = None if n2 is None else _ds(m, n2, 2 + m, dtype)
    res = P.corr2d(d1, d2, dtype=dtype)
    return res.sync, res.asyn


@pytest.mark.parametrize("m,n1,n2,dtype,fmt", CASES)
def test_prep_paths_agree(monkeypatch, m, n1, n2, dtype, fmt):
    base = _run(monkeypatch, {}, m, n1, n2, dtype, fmt)
    for env in ({"CORR2D_PREP_TMA_STORE": "0"}, {"CORR2D_PREP_TMA": "0"}):
        other = _run(monkeypatch, env, m, n1, n2, dtype, fmt)
        assert np.array_equal(base[0], other[0]) and np.array_equal(base[1], other[1]), env
    generic = _run(monkeypatch, {"CORR2D_PREP_FAST": "0"}, m, n1, n2, dtype, fmt)
    scale = float(max(np.abs(generic[0]).max(), np.abs(generic[1]).max()))
    tol = 1e-12 if dtype == "float64" else 1e-4   # fp32: both paths carry the F16F8 / bf16x3 rounding
    assert rel_err(base[0], generic[0], scale) <= tol and rel_err(base[1], generic[1], scale) <= tol


@pytest.mark.parametrize("m,n1,n2,alpha", [(11, 1000, None, 0.0), (21, 2000, 1500, 0.0), (5, 33, 17, 0.5),
                                           (32, 301, None, 1.0), (2, 40, None, 0.5)])
def test_small_m_path_matches_generic(monkeypatch, m, n1, n2, alpha):
    """m <= 32 fp64 (cfg1 / cfg2 shapes): the one-launch fused path (default), the
    two-kernel path with the warp-per-channel-pair K1 and the two-kernel path with
    the generic K1 -- statistics bit-identical (same sequential operations), maps
    within 1e-13 (a direct DFT instead of the Stockham stages, another
    contraction order)."""
    def run(env):
        for k in ("CORR2D_PREP_SMALL", "CORR2D_SMALL_FUSED"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        d1 = _ds(m, n1, 3 + m, "float64")
        d2 = None if n2 is None else _ds(m, n2, 4 + m, "float64")
        return P.corr2d(d1, d2, alpha=alpha)
    fused = run({})
    small = run({"CORR2D_SMALL_FUSED": "0"})
    generic = run({"CORR2D_SMALL_FUSED": "0", "CORR2D_PREP_SMALL": "0"})
    scale = float(max(np.abs(generic.sync).max(), np.abs(generic.asyn).max()))
    for r in (fused, small):
        assert np.array_equal(r.ref1, generic.ref1) and np.array_equal(r.ref2, generic.ref2)
        assert rel_err(r.sync, generic.sync, scale) <= 1e-13 and rel_err(r.asyn, generic.asyn, scale) <= 1e-13
