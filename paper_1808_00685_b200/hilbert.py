"""Hilbert-route correlation engine drop-in (reference: hilbert.py:1-115).

    sync(nu1, nu2)  = Norm * sum_j y1(nu1, t_j) y2(nu2, t_j)
    async(nu1, nu2) = Norm * sum_j y1(nu1, t_j) (N y2)(nu2, t_j),
    N[j, k] = 0 if j == k else 1 / (pi (k - j)),   Norm default 1/(m - 1).

GPU execution reuses the Fourier route's kernels with time-domain operands:
K1 (``corr2d_prep`` with CORR2D_PACK_F64_TIME) writes A_phi = Norm * y1 and
B = y2 without a DFT; because N is skew-symmetric, async = (-N y1)^T y2, so
A_psi = -Norm * N y1 comes from one ``corr2d_contract_f64`` call of A_phi
against the rows of -N (an n1 x m contraction); the second call writes the
sync / async planes exactly as on the Fourier route (FP64 DMMA, homo tiles
mirrored so async is exactly skew-symmetric).  The dense N is applied for
every m (the reference switches to a Toeplitz product above m = 4096,
hilbert.py:34-60 -- the same linear map).
"""

from __future__ import annotations

import numpy as np

from . import _abi, engine
from .dataset import CorrelationSpectra
from .engine_core import NormalizationSpec, check_pair, is_same_dynamic
from .errors import DataError
from .fourier import DeviceCorrelationSpectra


def hilbert_noda_matrix(m: int) -> np.ndarray:
    """The m x m skew-symmetric Hilbert-Noda matrix (hilbert.py:40-48); host only."""
    if m < 2:
        raise DataError(f"need m >= 2, got {m}")
    idx = np.arange(m)
    with np.errstate(divide="ignore"):
        matrix = 1.0 / (np.pi * (idx[None, :] - idx[:, None]))
    np.fill_diagonal(matrix, 0.0)
    return matrix


def _plan(dyn1, dyn2, norm, rows, device):
    homo = dyn2 is None or is_same_dynamic(dyn1, dyn2)
    if dyn2 is None:
        dyn2 = dyn1
    check_pair(dyn1, dyn2)
    norm = norm or NormalizationSpec.unit()
    constant = norm.constant(dyn1.m)
    _, dev = engine.require_device(device)
    recipe = engine.PrepRecipe(m_in=dyn1.m, m=dyn1.m, ref_mode=_abi.REF_NONE)
    plan = engine.CorrelationPlan(n1=dyn1.n, n2=dyn2.n, m=dyn1.m, recipe1=recipe,
                                  recipe2=None if homo else recipe, norm=constant, dtype="float64",
                                  rows=rows, device=dev, want_ref=False, route="hilbert")
    plan.bind(dyn1.device_values(dev), None if homo else dyn2.device_values(dev))
    return plan, homo, dyn2, constant


@engine.on_device
def correlate_ht(dyn1, dyn2=None, norm: NormalizationSpec | None = None, workers: int = 1, *,
                 out=None, return_device: bool = False, device=None, rows=None) -> CorrelationSpectra:
    """Synchronous and asynchronous correlation via the Hilbert route
    (hilbert.py:92-115).  Same keyword-only extras as ``correlate_ft``."""
    if workers < 1:
        raise DataError(f"workers must be >= 1, got {workers}")
    homo = dyn2 is None or is_same_dynamic(dyn1, dyn2)
    d2 = None if homo else dyn2
    dynb = dyn1 if homo else dyn2
    check_pair(dyn1, dynb)
    constant = (norm or NormalizationSpec.unit()).constant(dyn1.m)
    meta = dict(axis1=dyn1.spectral_axis, axis2=dynb.spectral_axis, ref1=dyn1.reference_used,
                ref2=dynb.reference_used, normalization=constant, engine="hilbert",
                is_homo=homo, scaling_exponent=dyn1.scaling_exponent)
    if not return_device and rows is None:
        _, dev = engine.require_device(device)
        blocks = engine.maybe_stream_blocks(dyn1.n, dynb.n, 8, dev)
        if blocks is not None:        # planes larger than device memory: stream row blocks
            s, a, info, _ = engine.run_streamed(lambda rws: _plan(dyn1, d2, norm, rws, device)[0],
                                                dyn1.n, dynb.n, np.float64, blocks, out)
            return CorrelationSpectra._trusted(sync=s, asyn=a, stats=info, **meta)
    plan, homo, dyn2, constant = _plan(dyn1, d2, norm, rows, device)
    plan.launch()
    engine.sync()
    *_, info = plan.check()
    meta["stats"] = info
    if return_device:
        return DeviceCorrelationSpectra(plan, meta)
    if rows is not None and (plan.row0, plan.row1) != (0, dyn1.n):
        raise DataError("a row-sharded call needs return_device=True")
    s, a = plan.fetch(out)
    return CorrelationSpectra._trusted(sync=s, asyn=a, **meta)


@engine.on_device
def sync_direct(dyn1, dyn2=None, norm: NormalizationSpec | None = None, workers: int = 1, *,
                device=None) -> np.ndarray:
    """Synchronous matrix by direct summation (hilbert.py:71-89)."""
    if workers < 1:
        raise DataError(f"workers must be >= 1, got {workers}")
    plan, *_ = _plan(dyn1, dyn2, norm, None, device)
    plan.launch()
    engine.sync()
    plan.check()
    s, _ = plan.fetch()
    return s


def hilbert_transform(dyn, *, device=None) -> np.ndarray:
    """N @ values for every spectral channel (hilbert.py:63-68), m x n, computed
    by one K1 time-domain pack and one FP64 contraction against the rows of N."""
    if dyn.m < 2:
        raise DataError(f"need m >= 2, got {dyn.m}")
    t = engine.torch()
    lib, dev = engine.require_device(device)
    m, n = dyn.m, dyn.n
    mp = lib.corr2d_packed_depth(m, _abi.PACK_F64_TIME)
    y = t.empty((n, mp), dtype=t.float64, device=dev)
    status = t.zeros(4, dtype=t.int32, device=dev)
    recipe = engine.PrepRecipe(m_in=m, m=m, ref_mode=_abi.REF_NONE)
    engine.launch_prep(lib, dyn.device_values(dev), recipe, norm=1.0, pack_kind=_abi.PACK_F64_TIME,
                       roles=_abi.ROLE_A, a_phi=y, ld_pack=mp, status=status)
    rows_n = t.from_numpy(-engine._noda_rows(m, mp)).to(dev)      # +N, zero padded
    z = t.empty((n, mp), dtype=t.float64, device=dev)
    scratch = t.empty((n, mp), dtype=t.float64, device=dev)
    stats = t.zeros(4, dtype=t.int64, device=dev)
    code = lib.corr2d_contract_f64(engine.ptr(y), engine.ptr(y), engine.ptr(rows_n), mp, n, m, mp, 0, 0, n,
                                   0, -1, engine.ptr(z), engine.ptr(scratch), mp, engine.ptr(stats),
                                   engine.stream_handle())
    _abi.check(code, lib)
    engine.sync()
    return np.ascontiguousarray(z[:, :m].cpu().numpy().T)
