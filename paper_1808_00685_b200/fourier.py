"""Fourier-route correlation engine drop-in (reference: fourier.py:40-125).

    C(nu1, nu2) = Norm * sum_w weight(w) Y1(nu1, w) conj(Y2(nu2, w)),
    sync = Re C,  async = Im C,  Norm default 1/(pi (m - 1)),

with Y the real DFT of each spectral channel along the perturbation axis
(frequencies 0..floor(m/2)) and weight 1 at DC / Nyquist, 2 elsewhere.

GPU execution: K1 (``corr2d_prep``) computes the DFT of every channel in
shared memory and packs the half spectrum into an exact real contraction of
depth m (weights and Norm folded into the row operand); K2
(``corr2d_contract_f64`` on the FP64 tensor pipe, or
``corr2d_contract_tc`` on tcgen05 for ``dtype="float32"``) writes the
sync / async planes directly -- no complex intermediate, no concatenate, no
Re/Im split copies, no O(n^2) host validation.  ``workers`` keeps its
reference meaning of host threads; results are identical for every value.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi, engine
from .dataset import CorrelationSpectra
from .engine_core import NormalizationSpec, check_pair, is_same_dynamic
from .errors import DataError, NumericError


@dataclass(eq=False)
class FourierWorkspace:
    """Retained half spectra of both inputs plus the per-frequency weights."""

    half_spectrum1: np.ndarray
    half_spectrum2: np.ndarray
    weights: np.ndarray
    m: int


def half_spectrum_weights(m: int) -> np.ndarray:
    """1 at frequency 0 (and at Nyquist for even m), 2 elsewhere (fourier.py:50-58)."""
    if m < 2:
        raise DataError(f"need m >= 2, got {m}")
    k = m // 2 + 1
    w = np.full(k, 2.0)
    w[0] = 1.0
    if m % 2 == 0:
        w[k - 1] = 1.0
    return w


def _half_spectrum(dyn, dev) -> np.ndarray:
    t = engine.torch()
    lib = _abi.load()
    m, n = dyn.m, dyn.n
    k = m // 2 + 1
    half = t.empty((k, n), dtype=t.complex128, device=dev)
    status = t.zeros(4, dtype=t.int32, device=dev)
    recipe = engine.PrepRecipe(m_in=m, m=m, ref_mode=_abi.REF_NONE)
    engine.launch_prep(lib, dyn.device_values(dev), recipe,
                       half_out=t.view_as_real(half), status=status)
    if engine.decode_status(status.cpu().numpy())[0]:
        raise NumericError("dynamic-spectra matrix contains non-finite values")
    return half.cpu().numpy()


def dft_channels(dyn, dyn2=None, workers: int = 1) -> FourierWorkspace:
    """Real DFT of every spectral channel, frequencies 0..floor(m/2)
    (fourier.py:61-82), computed by the K1 shared-memory Stockham FFT."""
    _, dev = engine.require_device()
    half1 = _half_spectrum(dyn, dev)
    if dyn2 is None or dyn2 is dyn:
        half2 = half1
    else:
        half2 = _half_spectrum(dyn2, dev)  # finiteness first, as the reference
        if dyn2.m != dyn.m:
            raise DataError(f"perturbation counts differ ({dyn.m} vs {dyn2.m})")
    return FourierWorkspace(half1, half2, half_spectrum_weights(dyn.m), dyn.m)


class DeviceCorrelationSpectra:
    """``correlate_ft(..., return_device=True)``: planes stay in HBM as CUDA
    tensors (rows [row0, row1) for a sharded call); ``to_host()`` copies."""

    def __init__(self, plan, meta):
        self.sync = plan.phi
        self.asyn = plan.psi
        self.rows = (plan.row0, plan.row1)
        self.meta = meta
        self._plan = plan

    def to_host(self, out=None) -> CorrelationSpectra:
        s, a = self._plan.fetch(out)
        return CorrelationSpectra._trusted(sync=s, asyn=a, **self.meta)


@engine.on_device
def correlate_ft(dyn1, dyn2=None, norm: NormalizationSpec | None = None, workers: int = 1, *,
                 dtype="float64", out=None, return_device: bool = False, device=None, rows=None,
                 distributed: bool = False, group=None, spectra: str = "broadcast"):
    """Synchronous and asynchronous correlation via the Fourier route
    (fourier.py:85-125).  Extras (keyword-only): ``dtype="float32"`` selects
    the tensor-core path (fp16 + e4m3 split products) with float32 planes;
    ``out=(sync, asyn)`` host buffers to fill; ``return_device`` keeps the
    planes in HBM; ``rows=(row0, row1)`` computes one row shard;
    ``distributed=True`` (one process per GPU under torch.distributed) returns
    this rank's band of the map (:class:`~.sharded.ShardedCorrelationSpectra`,
    see ``corr2d``)."""
    homo = dyn2 is None or is_same_dynamic(dyn1, dyn2)
    if dyn2 is None:
        dyn2 = dyn1
    check_pair(dyn1, dyn2)
    if workers < 1:
        raise DataError(f"workers must be >= 1, got {workers}")
    norm = norm or NormalizationSpec.noda()
    constant = norm.constant(dyn1.m)
    _, dev = engine.require_device(device)
    m = dyn1.m
    recipe = engine.PrepRecipe(m_in=m, m=m, ref_mode=_abi.REF_NONE)

    def make_plan(rws):
        pl = engine.CorrelationPlan(n1=dyn1.n, n2=dyn2.n, m=m, recipe1=recipe,
                                    recipe2=None if homo else recipe, norm=constant, dtype=dtype,
                                    rows=rws, device=dev, want_ref=False)
        return pl.bind(dyn1.device_values(dev), None if homo else dyn2.device_values(dev))

    meta = dict(axis1=dyn1.spectral_axis, axis2=dyn2.spectral_axis, ref1=dyn1.reference_used,
                ref2=dyn2.reference_used, normalization=constant, engine="fourier",
                is_homo=homo, scaling_exponent=dyn1.scaling_exponent)
    if distributed:
        # this rank's band of a multi-GPU map (sharded.py)
        from . import sharded
        plan = sharded.ShardedCorrelationPlan(n1=dyn1.n, n2=dyn2.n, m=m, recipe1=recipe,
                                              recipe2=None if homo else recipe, norm=constant, dtype=dtype,
                                              device=dev, group=group, spectra=spectra)
        plan.bind(dyn1.device_values(dev), None if homo else dyn2.device_values(dev))
        return sharded.run(plan, meta, axes=(dyn1.spectral_axis, dyn2.spectral_axis))
    if not return_device and rows is None:
        odt = np.dtype(dtype)
        blocks = engine.maybe_stream_blocks(dyn1.n, dyn2.n, odt.itemsize, dev)
        plan = None
        if blocks is None:
            try:
                plan = make_plan(rows)
            except NumericError as e:          # the device is fuller than the size check assumed
                if "out of memory" not in str(e):
                    raise
                blocks = engine.stream_blocks(dyn1.n, dyn2.n, odt.itemsize, engine.device_budget(dev))
        if blocks is not None:        # planes larger than device memory: stream row blocks
            s, a, info, _ = engine.run_streamed(make_plan, dyn1.n, dyn2.n, odt, blocks, out)
            return CorrelationSpectra._trusted(sync=s, asyn=a, stats=info, **meta)
    else:
        plan = None
    plan = plan or make_plan(rows)
    if not return_device and rows is None:
        # planes' D2H queued right behind the kernels; status checks overlap it
        s, a, (*_, info) = plan.run_to_host(out)
        meta["stats"] = info
        return CorrelationSpectra._trusted(sync=s, asyn=a, **meta)
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
