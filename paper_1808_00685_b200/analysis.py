"""Peak extraction and Noda-rule classification drop-in (reference:
analysis.py:1-201).

The O(n1 n2) part -- strict 8-neighbourhood local maxima of |sync| and |async|
above ``threshold_fraction`` of their maxima -- runs on the GPU as one scan of
the planes (K3, ``corr2d_find_peaks``; the maxima come from K2's fused
statistics for device results, else from ``corr2d_plane_absmax``).  Only the
candidate indices come back to the host, where the O(peaks) work follows the
reference: row-major order, homo upper triangle, the five sign rules with dead
band ``eps``, auto peaks on the homo diagonal.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _abi, engine
from .errors import DataError


class Verdict(enum.Enum):
    SAME_DIRECTION = "same-direction"
    OPPOSITE_DIRECTION = "opposite-direction"
    NU1_BEFORE = "nu1-before"
    NU1_AFTER = "nu1-after"
    INDETERMINATE = "indeterminate"


@dataclass(frozen=True)
class CrossPeakVerdict:
    direction: Verdict
    order: Verdict

    def __str__(self):
        return f"{self.direction.value}, {self.order.value}"


def classify_cross_peak(phi: float, psi: float, eps: float) -> CrossPeakVerdict:
    """The five sign rules (analysis.py:51-66): sign(sync) gives the direction,
    sign(async) the order, reversed when sync is negative; |.| <= eps is
    indeterminate."""
    if not eps > 0:
        raise DataError(f"eps must be positive, got {eps}")
    neg = phi < -eps
    direction = (Verdict.SAME_DIRECTION if phi > eps
                 else Verdict.OPPOSITE_DIRECTION if neg else Verdict.INDETERMINATE)
    if abs(psi) <= eps:
        return CrossPeakVerdict(direction, Verdict.INDETERMINATE)
    before = (psi > 0) != neg
    return CrossPeakVerdict(direction, Verdict.NU1_BEFORE if before else Verdict.NU1_AFTER)


@dataclass(frozen=True)
class AutoPeak:
    nu: float
    phi: float


@dataclass(frozen=True)
class CrossPeak:
    nu1: float
    nu2: float
    phi: float
    psi: float
    verdict: CrossPeakVerdict


def _num(x) -> str:
    return repr(float(x))   # shortest round-trip decimal (dataset.py:34-36)


@dataclass
class PeakReport:
    auto_peaks: list = field(default_factory=list)
    cross_peaks: list = field(default_factory=list)
    threshold_fraction: float = 0.1
    eps: float = 0.0
    is_homo: bool = True

    def to_table(self) -> str:
        out = []
        if self.is_homo:
            out.append("auto peaks (nu, sync):")
            out += [f"  {p.nu:g}  {p.phi:.6g}" for p in self.auto_peaks] or ["  none"]
        out.append("cross peaks (nu1, nu2, sync, async, verdict):")
        out += [f"  {p.nu1:g}  {p.nu2:g}  {p.phi:.6g}  {p.psi:.6g}  {p.verdict}"
                for p in self.cross_peaks] or ["  none"]
        return "\n".join(out) + "\n"

    def to_long_form(self) -> bytes:
        rows = ["kind,nu1,nu2,sync,async,direction,order"]
        rows += [f"auto,{_num(p.nu)},{_num(p.nu)},{_num(p.phi)},0.0,," for p in self.auto_peaks]
        rows += [f"cross,{_num(p.nu1)},{_num(p.nu2)},{_num(p.phi)},{_num(p.psi)},"
                 f"{p.verdict.direction.value},{p.verdict.order.value}" for p in self.cross_peaks]
        return ("\n".join(rows) + "\n").encode("utf-8")


def _planes(corr):
    """(sync, asyn, host_sync, host_asyn, maxima or None, axes, is_homo) on the device."""
    t = engine.torch()
    lib, dev = engine.require_device(None)
    if hasattr(corr, "_plan"):                        # DeviceCorrelationSpectra
        if tuple(corr.rows) != (0, len(corr.meta["axis1"])):
            raise DataError("find_peaks needs the whole map (not a row shard)")
        st = corr.meta.get("stats") or {}
        maxima = (st.get("max_abs_sync"), st.get("max_abs_async"))
        if None in maxima:
            maxima = None
        return (corr.sync, corr.asyn, None, None, maxima,
                (corr.meta["axis1"], corr.meta["axis2"]), bool(corr.meta["is_homo"]))
    sync = np.ascontiguousarray(corr.sync)
    asyn = np.ascontiguousarray(corr.asyn)
    if sync.dtype not in (np.float64, np.float32):
        sync, asyn = sync.astype(np.float64), asyn.astype(np.float64)
    return (t.from_numpy(sync).to(dev), t.from_numpy(asyn).to(dev), sync, asyn, None,
            (corr.axis1, corr.axis2), bool(corr.is_homo))


def find_peaks(corr, threshold_fraction: float = 0.1, eps: float | None = None) -> PeakReport:
    """Auto peaks (homo diagonal) and cross peaks above a threshold
    (analysis.py:152-201) for a ``CorrelationSpectra`` or a device result."""
    if not 0.0 < threshold_fraction < 1.0:
        raise DataError(f"threshold_fraction must lie in (0, 1), got {threshold_fraction}")
    t = engine.torch()
    lib, dev = engine.require_device(None)
    sync_d, asyn_d, sync_h, asyn_h, maxima, (axis1, axis2), homo = _planes(corr)
    n1, n2 = int(sync_d.shape[0]), int(sync_d.shape[1])
    dt = np.float32 if sync_d.dtype == t.float32 else np.float64
    code = _abi.F32 if dt == np.float32 else _abi.F64
    if maxima is None:
        buf = t.zeros(2, dtype=t.float64, device=dev)
        for j, plane in enumerate((sync_d, asyn_d)):
            _abi.check(lib.corr2d_plane_absmax(code, engine.ptr(plane), plane.stride(0), n1, n2,
                                               engine.ptr(buf[j:]), engine.stream_handle()), lib)
        maxima = tuple(buf.cpu().numpy())
    ms, ma = dt(maxima[0]), dt(maxima[1])            # exact: maxima of dt values
    scale = max(ms, ma)
    if eps is None:
        eps = 1e-3 * scale
    report = PeakReport(threshold_fraction=threshold_fraction, eps=eps, is_homo=homo)
    if scale == 0.0:
        return report

    if homo:
        diag = (np.diag(sync_h) if sync_h is not None else sync_d.diagonal().cpu().numpy())
        pad = np.concatenate(([-np.inf], diag, [-np.inf]))
        keep = (diag > pad[:-2]) & (diag > pad[2:]) & (diag > threshold_fraction * diag.max())
        report.auto_peaks = [AutoPeak(axis1[i], diag[i]) for i in np.flatnonzero(keep)]

    # thresholds in the planes' dtype, as numpy evaluates them (analysis.py:187-194)
    thr_s = float(threshold_fraction * ms) if ms > 0 else float("inf")
    thr_a = float(threshold_fraction * ma) if ma > 0 else float("inf")
    count = t.zeros(1, dtype=t.int64, device=dev)
    cap = 1 << 16
    while True:
        idx = t.empty(cap, dtype=t.int64, device=dev)
        _abi.check(lib.corr2d_find_peaks(code, engine.ptr(sync_d), engine.ptr(asyn_d), sync_d.stride(0), n1, n2,
                                         1 if homo else 0, thr_s, thr_a, engine.ptr(idx), cap,
                                         engine.ptr(count), engine.stream_handle()), lib)
        total = int(count.cpu().item())
        if total <= cap:
            break
        cap = total
    lin = t.sort(idx[:total]).values                 # np.argwhere's row-major order
    if sync_h is not None:
        li = lin.cpu().numpy()
        phis, psis = sync_h.reshape(-1)[li], asyn_h.reshape(-1)[li]
    else:
        ii, kk = lin // n2, lin % n2
        phis, psis = sync_d[ii, kk].cpu().numpy(), asyn_d[ii, kk].cpu().numpy()
        li = lin.cpu().numpy()
    for L, phi, psi in zip(li, phis, psis):
        i, k = divmod(int(L), n2)
        report.cross_peaks.append(CrossPeak(axis1[i], axis2[k], phi, psi, classify_cross_peak(phi, psi, eps)))
    return report
