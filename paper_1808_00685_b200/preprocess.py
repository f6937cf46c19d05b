"""Preprocessing drop-in (reference: preprocess.py:24-275), executed on the GPU.

Fixed pipeline order, as the reference: resample (optional) -> subtract the
reference spectrum -> divide each channel by sigma**alpha (optional), sigma
taken from the resampled data about the chosen reference.  All per-element
work runs in the fused K1 kernel (``corr2d_prep``); only O(m * m_in)
resampling coefficients and O(n) vectors are prepared or returned on the host.
``DynamicSpectra.values`` stays in HBM until first accessed from Python.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _abi, engine
from .dataset import SpectralDataset
from .errors import DataError, NumericError


class InterpolantKind(enum.Enum):
    LINEAR = "linear"
    CUBIC_SPLINE = "spline"

    @classmethod
    def from_name(cls, name: str) -> "InterpolantKind":
        for kind in cls:
            if kind.value == name:
                return kind
        raise DataError(f"unknown interpolant {name!r} (use 'linear' or 'spline')")


@dataclass(frozen=True)
class ReferenceSpec:
    """Reference spectrum: the perturbation mean, or a provided vector (preprocess.py:36-64)."""

    kind: str
    spectrum: np.ndarray | None = None

    @classmethod
    def mean(cls) -> "ReferenceSpec":
        return cls("mean")

    @classmethod
    def provided(cls, spectrum) -> "ReferenceSpec":
        vec = np.asarray(spectrum, dtype=np.float64)
        if vec.ndim != 1:
            raise DataError("provided reference must be a 1D vector")
        if not np.isfinite(vec).all():
            raise DataError("provided reference contains non-finite values")
        return cls("provided", vec)

    def check_length(self, n: int) -> None:
        if self.kind == "provided" and self.spectrum.size != n:
            raise DataError(f"reference length {self.spectrum.size} does not match n = {n}")

    def resolve(self, ds: SpectralDataset) -> np.ndarray:
        if self.kind == "mean":
            return mean_reference(ds)
        self.check_length(ds.n)
        return self.spectrum


@dataclass(frozen=True)
class ResampleSpec:
    target_count: int
    interpolant: InterpolantKind = InterpolantKind.CUBIC_SPLINE

    def __post_init__(self):
        if self.target_count < 4:
            raise DataError(f"resample target_count must be >= 4, got {self.target_count}")


@dataclass(frozen=True)
class PreprocessSpec:
    reference: ReferenceSpec = ReferenceSpec.mean()
    resample: ResampleSpec | None = None
    scaling_exponent: float = 0.0

    def __post_init__(self):
        if not 0.0 <= self.scaling_exponent <= 1.0:
            raise DataError(f"scaling exponent must lie in [0, 1], got {self.scaling_exponent}")


@dataclass(eq=False)
class DynamicSpectra:
    """Reference-subtracted (optionally scaled) m x n matrix with provenance
    (preprocess.py:90-120): the same dataclass fields, so ``dataclasses.fields``
    / ``replace`` / ``asdict`` work as on the reference type.

    ``values`` is a plain field from the caller's point of view.  When K1
    produced it (``preprocess_dataset``), it stays in HBM until Python first
    reads it; from then on -- and whenever it was set from a host array -- the
    HOST array is authoritative and every device use uploads it again, so an
    in-place edit of ``dyn.values`` (or of the caller's float64 array, which
    ``np.asarray`` aliases exactly as the reference does) is always honoured,
    as the reference re-reads ``dyn.values`` on every call."""

    spectral_axis: np.ndarray
    perturbation_axis: np.ndarray
    values: np.ndarray
    reference_used: np.ndarray
    scaling_exponent: float = 0.0
    sigma: np.ndarray | None = None

    def __post_init__(self):
        self.spectral_axis = np.asarray(self.spectral_axis, dtype=np.float64)
        self.perturbation_axis = np.asarray(self.perturbation_axis, dtype=np.float64)
        self.reference_used = np.asarray(self.reference_used, dtype=np.float64)
        shape = tuple(self._dev.shape) if self._host is None else self._host.shape
        m, n = self.perturbation_axis.size, self.spectral_axis.size
        if shape != (m, n):
            raise DataError(f"dynamic matrix shape {shape} does not match axes ({m}, {n})")
        if self.reference_used.shape != (n,):
            raise DataError("reference_used length does not match the spectral axis")

    def _get_values(self) -> np.ndarray:
        if self._host is None:
            # first host read: from now on the host array is the source of truth
            self._host = self._dev.double().cpu().numpy()
            self._dev = None
        return self._host

    def _set_values(self, v):
        if _is_tensor(v):
            self._dev, self._host = v, None
        else:
            self._host, self._dev = np.asarray(v, dtype=np.float64), None

    def device_values(self, dev):
        """The values as a contiguous CUDA tensor on `dev`: the K1 output itself
        while Python never saw the values, else a fresh upload of the host
        array (no cache that could go stale)."""
        t = engine.torch()
        if self._host is not None:
            return engine.to_device(self._host, dev)
        d = self._dev
        if d.device != dev:
            d = d.to(dev)
        if d.dtype not in (t.float64, t.float32):
            d = d.double()
        return d.contiguous()

    def device_identity(self):
        """The device tensor while it is authoritative (else None): lets the
        homo test compare two K1 outputs on the device."""
        return self._dev if self._host is None else None

    @property
    def m(self) -> int:
        return int(self.perturbation_axis.size)

    @property
    def n(self) -> int:
        return int(self.spectral_axis.size)


# `values` is a dataclass field (in __init__, fields(), replace(), asdict())
# backed by the lazy host/device storage above.
DynamicSpectra._host = None
DynamicSpectra._dev = None
DynamicSpectra.values = property(DynamicSpectra._get_values, DynamicSpectra._set_values)


def _is_tensor(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch")


# --------------------------------------------------------------------------
# device helpers
# --------------------------------------------------------------------------

def _raw_device(ds: SpectralDataset, dev):
    """Upload the intensities for this call (pinned host arrays copy at full
    PCIe rate).  No hidden cache: every call moves its inputs."""
    return engine.to_device(ds.intensities, dev)


def _run_prep(ds_values_dev, recipe: engine.PrepRecipe, *, want_values=True, want_ref=False,
              want_sigma=False, dev=None):
    """Launch K1 on the current stream and synchronise; returns device outputs
    and the host status word."""
    t = engine.torch()
    lib = engine._abi.load()
    n = ds_values_dev.shape[1]
    out = {}
    if want_values:
        out["values"] = t.empty((recipe.m, n), dtype=t.float64, device=dev)
    if want_ref:
        out["ref"] = t.empty(n, dtype=t.float64, device=dev)
    if want_sigma:
        out["sigma"] = t.empty(n, dtype=t.float64, device=dev)
    status = t.zeros(4, dtype=t.int32, device=dev)
    engine.launch_prep(lib, ds_values_dev, recipe, values_out=out.get("values"),
                       ref_out=out.get("ref"), sigma_out=out.get("sigma"), status=status)
    out["status"] = status.cpu().numpy()
    return out


def _recipe_for(ds: SpectralDataset, spec: PreprocessSpec, on_zero_variance: str, dev):
    plan = None
    m = ds.m
    if spec.resample is not None:
        plan = engine.resample_plan(ds.perturbation_axis, spec.resample.target_count,
                                    spec.resample.interpolant.value)
        m = spec.resample.target_count
    ref_mode, ref_in = _abi.REF_MEAN, None
    if spec.reference.kind == "provided":
        spec.reference.check_length(ds.n)
        ref_mode, ref_in = _abi.REF_PROVIDED, engine.to_device(spec.reference.spectrum, dev)
    return engine.PrepRecipe(m_in=ds.m, m=m, ref_mode=ref_mode, resample=plan, ref_in=ref_in,
                             alpha=float(spec.scaling_exponent),
                             substitute=(on_zero_variance == "substitute")), plan


def _zero_variance(spectral_axis, sigma_raw, alpha, policy):
    dead = sigma_raw == 0.0
    if dead.any() and policy not in ("error", "substitute"):
        raise DataError(f"unknown zero-variance policy {policy!r}")
    return engine.handle_zero_variance(spectral_axis, sigma_raw, alpha, policy == "substitute")


# --------------------------------------------------------------------------
# public functions (same names / semantics as the reference)
# --------------------------------------------------------------------------

def mean_reference(ds: SpectralDataset) -> np.ndarray:
    """Columnwise perturbation mean (preprocess.py:123-125), on the device."""
    _, dev = engine.require_device()
    recipe = engine.PrepRecipe(m_in=ds.m, m=ds.m)
    out = _run_prep(_raw_device(ds, dev), recipe, want_values=False, want_ref=True, dev=dev)
    return out["ref"].cpu().numpy()


def dynamic_spectra(ds: SpectralDataset, ref: ReferenceSpec | None = None) -> DynamicSpectra:
    """Subtract the reference from every spectrum (preprocess.py:128-137)."""
    return preprocess_dataset(ds, PreprocessSpec(reference=ref or ReferenceSpec.mean()))


def default_target_count(m: int) -> int:
    """Smallest power of two >= max(m, 4) (preprocess.py:140-144)."""
    if m < 2:
        raise DataError(f"m must be >= 2, got {m}")
    target = 4
    while target < m:
        target *= 2
    return target


def resample_to_axis(ds: SpectralDataset, new_axis,
                     kind: InterpolantKind = InterpolantKind.CUBIC_SPLINE) -> SpectralDataset:
    """Interpolate every channel onto `new_axis` within [t0, t_end] (preprocess.py:155-178)."""
    if not isinstance(kind, InterpolantKind):
        raise DataError(f"unknown interpolant {kind!r}")
    _, dev = engine.require_device()
    new_axis = np.asarray(new_axis, dtype=np.float64)
    plan = engine.axis_plan(ds.perturbation_axis, new_axis, kind.value)
    recipe = engine.PrepRecipe(m_in=ds.m, m=new_axis.size, ref_mode=_abi.REF_NONE, resample=plan)
    out = _run_prep(_raw_device(ds, dev), recipe, want_values=True, dev=dev)
    return SpectralDataset(ds.spectral_axis, new_axis, out["values"].cpu().numpy(), ds.axis_labels)


def resample_equidistant(ds: SpectralDataset, target_count: int,
                         kind: InterpolantKind = InterpolantKind.CUBIC_SPLINE) -> SpectralDataset:
    """Equidistant resampling over [t0, t_end] inclusive (preprocess.py:181-195)."""
    if target_count < 4:
        raise DataError(f"target_count must be >= 4, got {target_count}")
    t = ds.perturbation_axis
    return resample_to_axis(ds, np.linspace(t[0], t[-1], target_count), kind)


def stddev_spectrum(ds: SpectralDataset, ref: ReferenceSpec | None = None) -> np.ndarray:
    """Per-channel standard deviation about the reference, denominator m - 1
    (preprocess.py:198-211)."""
    if ds.m < 2:
        raise DataError(f"standard deviation needs m >= 2, got {ds.m}")
    _, dev = engine.require_device()
    spec = PreprocessSpec(reference=ref or ReferenceSpec.mean(), scaling_exponent=1.0)
    recipe, _ = _recipe_for(ds, spec, "substitute", dev)
    out = _run_prep(_raw_device(ds, dev), recipe, want_values=False, want_sigma=True, dev=dev)
    return out["sigma"].cpu().numpy()


def apply_scaling(dyn: DynamicSpectra, sigma, alpha: float,
                  on_zero_variance: str = "error") -> DynamicSpectra:
    """Divide each channel by sigma**alpha (preprocess.py:214-259)."""
    if not 0.0 <= alpha <= 1.0:
        raise DataError(f"scaling exponent must lie in [0, 1], got {alpha}")
    if dyn.scaling_exponent != 0.0:
        raise DataError("dynamic spectra are already scaled")
    sigma = np.asarray(sigma, dtype=np.float64)
    if sigma.shape != (dyn.n,):
        raise DataError(f"sigma length {sigma.size} does not match n = {dyn.n}")
    if alpha == 0.0:
        src = dyn.device_identity()
        return DynamicSpectra(dyn.spectral_axis, dyn.perturbation_axis, dyn.values if src is None else src,
                              dyn.reference_used, 0.0, sigma)
    _, dev = engine.require_device()
    sig = _zero_variance(dyn.spectral_axis, sigma, alpha, on_zero_variance)
    recipe = engine.PrepRecipe(m_in=dyn.m, m=dyn.m, ref_mode=_abi.REF_NONE, alpha=float(alpha),
                               sigma_in=engine.to_device(sig, dev), substitute=True)
    out = _run_prep(dyn.device_values(dev), recipe, want_values=True, dev=dev)
    return DynamicSpectra(dyn.spectral_axis, dyn.perturbation_axis, out["values"],
                          dyn.reference_used, alpha, sig)


def preprocess_dataset(ds: SpectralDataset, spec: PreprocessSpec | None = None,
                       on_zero_variance: str = "error") -> DynamicSpectra:
    """Resample -> subtract reference -> scale, one fused device pass
    (preprocess.py:262-275).  ``values`` stays on the device until accessed."""
    spec = spec or PreprocessSpec()
    _, dev = engine.require_device()
    recipe, plan = _recipe_for(ds, spec, on_zero_variance, dev)
    alpha = float(spec.scaling_exponent)
    out = _run_prep(_raw_device(ds, dev), recipe, want_values=True, want_ref=True,
                    want_sigma=alpha > 0.0, dev=dev)
    t_axis = plan.t_new if plan is not None else ds.perturbation_axis
    if engine.decode_status(out["status"])[0]:
        raise DataError("intensity matrix contains non-finite values")
    sigma = None
    if alpha > 0.0:
        sigma = _zero_variance(ds.spectral_axis, out["sigma"].cpu().numpy(), alpha, on_zero_variance)
    return DynamicSpectra(ds.spectral_axis, t_axis, out["values"], out["ref"].cpu().numpy(),
                          alpha if alpha > 0.0 else 0.0, sigma)
