"""Input and result containers of the drop-in (reference: dataset.py:50-170).

``SpectralDataset`` and ``CorrelationSpectra`` keep the reference's fields,
invariants and error messages.  Differences, all opt-in:

* ``SpectralDataset(..., dtype=np.float32)`` keeps single-precision storage for
  the fp32 tensor-core path (F16F8 by default, bf16x3 optional); the default is
  float64 like the reference.
* ``CorrelationSpectra`` built by the GPU engine skips the O(n^2) host
  re-validation (dataset.py:141-170): symmetry/skew-symmetry hold by
  construction (mirrored tiles) and finiteness was checked on the device in the
  contraction epilogue.  Constructing one by hand validates exactly like the
  reference.  fp32 results keep float32 planes; ``to_reference()`` converts to
  a real ``corrtwo.CorrelationSpectra`` when the reference is importable.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DataError

LABEL_SEP = " \\ "


def _check_monotonic(values: np.ndarray, name: str) -> None:
    """Strictly monotonic in either direction (dataset.py:39-47 semantics)."""
    d = np.diff(values)
    if d.size == 0 or np.all(d > 0) or np.all(d < 0):
        return
    zero = np.flatnonzero(d == 0)
    if zero.size:
        # position of the smallest |step| (1-based, counting the second element)
        raise DataError(f"{name} contains duplicate values (position {int(np.argmin(np.abs(d))) + 2})")
    flips = np.flatnonzero(np.sign(d) != np.sign(d[0]))
    raise DataError(f"{name} is not strictly monotonic (position {int(flips[0]) + 2})")


@dataclass(eq=False)
class SpectralDataset:
    """Perturbation-ordered series of 1D spectra; row j of `intensities` is the
    spectrum at perturbation_axis[j] (dataset.py:50-108)."""

    spectral_axis: np.ndarray
    perturbation_axis: np.ndarray
    intensities: np.ndarray
    axis_labels: tuple = ("nu", "t")
    dtype: object = None

    def __post_init__(self):
        self.spectral_axis = np.asarray(self.spectral_axis, dtype=np.float64)
        self.perturbation_axis = np.asarray(self.perturbation_axis, dtype=np.float64)
        store = np.float32 if np.dtype(self.dtype or np.float64) == np.float32 else np.float64
        self.intensities = np.ascontiguousarray(np.asarray(self.intensities, dtype=store))
        self.dtype = np.dtype(store)
        self.validate()

    @property
    def m(self) -> int:
        return int(self.perturbation_axis.size)

    @property
    def n(self) -> int:
        return int(self.spectral_axis.size)

    def validate(self) -> None:
        m, n = self.m, self.n
        if m < 2:
            raise DataError(f"m < 2: need at least two spectra, got {m}")
        if n < 2:
            raise DataError(f"n < 2: need at least two spectral values, got {n}")
        if self.intensities.shape != (m, n):
            raise DataError(f"intensity matrix shape {self.intensities.shape} does not match axes ({m}, {n})")
        for arr, label in ((self.spectral_axis, "spectral axis"), (self.perturbation_axis, "perturbation axis")):
            if not np.isfinite(arr).all():
                raise DataError(f"{label} contains non-finite values")
        finite = np.isfinite(self.intensities)
        if not finite.all():
            j, i = np.argwhere(~finite)[0]
            raise DataError(f"non-finite intensity at row {j + 1}, column {i + 1}")
        _check_monotonic(self.spectral_axis, "spectral axis")
        steps = np.diff(self.perturbation_axis)
        bad = np.flatnonzero(steps <= 0)
        if bad.size:
            raise DataError(f"perturbation axis must be strictly increasing (position {int(bad[0]) + 2})")

    def equals(self, other: "SpectralDataset") -> bool:
        return (np.array_equal(self.spectral_axis, other.spectral_axis)
                and np.array_equal(self.perturbation_axis, other.perturbation_axis)
                and np.array_equal(self.intensities, other.intensities)
                and tuple(self.axis_labels) == tuple(other.axis_labels))


@dataclass(eq=False)
class CorrelationSpectra:
    """Synchronous (sync = Phi) and asynchronous (asyn = Psi) correlation planes
    with provenance (dataset.py:111-170): the reference's dataclass fields, so
    ``dataclasses.fields`` / ``replace`` / ``asdict`` behave as on the reference
    type (``replace`` re-validates, as there).  ``stats`` (device-side max|.|)
    is a plain attribute, not a field."""

    axis1: np.ndarray
    axis2: np.ndarray
    sync: np.ndarray
    asyn: np.ndarray
    ref1: np.ndarray
    ref2: np.ndarray
    normalization: float
    engine: str
    is_homo: bool
    scaling_exponent: float = 0.0

    SYMMETRY_TOL = 1e-12
    stats = None

    def __post_init__(self):
        for name in ("axis1", "axis2", "sync", "asyn", "ref1", "ref2"):
            setattr(self, name, np.asarray(getattr(self, name), dtype=np.float64))
        self.is_homo = bool(self.is_homo)
        self.validate()

    @classmethod
    def _trusted(cls, axis1, axis2, sync, asyn, ref1, ref2, normalization, engine,
                 is_homo, scaling_exponent, stats=None):
        """Engine-side constructor: invariants were established on the device."""
        obj = cls.__new__(cls)
        obj.axis1, obj.axis2 = axis1, axis2
        obj.sync, obj.asyn = sync, asyn
        obj.ref1, obj.ref2 = ref1, ref2
        obj.normalization, obj.engine = normalization, engine
        obj.is_homo, obj.scaling_exponent = bool(is_homo), scaling_exponent
        obj.stats = stats
        obj._validate_shapes()
        return obj

    @property
    def n1(self) -> int:
        return int(self.axis1.size)

    @property
    def n2(self) -> int:
        return int(self.axis2.size)

    def _validate_shapes(self) -> None:
        if self.engine not in ("fourier", "hilbert"):
            raise DataError(f"unknown engine tag {self.engine!r}")
        shape = (self.n1, self.n2)
        if tuple(self.sync.shape) != shape:
            raise DataError(f"sync shape {tuple(self.sync.shape)} does not match axes {shape}")
        if tuple(self.asyn.shape) != tuple(self.sync.shape):
            raise DataError(f"dimension mismatch: sync {tuple(self.sync.shape)} vs async {tuple(self.asyn.shape)}")
        if self.ref1.shape != (self.n1,) or self.ref2.shape != (self.n2,):
            raise DataError("reference spectra lengths do not match the axes")
        if not self.normalization > 0:
            raise DataError("normalization constant must be positive")

    def validate(self) -> None:
        """Full host validation, reference semantics (dataset.py:141-170)."""
        self._validate_shapes()
        if not np.isfinite(self.sync).all():
            raise DataError("sync matrix contains non-finite values")
        if not np.isfinite(self.asyn).all():
            raise DataError("asyn matrix contains non-finite values")
        if self.is_homo:
            if not np.array_equal(self.axis1, self.axis2):
                raise DataError("homo result requires identical axes")
            scale = max(float(np.abs(self.sync).max()), float(np.abs(self.asyn).max()))
            tol = self.SYMMETRY_TOL * scale
            if float(np.abs(self.sync - self.sync.T).max()) > tol:
                raise DataError("homo sync matrix is not symmetric")
            if float(np.abs(self.asyn + self.asyn.T).max()) > tol:
                raise DataError("homo async matrix is not skew-symmetric")

    def to_reference(self):
        """A genuine ``corrtwo.CorrelationSpectra`` (tests / interop only)."""
        import corrtwo  # noqa: F401  (only when the reference is installed)
        return corrtwo.CorrelationSpectra(
            axis1=self.axis1, axis2=self.axis2, sync=np.asarray(self.sync, dtype=np.float64),
            asyn=np.asarray(self.asyn, dtype=np.float64), ref1=self.ref1, ref2=self.ref2,
            normalization=self.normalization, engine=self.engine, is_homo=self.is_homo,
            scaling_exponent=self.scaling_exponent)

    def __repr__(self) -> str:
        return (f"CorrelationSpectra(n1={self.n1}, n2={self.n2}, dtype={self.sync.dtype}, "
                f"engine={self.engine!r}, is_homo={self.is_homo}, normalization={self.normalization!r})")
