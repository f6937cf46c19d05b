"""CPU oracle for the corr2D Fourier-route hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy/scipy restatement of the reference package
`corrtwo` 0.1.0 (the Python re-implementation of the R package corr2D,
arXiv 1808.00685) for exactly the path the B200 build accelerates:

    preprocess_dataset  (resample -> reference subtraction -> sigma**alpha scaling)
    dft_channels        (real FFT along the perturbation axis)
    correlate_ft        (weighted half-spectrum cross sum, x Norm, sync = Re, async = Im)

Every function cites the reference file:line it restates (paths relative to
`/root/reference/pkg/src/corrtwo/`).  The arithmetic of the reference lives in
third-party libraries that are *not* vendored under /root/reference:

    * numpy 2.3.5 (`np.matmul` complex128 -> scipy-openblas 0.3.30 ``zgemm``),
    * scipy 1.18.1 (``scipy.fft.rfft`` -> ducc0/pocketfft r2c;
      ``scipy.interpolate.CubicSpline`` with ``bc_type="natural"``).

The restatement calls the same numpy/scipy primitives (rfft, matmul), so on
the same inputs it reproduces the reference bit-for-bit; that is pinned by
`tests/test_oracle_golden.py` against fixtures produced by the reference itself
(`tests/golden/make_golden.py`, run in the build container where
/root/reference is importable).

Who may use this module: ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference``), as the
*checker / CPU baseline only*.  The product package
``paper_1808_00685_b200`` never imports it; its GPU path has no CPU fallback.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.fft

try:  # BLAS pinning like engine_core.map_row_blocks (engine_core.py:121)
    from threadpoolctl import threadpool_limits
except Exception:  # pragma: no cover - threadpoolctl is in the image
    threadpool_limits = None


# --------------------------------------------------------------------------
# weights / normalisation
# --------------------------------------------------------------------------

def half_spectrum_weights(m: int) -> np.ndarray:
    """fourier.py:50-58 -- weight 1 at DC (and Nyquist for even m), else 2."""
    if m < 2:
        raise ValueError(f"need m >= 2, got {m}")
    w = np.full(m // 2 + 1, 2.0)
    w[0] = 1.0
    if m % 2 == 0:
        w[-1] = 1.0
    return w


def noda_constant(m: int) -> float:
    """engine_core.py:62-66 -- default Fourier normalisation 1/(pi (m-1))."""
    return 1.0 / (math.pi * (m - 1))


def unit_constant(m: int) -> float:
    """engine_core.py:67-68 -- 1/(m-1)."""
    return 1.0 / (m - 1)


# --------------------------------------------------------------------------
# preprocessing (preprocess.py)
# --------------------------------------------------------------------------

def mean_reference(intensities: np.ndarray) -> np.ndarray:
    """preprocess.py:123-125 -- column mean over the perturbation axis."""
    return np.asarray(intensities, dtype=float).mean(axis=0)


def interp_linear(t_old, values, t_new):
    """preprocess.py:147-152 -- clipped searchsorted + v0 + frac (v1 - v0)."""
    t_old = np.asarray(t_old, dtype=float)
    t_new = np.asarray(t_new, dtype=float)
    idx = np.clip(np.searchsorted(t_old, t_new, side="right") - 1, 0, t_old.size - 2)
    t0, t1 = t_old[idx], t_old[idx + 1]
    frac = (t_new - t0) / (t1 - t0)
    return values[idx] + frac[:, None] * (values[idx + 1] - values[idx])


def natural_spline_matrix(t_old, t_new) -> np.ndarray:
    """Natural cubic spline as a linear map S (len(t_new) x len(t_old)).

    Restates preprocess.py:174-175 (``CubicSpline(t, y, bc_type="natural")``)
    through the textbook construction also used by the reference's own test
    oracle (tests/oracles.py:72-107): second derivatives M with M_0 = M_last = 0
    from the tridiagonal system, then the cubic on the containing interval.
    Because the spline is linear in the data, applying it to the identity gives
    the matrix; ``S @ y`` equals the spline of ``y`` evaluated at ``t_new``.
    """
    x = np.asarray(t_old, dtype=float)
    xq = np.asarray(t_new, dtype=float)
    n = x.size
    h = np.diff(x)
    eye = np.eye(n)
    second = np.zeros((n, n))  # second[:, k] = M for data e_k
    if n > 2:
        system = np.zeros((n - 2, n - 2))
        for i in range(1, n - 1):
            r = i - 1
            system[r, r] = 2.0 * (h[i - 1] + h[i])
            if r > 0:
                system[r, r - 1] = h[i - 1]
            if r < n - 3:
                system[r, r + 1] = h[i]
        rhs = 6.0 * ((eye[2:] - eye[1:-1]) / h[1:, None] - (eye[1:-1] - eye[:-2]) / h[:-1, None])
        second[1:-1] = np.linalg.solve(system, rhs)
    out = np.empty((xq.size, n))
    for q_i, q in enumerate(xq):
        i = int(np.clip(np.searchsorted(x, q, side="right") - 1, 0, n - 2))
        d = q - x[i]
        hi = h[i]
        a = eye[i]
        b = (eye[i + 1] - eye[i]) / hi - hi * (2.0 * second[i] + second[i + 1]) / 6.0
        c = second[i] / 2.0
        e = (second[i + 1] - second[i]) / (6.0 * hi)
        out[q_i] = a + b * d + c * d ** 2 + e * d ** 3
    return out


def resample_equidistant(t_old, intensities, target_count: int, kind: str = "spline"):
    """preprocess.py:181-195 (+ resample_to_axis :155-178).

    New axis ``np.linspace(t[0], t[-1], N)``; linear when kind == "linear" or
    m < 3 (:171), natural cubic spline otherwise.
    """
    t_old = np.asarray(t_old, dtype=float)
    t_new = np.linspace(t_old[0], t_old[-1], target_count)
    if kind == "linear" or t_old.size < 3:
        values = interp_linear(t_old, intensities, t_new)
    else:
        from scipy.interpolate import CubicSpline  # the reference's own dependency
        values = CubicSpline(t_old, intensities, axis=0, bc_type="natural")(t_new)
    return t_new, values


def stddev_spectrum(intensities: np.ndarray, reference: np.ndarray) -> np.ndarray:
    """preprocess.py:198-211 -- sqrt(sum_j (y_j - ref)^2 / (m - 1))."""
    m = intensities.shape[0]
    centered = intensities - reference[None, :]
    return np.sqrt((centered ** 2).sum(axis=0) / (m - 1))


def preprocess(t, intensities, *, resample=None, kind="spline", reference=None,
               alpha=0.0, on_zero_variance="error"):
    """preprocess.py:262-275 -- resample -> reference -> sigma -> scale.

    Returns (t_used, values, reference_used, sigma_or_None).  Zero-variance
    channels under alpha > 0 raise ValueError (policy "error") or get sigma=1
    (policy "substitute"), as apply_scaling (:214-259).
    """
    intensities = np.asarray(intensities, dtype=float)
    t = np.asarray(t, dtype=float)
    if resample is not None:
        t, intensities = resample_equidistant(t, intensities, resample, kind)
    ref = mean_reference(intensities) if reference is None else np.asarray(reference, dtype=float)
    values = intensities - ref[None, :]
    if alpha > 0.0:
        sigma = stddev_spectrum(intensities, ref)
        dead = sigma == 0.0
        if np.any(dead):
            if on_zero_variance == "error":
                raise ValueError("zero-variance spectral channel(s)")
            sigma = np.where(dead, 1.0, sigma)
        values = values / sigma[None, :] ** alpha
        return t, values, ref, sigma
    return t, values, ref, None


# --------------------------------------------------------------------------
# Fourier engine (fourier.py)
# --------------------------------------------------------------------------

def dft_channels(values: np.ndarray, workers: int = 1) -> np.ndarray:
    """fourier.py:61-82 -- rfft along the perturbation axis (K x n complex128)."""
    return scipy.fft.rfft(np.asarray(values, dtype=float), axis=0, workers=workers)


def _row_blocks(n_rows: int, workers: int):
    """engine_core.py:106-112 -- linspace bounds, at most `workers` blocks."""
    count = min(workers, n_rows)
    bounds = np.linspace(0, n_rows, count + 1).astype(int)
    return [slice(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]


def correlate_ft(values1, values2=None, norm: float | None = None, workers: int = 1,
                 rows: slice | None = None):
    """fourier.py:85-125 -- returns (sync, asyn, constant).

    C = Norm * sum_w weight(w) Y1(nu1, w) conj(Y2(nu2, w)); sync = Re, async = Im.
    ``rows`` restricts the output to a row block of the first operand -- the
    "row-block oracle" of SURVEY.md 8(c): the reference's rows R of the full
    result equal correlate_ft(dyn1[:, R], dyn2) bit-for-bit.
    """
    values1 = np.asarray(values1, dtype=float)
    homo = values2 is None
    values2 = values1 if homo else np.asarray(values2, dtype=float)
    m = values1.shape[0]
    constant = noda_constant(m) if norm is None else float(norm)
    half1 = dft_channels(values1 if rows is None else values1[:, rows], workers)
    half2 = half1 if (homo and rows is None) else dft_channels(values2, workers)
    w = half_spectrum_weights(m)
    weighted1 = half1.T * w
    conj2 = np.conj(half2)

    def block(r):
        return weighted1[r] @ conj2

    blocks = _row_blocks(weighted1.shape[0], workers)
    ctx = threadpool_limits(limits=1) if threadpool_limits is not None else _Null()
    with ctx:
        if workers == 1 or len(blocks) == 1:
            parts = [block(b) for b in blocks]
        else:
            with ThreadPoolExecutor(max_workers=len(blocks)) as pool:
                parts = list(pool.map(block, blocks))
    corr = np.concatenate(parts, axis=0)
    corr *= constant
    return corr.real.copy(), corr.imag.copy(), constant


def hilbert_noda_matrix(m: int) -> np.ndarray:
    """hilbert.py:40-48 -- N[j, k] = 1/(pi (k - j)), 0 on the diagonal."""
    idx = np.arange(m)
    with np.errstate(divide="ignore"):
        n = 1.0 / (np.pi * (idx[None, :] - idx[:, None]))
    np.fill_diagonal(n, 0.0)
    return n


def correlate_ht(values1, values2=None, norm: float | None = None):
    """hilbert.py:92-115 -- returns (sync, asyn, constant).

    sync = Norm * Y1^T Y2, async = Norm * Y1^T (N Y2), Norm default 1/(m - 1)
    (the dense N of hilbert.py:51-53; the reference's Toeplitz branch above
    m = 4096 applies the same matrix).
    """
    values1 = np.asarray(values1, dtype=float)
    values2 = values1 if values2 is None else np.asarray(values2, dtype=float)
    m = values1.shape[0]
    constant = unit_constant(m) if norm is None else float(norm)
    transformed = hilbert_noda_matrix(m) @ values2
    sync = constant * (values1.T @ values2)
    asyn = constant * (values1.T @ transformed)
    return sync, asyn, constant


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
