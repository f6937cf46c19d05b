"""Device orchestration: buffers, launches and error checks around libcorr2d.

PyTorch is used only as plumbing -- device allocation (caching allocator),
the current CUDA stream, pinned host buffers and CUDA graphs.  All arithmetic
of the hot path runs in the hand-written sm_100a kernels behind the C ABI.

The central object is :class:`CorrelationPlan`: for one problem shape it owns
the packed-operand workspaces and the output planes, ``launch()`` enqueues the
whole device pipeline on the current stream without synchronising (so it can
be captured in a CUDA graph), and ``finish()`` synchronises, turns the device
status words into the reference's exceptions and copies results to the host.
"""

from __future__ import annotations

import ctypes
import os
import threading
import warnings
from dataclasses import dataclass

import numpy as np

from . import _abi
from .errors import DataError, NumericError

_torch = None


def fp32_pack_kind() -> int:
    """Operand format of the float32 (tensor-core) path: CORR2D_PACK_F16F8
    (fp16 hi.hi + e4m3 cross terms, default) or CORR2D_PACK_BF16X2 (bf16x3);
    CORR2D_FP32_FORMAT=bf16x3 selects the latter (include/corr2d.h)."""
    fmt = os.environ.get("CORR2D_FP32_FORMAT", "f16f8").lower()
    if fmt == "bf16x3":
        return _abi.PACK_BF16X2
    if fmt == "f16f8":
        return _abi.PACK_F16F8
    raise DataError(f"CORR2D_FP32_FORMAT must be f16f8 or bf16x3, got {fmt!r}")


def f64_pack_kind() -> int:
    """Operand format of the float64 Fourier route: CORR2D_PACK_F64_GAUSS (three
    real products per bin, default) or CORR2D_PACK_F64 (four; CORR2D_F64_FORMAT=
    four), both exact rewrites of the complex half-spectrum sum (corr2d.h)."""
    fmt = os.environ.get("CORR2D_F64_FORMAT", "gauss").lower()
    if fmt == "gauss":
        return _abi.PACK_F64_GAUSS
    if fmt == "four":
        return _abi.PACK_F64
    raise DataError(f"CORR2D_F64_FORMAT must be gauss or four, got {fmt!r}")


def launch_contract_f64(lib, pack_kind, a_phi, a_psi, b, ld_pack, n1, n2, mp, homo, row0, row1, tile0, tile1,
                        phi, psi, ld_out, stats):
    """The fp64 contraction for either operand format (pointers are tensors)."""
    if pack_kind == _abi.PACK_F64_GAUSS:
        code = lib.corr2d_contract_f64_gauss(
            ptr(a_phi), ptr(b), ld_pack, n1, n2, mp // 3, homo, row0, row1, tile0, tile1,
            ptr(phi), ptr(psi), ld_out, ptr(stats), stream_handle())
    else:
        code = lib.corr2d_contract_f64(
            ptr(a_phi), ptr(a_psi), ptr(b), ld_pack, n1, n2, mp, homo, row0, row1, tile0, tile1,
            ptr(phi), ptr(psi), ld_out, ptr(stats), stream_handle())
    _abi.check(code, lib)


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_device(device=None):
    """The CUDA device to run on; raises BackendUnavailable without one."""
    t = torch()
    lib = _abi.load()
    if not t.cuda.is_available():
        raise _abi.BackendUnavailable("no CUDA device visible: the corr2d GPU path has no CPU fallback")
    if device is None:
        dev = t.device("cuda", t.cuda.current_device())
    elif isinstance(device, t.device):
        dev = device if device.index is not None else t.device("cuda", t.cuda.current_device())
    else:
        dev = t.device("cuda", int(device))
    return lib, dev


class device_scope:
    """Run a call on `dev`: makes it the current CUDA device (the C entry points
    read the SM count and launch on the current device) and its current stream
    the one kernels are launched on."""

    def __init__(self, dev):
        self.dev = dev
        self._ctx = None

    def __enter__(self):
        t = torch()
        if self.dev is not None and self.dev.type == "cuda" and self.dev.index != t.cuda.current_device():
            self._ctx = t.cuda.device(self.dev)
            self._ctx.__enter__()
        return self.dev

    def __exit__(self, *exc):
        if self._ctx is not None:
            self._ctx.__exit__(*exc)
        return False


def on_device(fn):
    """Decorator for public entry points with a ``device=`` keyword: the whole
    call (plan build, launches, synchronisation, copies) runs with that device
    current, so kernels, streams and pointers all belong to it."""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        device = kwargs.get("device")
        if device is None:
            return fn(*args, **kwargs)
        _, dev = require_device(device)
        kwargs["device"] = dev
        with device_scope(dev):
            return fn(*args, **kwargs)
    return wrapper


def stream_handle():
    return ctypes_void(torch().cuda.current_stream().cuda_stream)


def ctypes_void(x):
    return None if x is None or x == 0 else int(x)


def ptr(t):
    return None if t is None else int(t.data_ptr())


def to_device(arr, dev, dtype=None):
    t = torch()
    if isinstance(arr, t.Tensor):
        out = arr.to(device=dev, dtype=dtype or arr.dtype)
        return out.contiguous()
    a = np.ascontiguousarray(arr)
    host = t.from_numpy(a)
    if dtype is not None and host.dtype != dtype:
        host = host.to(dtype)
    return host.to(dev, non_blocking=False)


# --------------------------------------------------------------------------
# resampling plans (host side, tiny: O(m * m_in))
# --------------------------------------------------------------------------

@dataclass
class ResamplePlan:
    kind: int                     # _abi.RESAMPLE_*
    t_new: np.ndarray
    lin_idx: np.ndarray | None = None
    lin_frac: np.ndarray | None = None
    matrix: np.ndarray | None = None
    _dev: dict | None = None

    def device(self, dev):
        if self._dev is None:
            self._dev = {}
        key = str(dev)
        if key not in self._dev:
            t = torch()
            d = {}
            if self.lin_idx is not None:
                d["idx"] = to_device(self.lin_idx.astype(np.int32), dev)
                d["frac"] = to_device(self.lin_frac.astype(np.float64), dev)
            if self.matrix is not None:
                d["mat"] = to_device(np.ascontiguousarray(self.matrix, dtype=np.float64), dev)
            self._dev[key] = d
        return self._dev[key]


def linear_plan(t_old: np.ndarray, t_new: np.ndarray) -> ResamplePlan:
    """Index/fraction pairs computed with the reference's own numpy ops
    (preprocess.py:149-151), so the device interpolation matches bit-for-bit."""
    t_old = np.asarray(t_old, dtype=np.float64)
    t_new = np.asarray(t_new, dtype=np.float64)
    idx = np.clip(np.searchsorted(t_old, t_new, side="right") - 1, 0, t_old.size - 2)
    lo, hi = t_old[idx], t_old[idx + 1]
    frac = (t_new - lo) / (hi - lo)
    return ResamplePlan(_abi.RESAMPLE_LINEAR, t_new, lin_idx=idx, lin_frac=frac)


def spline_matrix(t_old: np.ndarray, t_new: np.ndarray) -> np.ndarray:
    """Natural cubic spline (zero end curvature) as a dense len(t_new) x len(t_old)
    linear map: value(t_new) = S @ y.  Restates preprocess.py:174-175
    (scipy CubicSpline, bc_type="natural") via the moment equations
      h_{i-1} M_{i-1} + 2 (h_{i-1} + h_i) M_i + h_i M_{i+1} = 6 (d_i - d_{i-1}),
    solved once for all unit data vectors."""
    x = np.asarray(t_old, dtype=np.float64)
    q = np.asarray(t_new, dtype=np.float64)
    n = x.size
    h = np.diff(x)
    ident = np.eye(n)
    moments = np.zeros((n, n))
    if n > 2:
        k = n - 2
        lhs = np.diag(2.0 * (h[:-1] + h[1:]))
        if k > 1:
            lhs += np.diag(h[1:-1], 1) + np.diag(h[1:-1], -1)
        slope = (ident[1:] - ident[:-1]) / h[:, None]          # (n-1) x n divided differences
        moments[1:-1] = np.linalg.solve(lhs, 6.0 * (slope[1:] - slope[:-1]))
    seg = np.clip(np.searchsorted(x, q, side="right") - 1, 0, n - 2)
    d = (q - x[seg])[:, None]
    hs = h[seg][:, None]
    y0, y1 = ident[seg], ident[seg + 1]
    m0, m1 = moments[seg], moments[seg + 1]
    b = (y1 - y0) / hs - hs * (2.0 * m0 + m1) / 6.0
    return y0 + d * (b + d * (m0 / 2.0 + d * (m1 - m0) / (6.0 * hs)))


def resample_plan(t_old, target_count: int, interpolant: str) -> ResamplePlan:
    """np.linspace(t[0], t[-1], N) target axis (preprocess.py:195); linear when
    requested or m < 3 (:171), natural spline otherwise."""
    t_old = np.asarray(t_old, dtype=np.float64)
    t_new = np.linspace(t_old[0], t_old[-1], int(target_count))
    return axis_plan(t_old, t_new, interpolant)


def axis_plan(t_old, t_new, interpolant: str) -> ResamplePlan:
    t_old = np.asarray(t_old, dtype=np.float64)
    t_new = np.asarray(t_new, dtype=np.float64)
    if t_new[0] < t_old[0] or t_new[-1] > t_old[-1]:
        raise DataError(
            f"target axis [{t_new[0]:g}, {t_new[-1]:g}] extends beyond "
            f"the data range [{t_old[0]:g}, {t_old[-1]:g}]")
    if interpolant == "linear" or t_old.size < 3:
        return linear_plan(t_old, t_new)
    if interpolant == "spline":
        return ResamplePlan(_abi.RESAMPLE_MATRIX, t_new, matrix=spline_matrix(t_old, t_new))
    raise DataError(f"unknown interpolant {interpolant!r}")


# --------------------------------------------------------------------------
# K1 launcher
# --------------------------------------------------------------------------

@dataclass
class PrepRecipe:
    """How one dataset becomes packed operands / dynamic values on the device."""
    m_in: int
    m: int
    ref_mode: int = _abi.REF_MEAN     # REF_NONE: input already dynamic
    resample: ResamplePlan | None = None
    ref_in: object = None             # device tensor (n,) for REF_PROVIDED
    sigma_in: object = None           # device tensor (n,): provided sigma
    alpha: float = 0.0
    substitute: bool = False


def small_fused_enabled() -> bool:
    """The small-m path (csrc/small_path.cu; CORR2D_SMALL_FUSED=0 selects the
    generic K1 + fp64 contraction instead, for A/B comparisons)."""
    import os
    return os.environ.get("CORR2D_SMALL_FUSED", "1") != "0"


def small_one_kernel() -> bool:
    """CORR2D_SMALL_ONEKERNEL=1: the small-m path's one-kernel variant
    (small_fused_kernel: no operand rows in global memory) instead of K1 +
    streamed contraction; read at every launch."""
    import os
    return os.environ.get("CORR2D_SMALL_ONEKERNEL", "0") == "1"


def launch_prep(lib, raw, recipe: PrepRecipe, *, norm=0.0, pack_kind=_abi.PACK_NONE, roles=0,
                a_phi=None, a_psi=None, b=None, ld_pack=0, split_plane=0,
                values_out=None, half_out=None, ref_out=None, sigma_out=None, status=None):
    t = torch()
    if raw.dtype == t.float64:
        in_dtype = _abi.F64
    elif raw.dtype == t.float32:
        in_dtype = _abi.F32
    else:
        raise DataError(f"unsupported intensity dtype {raw.dtype}")
    m_in, n = raw.shape
    rs = recipe.resample
    rsd = rs.device(raw.device) if rs is not None else {}
    code = lib.corr2d_prep(
        in_dtype, ptr(raw), raw.stride(0), m_in, n,
        rs.kind if rs is not None else _abi.RESAMPLE_NONE,
        ptr(rsd.get("idx")), ptr(rsd.get("frac")), ptr(rsd.get("mat")), recipe.m,
        int(recipe.ref_mode), ptr(recipe.ref_in), ptr(recipe.sigma_in), float(recipe.alpha),
        1 if recipe.substitute else 0, float(norm), pack_kind, roles,
        ptr(a_phi), ptr(a_psi), ptr(b), int(ld_pack), int(split_plane),
        ptr(values_out), n if values_out is not None else 0, ptr(half_out),
        ptr(ref_out), ptr(sigma_out), ptr(status), stream_handle())
    _abi.check(code, lib)


def decode_status(st: np.ndarray):
    """(nonfinite count, zero-variance count, first zero-variance channel or -1)."""
    first = int(st[_abi.ST_FIRST_ZEROVAR])
    return int(st[_abi.ST_NONFINITE]), int(st[_abi.ST_ZEROVAR]), (_abi.INT32_MAX - first) if first else -1


def handle_zero_variance(spectral_axis, sigma_raw: np.ndarray, alpha: float, substitute: bool):
    """apply_scaling's zero-variance policy (preprocess.py:238-254), given the
    device sigma BEFORE substitution.  Raises NumericError ("error" policy) or
    warns and returns the substituted sigma ("substitute" policy)."""
    dead = sigma_raw == 0.0
    if not dead.any():
        return sigma_raw
    positions = np.asarray(spectral_axis)[dead]
    shown = ", ".join(f"{p:g}" for p in positions[:5])
    if not substitute:
        more = " ..." if positions.size > 5 else ""
        raise NumericError(f"zero-variance spectral channel(s) at {shown}{more}; "
                           f"cannot scale with alpha = {alpha:g}")
    warnings.warn(f"substituting sigma = 1 for zero-variance channel(s) at {shown}",
                  RuntimeWarning, stacklevel=4)
    return np.where(dead, 1.0, sigma_raw)


# --------------------------------------------------------------------------
# the correlation plan (K1 x {1,2} -> K2)
# --------------------------------------------------------------------------

def _noda_rows(m: int, ld: int) -> np.ndarray:
    """-N as m rows of ld float64 (zero padded): N[j, k] = 1 / (pi (k - j)),
    0 on the diagonal -- the Hilbert-Noda matrix of hilbert.py:40-48."""
    idx = np.arange(m)
    with np.errstate(divide="ignore"):
        n = 1.0 / (np.pi * (idx[None, :] - idx[:, None]))
    np.fill_diagonal(n, 0.0)
    out = np.zeros((m, ld))
    out[:, :m] = -n
    return out


class CorrelationPlan:
    """Device pipeline for one correlation shape.

    inputs  : one (homo) or two (hetero) device tensors m_in x n (f64 or f32)
    outputs : sync / async planes for rows [row0, row1) x n2 (f64 or f32)
    """

    def __init__(self, *, n1, n2, m, recipe1: PrepRecipe, recipe2: PrepRecipe | None,
                 norm: float, dtype="float64", rows=None, device=None, want_ref=True,
                 want_sigma=False, tiles=None, route="fourier"):
        self.lib, self.dev = require_device(device)
        t = torch()
        self.homo = recipe2 is None
        if self.homo and n1 != n2:
            raise DataError("homo correlation needs n1 == n2")
        self.n1, self.n2, self.m = int(n1), int(n2), int(m)
        self.recipe1, self.recipe2 = recipe1, recipe2
        self.norm = float(norm)
        self.dtype = np.dtype(dtype)
        if route not in ("fourier", "hilbert"):
            raise DataError(f"unknown route {route!r}")
        self.route = route
        if route == "hilbert":
            # Hilbert-Noda route (hilbert.py:92-115): time-domain operands, fp64 only
            if self.dtype != np.float64:
                raise DataError("the Hilbert route computes in float64 only")
            self.pack_kind, odt, pdt = _abi.PACK_F64_TIME, t.float64, t.float64
        elif self.dtype == np.float64:
            self.pack_kind, odt, pdt = f64_pack_kind(), t.float64, t.float64
        elif self.dtype == np.float32:
            self.pack_kind, odt, pdt = fp32_pack_kind(), t.float32, t.bfloat16
        else:
            raise DataError(f"unsupported compute dtype {dtype}")
        self.gauss = self.pack_kind == _abi.PACK_F64_GAUSS
        self.mp = self.lib.corr2d_packed_depth(self.m, self.pack_kind)
        if self.mp <= 0:
            _abi.check(_abi.ERR_DATA, self.lib)
        self.row0, self.row1 = (0, self.n1) if rows is None else (int(rows[0]), int(rows[1]))
        # tile-range partition of the (shard's) tile enumeration; -1 = to the end
        self.tile0, self.tile1 = (0, -1) if tiles is None else (int(tiles[0]), int(tiles[1]))
        bf16 = self.pack_kind in (_abi.PACK_BF16X2, _abi.PACK_F16F8)
        # row pitch of the packed operands: bf16 rows carry hi and lo of every
        # slot, interleaved per 32-slot block, then the fp32 DC / Nyquist pair
        # in a 128-byte pad (include/corr2d.h)
        self.ld_pack = 2 * self.mp + 64 if bf16 else self.mp
        # small m (fp64 Fourier route, m <= 32, no resampling, whole map): the
        # whole call is one C call (csrc/small_path.cu): K1 once per channel +
        # the streamed contraction, or the one-kernel variant
        self.small = (route == "fourier" and self.dtype == np.float64
                      and small_fused_enabled() and 2 <= self.m <= 32
                      and all(r is None or (r.resample is None and r.m_in == r.m) for r in (recipe1, recipe2))
                      and (recipe2 is None or (recipe2.alpha == recipe1.alpha
                                               and recipe2.substitute == recipe1.substitute))
                      and self.row0 == 0 and self.row1 == self.n1 and tiles is None)
        dev = self.dev
        R1, R2 = self.n1, self.n2
        alloc = t.empty
        if self.small:
            # the small path's Gauss operand rows (the two-kernel variant's K1 ->
            # contraction, L2-resident; the one-kernel variant keeps them in
            # shared memory)
            self.ld_pack = self.lib.corr2d_small_ops_depth(self.m)
            self.mp = self.ld_pack
        O1, O2 = (R1, R2)
        self.a_phi = alloc((O1, self.ld_pack), dtype=pdt, device=dev)
        # bf16: one format for both roles (a_psi unused, homo B == A)
        self.a_psi = None if (bf16 or self.gauss) else alloc((O1, self.ld_pack), dtype=pdt, device=dev)
        if route == "hilbert":
            # A_psi = -Norm * (N y1) comes from one contraction of A_phi = Norm * y1
            # against the rows of -N (m x mp, zero padded); columns m..mp of
            # A_psi are never written and stay 0
            self.a_psi = t.zeros((R1, self.ld_pack), dtype=pdt, device=dev)
            self.noda_neg = t.from_numpy(_noda_rows(self.m, self.ld_pack)).to(dev)
            self.noda_scratch = t.empty((self.n1, self.ld_pack), dtype=pdt, device=dev)
        self.b = alloc((O2, self.ld_pack), dtype=pdt, device=dev) if not self.homo else None
        if self.homo:
            self.b_homo = self.a_phi if bf16 else alloc((O1, self.ld_pack), dtype=pdt, device=dev)
        else:
            self.b_homo = None
        nrows = self.row1 - self.row0
        try:
            self.phi = t.empty((nrows, self.n2), dtype=odt, device=dev)
            self.psi = t.empty((nrows, self.n2), dtype=odt, device=dev)
        except t.cuda.OutOfMemoryError:
            raise NumericError(
                f"out of memory assembling the complex correlation matrix; it needs "
                f"16*{self.n1}*{self.n2} bytes = {16 * self.n1 * self.n2 / 1e9:.2f} GB") from None
        self.stats = t.zeros(4, dtype=t.int64, device=dev)
        # fused small-m path: self-resetting K1 status / stat accumulators
        self.work = t.zeros(16, dtype=t.int32, device=dev) if self.small else None
        self.status1 = t.zeros(4, dtype=t.int32, device=dev)
        self.status2 = t.zeros(4, dtype=t.int32, device=dev)
        self.ref1 = alloc(R1, dtype=t.float64, device=dev) if want_ref else None
        self.ref2 = (alloc(R2, dtype=t.float64, device=dev) if (want_ref and not self.homo) else None)
        self.sigma1 = alloc(R1, dtype=t.float64, device=dev) if want_sigma else None
        self.sigma2 = (alloc(R2, dtype=t.float64, device=dev) if (want_sigma and not self.homo) else None)
        self.raw1 = self.raw2 = None
        if self.small:
            # pipelined small-m calls (corr2d_correlate_small_f64_slot): two
            # scratch slots -- operand rows, stats, work and status words --
            # used by alternate launches, and the plan's {busy, arrival} words
            names = ("a_phi", "b", "b_homo", "stats", "work", "status1", "status2")
            second = {k: (None if getattr(self, k) is None else
                          (t.zeros_like(getattr(self, k)) if k in ("stats", "work", "status1", "status2")
                           else t.empty_like(getattr(self, k)))) for k in names}
            self._slots = [{k: getattr(self, k) for k in names}, second]
            self._slot = 0
            self.pipe = t.zeros(16, dtype=t.int64, device=dev)

    @property
    def bop(self):
        return self.b_homo if self.homo else self.b

    def bind(self, raw1, raw2=None):
        if raw1.shape[1] != self.n1 or (raw2 is not None and raw2.shape[1] != self.n2):
            raise DataError("bound inputs do not match the plan's shape")
        self.raw1, self.raw2 = raw1, raw2
        return self

    def tile_count(self) -> int:
        """Tiles in the contraction kernel's enumeration for this plan (the unit
        of the multi-GPU tile-range partition; include/corr2d.h)."""
        if self.small:
            n = self.lib.corr2d_small_block_count(self.n1, self.n2, 1 if self.homo else 0)
            if n < 0:
                raise DataError("bad contraction shape")
            return int(n)
        n = self.lib.corr2d_contract_tile_count(self.pack_kind, self.n1, self.n2, 1 if self.homo else 0,
                                                self.row0, self.row1, self.n2)
        if n < 0:
            raise DataError("bad contraction shape")
        return int(n)

    @property
    def launches_per_step(self) -> int:
        """Kernels of ours one launch() enqueues: K1 per dataset + K2 (the
        small-m path: one fused kernel, or K1 + contraction)."""
        if self.small:
            return 1 if small_one_kernel() else int(self.lib.corr2d_small_launches(self.n1, self.n2,
                                                                                   1 if self.homo else 0))
        return (1 if self.homo else 2) + (2 if self.route == "hilbert" else 1)

    def launch(self):
        """Enqueue K1 (x1 or x2) and K2 on the current stream; no host sync."""
        self.launch_prep_only()
        self.launch_contract()

    def launch_prep_only(self):
        if self.small:
            return                      # K1 runs inside the fused kernel (launch_contract)
        lib = self.lib
        roles1 = _abi.ROLE_A | (_abi.ROLE_B if self.homo else 0)
        if self.pack_kind in (_abi.PACK_BF16X2, _abi.PACK_F16F8) and self.homo:
            roles1 = _abi.ROLE_A
        launch_prep(lib, self.raw1, self.recipe1, norm=self.norm, pack_kind=self.pack_kind, roles=roles1,
                    a_phi=self.a_phi, a_psi=self.a_psi, b=self.b_homo if self.homo else None,
                    ld_pack=self.ld_pack, ref_out=self.ref1,
                    sigma_out=self.sigma1, status=self.status1)
        if not self.homo:
            launch_prep(lib, self.raw2, self.recipe2, norm=self.norm, pack_kind=self.pack_kind,
                        roles=_abi.ROLE_B, b=self.b, ld_pack=self.ld_pack,
                        ref_out=self.ref2, sigma_out=self.sigma2, status=self.status2)

    def launch_contract(self):
        lib = self.lib
        if self.small:
            self._launch_small()
            return
        homo = 1 if self.homo else 0
        if self.route == "hilbert":
            # A_psi[i, s] = sum_k A_phi[i, k] * (-N[s, k]) = -Norm (N y1)[s, i]
            code = lib.corr2d_contract_f64(
                ptr(self.a_phi), ptr(self.a_phi), ptr(self.noda_neg), self.ld_pack, self.n1, self.m, self.mp,
                0, 0, self.n1, 0, -1, ptr(self.a_psi), ptr(self.noda_scratch), self.ld_pack,
                ptr(self.stats), stream_handle())
            _abi.check(code, lib)
        if self.pack_kind in (_abi.PACK_F64, _abi.PACK_F64_TIME, _abi.PACK_F64_GAUSS):
            launch_contract_f64(lib, self.pack_kind, self.a_phi, self.a_psi, self.bop, self.ld_pack, self.n1,
                                self.n2, self.mp, homo, self.row0, self.row1, self.tile0, self.tile1,
                                self.phi, self.psi, self.phi.stride(0), self.stats)
            return
        else:
            code = lib.corr2d_contract_tc(
                self.pack_kind, ptr(self.a_phi), ptr(self.bop), self.ld_pack, self.n1, self.n2, self.mp, self.m, homo,
                self.row0, self.row1, self.tile0, self.tile1, ptr(self.phi), ptr(self.psi), self.phi.stride(0),
                ptr(self.stats), stream_handle())
        _abi.check(code, lib)

    def _launch_small(self):
        t = torch()
        raw1, raw2 = self.raw1, self.raw2
        if raw1.dtype not in (t.float64, t.float32) or (raw2 is not None and raw2.dtype != raw1.dtype):
            raise DataError(f"unsupported intensity dtype {raw1.dtype}")
        r1, r2 = self.recipe1, self.recipe2 or self.recipe1
        one = small_one_kernel()
        # alternate scratch slots: this launch's K1 may run while the previous
        # launch's contraction still reads the other slot
        self._slot ^= 1
        for k, v in self._slots[self._slot].items():
            setattr(self, k, v)
        code = self.lib.corr2d_correlate_small_f64_slot(
            _abi.F64 if raw1.dtype == t.float64 else _abi.F32,
            ptr(raw1), raw1.stride(0), ptr(raw2), raw2.stride(0) if raw2 is not None else 0,
            self.m, self.n1, self.n2,
            int(r1.ref_mode), ptr(r1.ref_in), ptr(r1.sigma_in), int(r2.ref_mode), ptr(r2.ref_in), ptr(r2.sigma_in),
            float(r1.alpha), 1 if r1.substitute else 0, self.norm,
            *((None, None) if one else (ptr(self.a_phi), ptr(self.bop))), self.ld_pack,
            ptr(self.ref1), ptr(self.sigma1), ptr(self.ref2), ptr(self.sigma2),
            ptr(self.phi), ptr(self.psi), self.phi.stride(0),
            ptr(self.status1), ptr(self.status2), ptr(self.stats), ptr(self.work), stream_handle(),
            self._slot, ptr(self.pipe))
        _abi.check(code, self.lib)

    def check(self, axes=(None, None), labels=("first", "second")):
        """After the stream synchronised: raise the reference's errors, apply
        the zero-variance policy; returns host (ref1, ref2, sigma1, sigma2, stats).
        Every status / stat / reference / sigma word comes back in ONE
        device -> host transfer."""
        h = readback({"st1": self.status1, "st2": None if self.homo else self.status2, "stats": self.stats,
                      "ref1": None if self.ref1 is None else self.ref1[:self.n1],
                      "ref2": None if self.ref2 is None else self.ref2[:self.n2],
                      "sig1": None if self.sigma1 is None else self.sigma1[:self.n1],
                      "sig2": None if self.sigma2 is None else self.sigma2[:self.n2]})
        for st, lab in ((h["st1"], labels[0]), (h["st2"], labels[1])):
            if st is not None and int(st[_abi.ST_NONFINITE]):
                raise NumericError(f"{lab} dynamic-spectra matrix contains non-finite values")
        sig = []
        for recipe, sh, axis in ((self.recipe1, h["sig1"], axes[0]), (self.recipe2, h["sig2"], axes[1])):
            if recipe is None or sh is None:
                sig.append(None)
                continue
            sig.append(handle_zero_variance(axis, sh, recipe.alpha, recipe.substitute))
        stats = h["stats"]
        if int(stats[2]):
            raise NumericError("correlation produced non-finite values")
        info = {"max_abs_sync": float(stats[0:1].view(np.float64)[0]),
                "max_abs_async": float(stats[1:2].view(np.float64)[0])}
        ref1 = h["ref1"]
        ref2 = h["ref2"] if h["ref2"] is not None else ref1
        if self.homo:
            sig.append(None)
            sig[1] = sig[0]
        return ref1, ref2, sig[0], sig[1], info

    def fetch(self, out=None, wait: bool = True):
        """Device -> host copy of both planes (into `out` or fresh pinned
        buffers).  wait=False queues the copies behind the launched kernels
        and returns (sync, asyn, done): done() waits for them."""
        t = torch()
        if out is None:
            hs = t.empty(self.phi.shape, dtype=self.phi.dtype, pin_memory=True)
            ha = t.empty(self.psi.shape, dtype=self.psi.dtype, pin_memory=True)
        else:
            hs, ha = (t.from_numpy(o) if isinstance(o, np.ndarray) else o for o in out)
        if self._fetch_mirrored_ok(hs, ha):
            done = fetch_mirrored(self.lib, self.phi, self.psi, hs, ha, wait=wait)
        else:
            global last_fetch_bytes
            last_fetch_bytes = hs.numel() * hs.element_size() + ha.numel() * ha.element_size()
            done = copy_d2h([(hs, self.phi), (ha, self.psi)], wait=wait)
        if wait:
            return hs.numpy(), ha.numpy()
        return hs.numpy(), ha.numpy(), done

    def _fetch_mirrored_ok(self, hs, ha) -> bool:
        """A whole homo Fourier map of at least MIRROR_MIN_N rows, contiguous on
        both sides, with a nonzero MIRROR_FILL_PCT: its D2H leaves part of the
        lower triangle to the host (fetch_mirrored)."""
        if os.environ.get("CORR2D_FETCH_FULL") == "1" or MIRROR_FILL_PCT <= 0:
            return False
        n = self.n1
        return (self.homo and self.route == "fourier" and n >= MIRROR_MIN_N
                and (self.row0, self.row1) == (0, n) and (self.tile0, self.tile1) == (0, -1)
                and all(x.dim() == 2 and tuple(x.shape) == (n, n) and x.is_contiguous()
                        for x in (self.phi, self.psi, hs, ha))
                and hs.dtype == self.phi.dtype and ha.dtype == self.psi.dtype)

    def run_to_host(self, out=None, axes=(None, None), labels=("first", "second")):
        """launch() + the planes' D2H queued right behind the kernels, the
        status readback / error checks overlapping that transfer; returns
        (sync, asyn, check() results).  The copies have landed when this
        returns or raises."""
        self.launch()
        s, a, done = self.fetch(out, wait=False)
        try:
            res = self.check(axes=axes, labels=labels)
        finally:
            done()
        return s, a, res


def readback(tensors: dict) -> dict:
    """Small device tensors -> host numpy arrays with ONE device -> host copy
    (their bytes concatenated on the device), instead of one synchronous
    transfer each.  None entries stay None."""
    t = torch()
    live = [(k, x) for k, x in tensors.items() if x is not None and x.numel()]
    out = {k: (None if x is None else np.empty(0, dtype=_np_dtype(x))) for k, x in tensors.items()}
    if not live:
        return out
    flat = t.cat([x.contiguous().reshape(-1).view(t.uint8) for _, x in live]).cpu().numpy()
    o = 0
    for k, x in live:
        nb = x.numel() * x.element_size()
        out[k] = flat[o:o + nb].view(_np_dtype(x)).reshape(tuple(x.shape))
        o += nb
    return out


def _np_dtype(x):
    return {"torch.float64": np.float64, "torch.float32": np.float32, "torch.int32": np.int32,
            "torch.int64": np.int64}[str(x.dtype)]


def device_budget(dev) -> int:
    """Bytes of device memory the output planes of one launch may take:
    CORR2D_DEVICE_BUDGET (bytes) if set, else 85 % of the free memory."""
    import os
    env = os.environ.get("CORR2D_DEVICE_BUDGET")
    if env:
        return int(float(env))
    free, _ = torch().cuda.mem_get_info(dev)
    return int(free * 0.85)


_total_mem = {}


def planes_fit_easily(n1: int, n2: int, elem: int, dev) -> bool:
    """True when the two output planes take under 1/8 of the device's total
    memory: such maps never stream, and the call skips the (synchronising)
    free-memory query of device_budget."""
    import os
    if os.environ.get("CORR2D_DEVICE_BUDGET"):
        return False
    key = str(dev)
    if key not in _total_mem:
        _total_mem[key] = torch().cuda.get_device_properties(dev).total_memory
    return 2 * n1 * n2 * elem * 8 <= _total_mem[key]


def maybe_stream_blocks(n1: int, n2: int, elem: int, dev):
    """stream_blocks against the device budget, or None without querying the
    free memory when the planes fit easily."""
    if planes_fit_easily(n1, n2, elem, dev):
        return None
    return stream_blocks(n1, n2, elem, device_budget(dev))


def stream_blocks(n1: int, n2: int, elem: int, budget: int, align: int = 128):
    """Row blocks [r0, r1) (multiples of `align`, the contraction kernels' row
    tile) whose two output planes fit in `budget` bytes, or None when the whole
    map fits.  Maps larger than device memory are then computed block by block
    and streamed to the host result, as the reference computes any map that
    fits in host memory (row shards are bit-identical to the whole map)."""
    if n1 * n2 * 2 * elem <= budget:
        return None
    rows = max(align, (budget // (n2 * 2 * elem)) // align * align)
    return [(r, min(n1, r + rows)) for r in range(0, n1, rows)]


def run_streamed(make_plan, n1: int, n2: int, dtype, blocks, out=None, check=None):
    """Launch one plan per row block (make_plan(rows) -> bound plan), copy each
    block's planes into the host result; returns (sync, asyn, stats)."""
    import warnings
    if out is None:
        hs = np.empty((n1, n2), dtype=dtype)
        ha = np.empty((n1, n2), dtype=dtype)
    else:
        hs, ha = out
    stats = {"max_abs_sync": 0.0, "max_abs_async": 0.0}
    first = None
    plan = None
    for k, (r0, r1) in enumerate(blocks):
        plan = None                   # release the previous block's planes first
        plan = make_plan((r0, r1))
        plan.launch()
        sync()
        with warnings.catch_warnings():
            if k:
                warnings.simplefilter("ignore", RuntimeWarning)   # zero-variance notice once
            res = check(plan) if check is not None else plan.check()
        if first is None:
            first = res
        info = res[-1]
        stats["max_abs_sync"] = max(stats["max_abs_sync"], info["max_abs_sync"])
        stats["max_abs_async"] = max(stats["max_abs_async"], info["max_abs_async"])
        plan.fetch((hs[r0:r1], ha[r0:r1]))
    return hs, ha, stats, first


_copy_streams = {}


# homo maps from this many rows on send only part of their lower triangle, the
# host fills the rest as the mirror (fetch_mirrored); band = rows per transfer
# band (a multiple of the 256-row contraction tile); fill_pct = the share of each
# band's lower part the host fills.  The transpose fill competes with the DMA for
# the host's memory bandwidth: on the B200 boxes' 16-thread hosts 25-35 % is
# best (public-call e2e cfg5 154 -> 143-148 ms, cfg3 76.7 -> 75.0 ms), the
# upper triangle alone (100 %) loses 30 % (profiles/r2_fetch_e2e_ab.txt,
# r2_fetch_probe.txt).  CORR2D_FETCH_FILL_PCT=0 = the plain full-plane copy.
MIRROR_MIN_N = 16384   # cfg4's 8192^2 fp64 map loses 7 % with it (19.3 -> 20.8 ms per call)
MIRROR_BAND = 1024
MIRROR_FILL_PCT = int(os.environ.get("CORR2D_FETCH_FILL_PCT", "30"))
MIRROR_THREADS = int(os.environ.get("CORR2D_FETCH_THREADS", "0"))   # 0 = the host threads available (<= 32)
last_fetch_bytes = 0   # device -> host bytes of the last plan fetch (bench.py's e2e line)


def fetch_mirrored(lib, phi, psi, hs, ha, wait: bool = True, band: int = MIRROR_BAND, fill_pct: int | None = None,
                   threads: int | None = None):
    """Device -> host copy of a homo map's two n x n planes through
    corr2d_fetch_mirrored: row bands cross PCIe without the first fill_pct %
    of their lower part, which host threads fill as (sync^T, -async^T) from
    rows already landed while later bands are in flight (csrc/fetch.cu);
    bit-identical to a full-plane copy.  Ordered after the current stream's work; wait=False returns at once
    with the function that waits for completion (the call runs on a helper
    thread; ctypes releases the GIL)."""
    global last_fetch_bytes
    t = torch()
    n = phi.shape[0]
    dt = _abi.F64 if phi.dtype == t.float64 else _abi.F32
    if threads is None:
        threads = MIRROR_THREADS or min(32, len(os.sched_getaffinity(0)))
    if fill_pct is None:
        fill_pct = MIRROR_FILL_PCT
    dev = phi.device
    stream = stream_handle()
    nbytes = ctypes.c_int64(0)
    box = {}

    def run():
        try:
            with t.cuda.device(dev):
                rc = lib.corr2d_fetch_mirrored(dt, phi.data_ptr(), psi.data_ptr(), n, n, hs.data_ptr(),
                                               ha.data_ptr(), n, band, fill_pct, threads, ctypes.byref(nbytes), stream)
                _abi.check(rc, lib)   # the error message is per thread: raise here
        except Exception as e:        # re-raised by finish() on the caller's thread
            box["exc"] = e

    def finish():
        if "exc" in box:
            raise box["exc"]
        global last_fetch_bytes
        last_fetch_bytes = int(nbytes.value)

    if wait:
        run()
        finish()
        return None
    th = threading.Thread(target=run, name="corr2d-fetch", daemon=True)
    th.start()

    def done():
        th.join()
        finish()
    return done


def copy_d2h(pairs, streams: int = 4, chunk_bytes: int = 256 << 20, wait: bool = True):
    """Device -> host copies of (host, device) tensor pairs, split into row
    chunks over several copy streams: one stream reaches ~51 GB/s on the B200
    boxes' PCIe link, four ~56 GB/s (tools/d2h_probe.py).  Ordered after the
    current stream's work; returns when every chunk has landed -- or, with
    wait=False, at once, returning the function that waits for them (the
    caller overlaps its status readback with the transfer)."""
    t = torch()
    cur = t.cuda.current_stream()
    dev = cur.device
    pool = _copy_streams.get(dev)
    if pool is None:
        pool = _copy_streams[dev] = [t.cuda.Stream(device=dev) for _ in range(streams)]
    ready = t.cuda.Event()
    ready.record(cur)
    for st in pool:
        st.wait_event(ready)
    k = 0
    for host, src in pairs:
        rows = max(1, chunk_bytes // max(1, src[0].numel() * src.element_size())) if src.dim() > 1 else src.numel()
        for r0 in range(0, src.shape[0], rows):
            with t.cuda.stream(pool[k % len(pool)]):
                host[r0:r0 + rows].copy_(src[r0:r0 + rows], non_blocking=True)
            k += 1

    def done():
        for st in pool:
            st.synchronize()
    if wait:
        done()
        return None
    return done


def sync():
    torch().cuda.current_stream().synchronize()
