"""ctypes binding of libcorr2d.so (C ABI declared in include/corr2d.h).

The library is loaded lazily on first use.  There is no CPU fallback: if the
shared object is missing or no CUDA device is visible, every GPU entry point
raises :class:`BackendUnavailable` with the reason.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import DataError, NumericError

LIB_PATH = Path(__file__).resolve().parent / "libcorr2d.so"

OK, ERR_DATA, ERR_NUMERIC, ERR_OOM, ERR_CUDA, ERR_UNSUPPORTED = range(6)
F64, F32 = 0, 1
RESAMPLE_NONE, RESAMPLE_LINEAR, RESAMPLE_MATRIX = 0, 1, 2
PACK_NONE, PACK_F64, PACK_BF16X2, PACK_F64_TIME, PACK_F16F8, PACK_F64_GAUSS = 0, 1, 2, 3, 4, 5
ROLE_A, ROLE_B = 1, 2
REF_MEAN, REF_PROVIDED, REF_NONE = 0, 1, 2
ST_NONFINITE, ST_ZEROVAR, ST_FIRST_ZEROVAR = 0, 1, 2
INT32_MAX = 2**31 - 1

# every symbol include/corr2d.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "corr2d_last_error", "corr2d_abi_version", "corr2d_device_info", "corr2d_packed_depth",
    "corr2d_fft_factors", "corr2d_prep", "corr2d_contract_f64", "corr2d_contract_f64_gauss", "corr2d_contract_bf16x3",
    "corr2d_contract_tc", "corr2d_contract_tile_count", "corr2d_plane_absmax", "corr2d_find_peaks",
    "corr2d_fetch_mirrored",
    "corr2d_format_repr", "corr2d_format_rows", "corr2d_small_block_count", "corr2d_small_launches", "corr2d_small_ops_depth",
    "corr2d_correlate_small_f64", "corr2d_correlate_small_f64_slot",
)


class BackendUnavailable(RuntimeError):
    """libcorr2d.so is not built / not loadable, or no CUDA device."""


_lock = threading.Lock()
_lib = None

c_int, c_i64, c_double, c_void = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


def _declare(lib):
    lib.corr2d_last_error.restype = ctypes.c_char_p
    lib.corr2d_last_error.argtypes = []
    lib.corr2d_abi_version.restype = c_int
    lib.corr2d_device_info.argtypes = [c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int), ctypes.POINTER(c_int)]
    lib.corr2d_packed_depth.argtypes = [c_int, c_int]
    lib.corr2d_fft_factors.argtypes = [c_int, ctypes.POINTER(c_int), c_int]
    lib.corr2d_prep.argtypes = [
        c_int, c_void, c_i64, c_int, c_int,          # in_dtype raw ld_raw m_in n
        c_int, c_void, c_void, c_void, c_int,        # resample idx frac matrix m
        c_int, c_void, c_void, c_double, c_int,      # ref_mode ref_in sigma_in alpha substitute
        c_double, c_int, c_int,                      # norm pack_kind roles
        c_void, c_void, c_void, c_i64, c_i64,        # a_phi a_psi b ld_pack split_plane
        c_void, c_i64, c_void,                       # values ld_values half
        c_void, c_void, c_void, c_void,              # ref_out sigma_out status stream
    ]
    lib.corr2d_contract_f64.argtypes = [
        c_void, c_void, c_void, c_i64, c_int, c_int, c_int, c_int, c_int, c_int, c_i64, c_i64,
        c_void, c_void, c_i64, c_void, c_void,
    ]
    lib.corr2d_contract_f64_gauss.argtypes = [
        c_void, c_void, c_i64, c_int, c_int, c_int, c_int, c_int, c_int, c_i64, c_i64,
        c_void, c_void, c_i64, c_void, c_void,
    ]
    lib.corr2d_contract_bf16x3.argtypes = [
        c_void, c_void, c_i64, c_i64, c_i64, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
        c_i64, c_i64, c_void, c_void, c_i64, c_void, c_void,
    ]
    lib.corr2d_contract_tc.argtypes = [
        c_int, c_void, c_void, c_i64, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
        c_i64, c_i64, c_void, c_void, c_i64, c_void, c_void,
    ]
    lib.corr2d_contract_tile_count.argtypes = [c_int, c_int, c_int, c_int, c_int, c_int, c_i64]
    lib.corr2d_contract_tile_count.restype = c_i64
    lib.corr2d_plane_absmax.argtypes = [c_int, c_void, c_i64, c_int, c_int, c_void, c_void]
    lib.corr2d_fetch_mirrored.argtypes = [c_int, c_void, c_void, c_i64, c_int, c_void, c_void, c_i64, c_int, c_int,
                                          c_int, c_void, c_void]
    lib.corr2d_find_peaks.argtypes = [c_int, c_void, c_void, c_i64, c_int, c_int, c_int, c_double, c_double,
                                      c_void, c_i64, c_void, c_void]
    lib.corr2d_format_repr.argtypes = [c_void, c_i64, c_void, c_i64, c_void]
    lib.corr2d_format_rows.argtypes = [c_int, c_void, c_void, c_void, c_void, c_i64, c_int, c_int, c_int,
                                       ctypes.c_char, c_int, c_int, c_void, c_i64, c_void]
    lib.corr2d_small_block_count.argtypes = [c_int, c_int, c_int]
    lib.corr2d_small_block_count.restype = c_i64
    lib.corr2d_small_launches.argtypes = [c_int, c_int, c_int]
    lib.corr2d_small_launches.restype = c_int
    lib.corr2d_small_ops_depth.argtypes = [c_int]
    lib.corr2d_correlate_small_f64.argtypes = [
        c_int, c_void, c_i64, c_void, c_i64,          # in_dtype raw1 ld_raw1 raw2 ld_raw2
        c_int, c_int, c_int,                          # m n1 n2
        c_int, c_void, c_void, c_int, c_void, c_void,  # ref_mode1 ref_in1 sigma_in1, same for dataset 2
        c_double, c_int, c_double,                    # alpha substitute norm
        c_void, c_void, c_i64,                        # ops_a ops_b ld_ops
        c_void, c_void, c_void, c_void,               # ref_out1 sigma_out1 ref_out2 sigma_out2
        c_void, c_void, c_i64,                        # phi psi ld_out
        c_void, c_void, c_void, c_void, c_void,       # status1 status2 stats work stream
    ]
    lib.corr2d_correlate_small_f64_slot.argtypes = list(lib.corr2d_correlate_small_f64.argtypes) + [
        c_int, c_void,                                # slot pipe
    ]
    for name in ("corr2d_format_repr", "corr2d_format_rows", "corr2d_correlate_small_f64",
                 "corr2d_correlate_small_f64_slot", "corr2d_small_ops_depth",
                 "corr2d_prep", "corr2d_contract_f64", "corr2d_contract_f64_gauss", "corr2d_contract_bf16x3",
                 "corr2d_contract_tc", "corr2d_device_info", "corr2d_packed_depth", "corr2d_fft_factors",
                 "corr2d_plane_absmax", "corr2d_find_peaks", "corr2d_fetch_mirrored"):
        getattr(lib, name).restype = c_int


def load(path: Path | None = None):
    """Load (once) and return the ctypes library handle."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # CORR2D_LIB: load an alternative build (experiments only)
        p = Path(path) if path else Path(os.environ.get("CORR2D_LIB", LIB_PATH))
        if not p.exists():
            raise BackendUnavailable(
                f"{p} is not built; run `python -m paper_1808_00685_b200.build` "
                "(the GPU path has no CPU fallback)")
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as e:  # pragma: no cover
            raise BackendUnavailable(f"cannot load {p}: {e}") from None
        _declare(lib)
        if path is None:
            _lib = lib
        return lib


def last_error(lib=None) -> str:
    lib = lib or load()
    msg = lib.corr2d_last_error()
    return msg.decode() if msg else ""


def check(code: int, lib=None):
    if code == OK:
        return
    msg = last_error(lib)
    if code == ERR_DATA:
        raise DataError(msg)
    if code in (ERR_NUMERIC, ERR_OOM):
        raise NumericError(msg)
    if code == ERR_UNSUPPORTED:
        raise DataError(f"unsupported by the GPU path: {msg}")
    raise RuntimeError(f"CUDA failure in libcorr2d: {msg}")
