"""The C-ABI library: loads on a CPU-only host, exports every symbol
include/corr2d.h declares, host-only helpers work, and compute entry points
fail loudly (no CPU fallback) when no GPU is present."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_1808_00685_b200 import _abi

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "corr2d.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(corr2d_\w+)\(", text, re.M)))


def test_header_declares_abi_exports():
    assert set(declared_symbols()) == set(_abi.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_has_no_torch_dependency():
    out = subprocess.run(["ldd", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "torch" not in out and "c10" not in out


def test_sm100a_cubin_present():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_helpers():
    lib = _abi.load()
    assert lib.corr2d_abi_version() == 3
    assert lib.corr2d_packed_depth(11, _abi.PACK_F64) == 12
    assert lib.corr2d_packed_depth(64, _abi.PACK_F64) == 64
    assert lib.corr2d_packed_depth(512, _abi.PACK_BF16X2) == 768   # [Re' | Im' | -Im'], 256 each
    assert lib.corr2d_packed_depth(37, _abi.PACK_BF16X2) == 96
    assert lib.corr2d_packed_depth(512, _abi.PACK_F16F8) == 768     # same slots, fp16 + e4m3 bytes
    # tile enumerations: fp64 64-tiles upper triangle; bf16 whole map = CTA-pair tiles
    assert lib.corr2d_contract_tile_count(_abi.PACK_F64, 16384, 16384, 1, 0, 16384, 16384) == 256 * 257 // 2
    T, P = 256, 128
    assert lib.corr2d_contract_tile_count(_abi.PACK_BF16X2, 32768, 32768, 1, 0, 32768, 32768) == P * T - P * (P - 1)
    assert lib.corr2d_contract_tile_count(_abi.PACK_BF16X2, 32768, 32768, 1, 0, 16384, 32768) == 128 * 256 - 128 * 127 // 2
    assert lib.corr2d_contract_tile_count(_abi.PACK_F16F8, 32768, 32768, 1, 0, 32768, 32768) == P * T - P * (P - 1)
    buf = (ctypes.c_int * 24)()
    k = lib.corr2d_fft_factors(512, buf, 24)
    assert list(buf[:k]) == [8, 8, 8]
    k = lib.corr2d_fft_factors(1000, buf, 24)
    assert sorted(buf[:k]) == [5, 5, 5, 8]
    k = lib.corr2d_fft_factors(509, buf, 24)
    assert list(buf[:k]) == [509]


def test_argument_errors_map_to_data_error():
    lib = _abi.load()
    code = lib.corr2d_contract_f64(None, None, None, 0, 1, 1, 4, 0, 0, 1, 0, -1, None, None, 1, None, None)
    assert code == _abi.ERR_DATA
    with pytest.raises(_abi.DataError, match="null pointer"):
        _abi.check(code, lib)


def test_gpu_entry_points_fail_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np
    import paper_1808_00685_b200 as P
    dyn = P.DynamicSpectra(np.arange(4.0), np.arange(6.0), np.ones((6, 4)), np.zeros(4))
    with pytest.raises(_abi.BackendUnavailable):
        P.correlate_ft(dyn)
    lib = _abi.load()
    sms = ctypes.c_int()
    assert lib.corr2d_device_info(0, ctypes.byref(sms), None, None) == _abi.ERR_CUDA


def _small_decode(b, T, I0, I1, homo, T2=None):
    """Python restatement of fused_decode (csrc/small.cu) -- the 32 x 32 tile
    enumeration of a row shard [I0, I1) that the one-kernel small-m path and the
    multi-GPU tile ranges index."""
    if not homo:
        return I0 + b // T2, b % T2, "plain"
    d = 0
    S = lambda dd: dd * T - dd * (dd - 1) // 2
    while S(d + 1) <= b:
        d += 1
    I = I0 + d
    o = b - S(d)
    if o < I0:
        return o, I, "trans"
    J = I + (o - I0)
    return I, J, ("diag" if J == I else ("mirror" if J < I1 else "plain"))


@pytest.mark.parametrize("n,rows", [(1000, (0, 1000)), (517, (0, 517)), (517, (64, 320)), (33, (0, 33)),
                                    (700, (32, 96)), (700, (640, 700))])
def test_small_path_tile_enumeration_covers_each_output_tile_once(n, rows):
    """corr2d_small_tile_count (host code, no GPU needed) matches the enumeration,
    and the enumeration writes every 32 x 32 output tile of the shard exactly
    once (homo: direct, mirrored or transposed), the property behind the
    bit-identity of row shards and tile-range partitions."""
    lib = _abi.load()
    r0, r1 = rows
    T = (n + 31) // 32
    I0, I1 = r0 // 32, (r1 + 31) // 32
    for homo in (1, 0):
        n2 = n if homo else n - 7
        T2 = (n2 + 31) // 32
        count = lib.corr2d_small_tile_count(n, n2, homo, r0, r1)
        R = I1 - I0
        assert count == (R * T - R * (R - 1) // 2 if homo else R * T2)
        written = {}
        for b in range(count):
            I, J, mode = _small_decode(b, T, I0, I1, homo, T2)
            targets = []
            if mode in ("plain", "mirror", "diag"):
                targets.append((I, J))
            if mode in ("mirror", "trans"):
                targets.append((J, I))
            for t in targets:
                if I0 <= t[0] < I1:
                    written[t] = written.get(t, 0) + 1
        want = {(i, j) for i in range(I0, I1) for j in range(T if homo else T2)}
        assert set(written) == want and all(v == 1 for v in written.values())


def test_small_path_depth_and_bad_arguments():
    lib = _abi.load()
    assert [lib.corr2d_small_depth(m) for m in (2, 8, 11, 21, 32)] == [8, 8, 16, 24, 32]
    assert lib.corr2d_small_depth(1) < 0 and lib.corr2d_small_depth(33) < 0
    assert lib.corr2d_small_tile_count(10, 12, 1, 0, 10) < 0       # homo needs n1 == n2
    assert lib.corr2d_small_tile_count(64, 64, 1, 0, 65) < 0       # rows past n1
