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


def _small_decode(b, T1, T2, homo):
    """Python restatement of small_decode (csrc/small.cu): block b of the
    one-kernel small-m path -> (row block I, column block J); homo: the upper
    triangle row by row."""
    if not homo:
        return b // T2, b % T2
    d = 0
    S = lambda dd: dd * T1 - dd * (dd - 1) // 2
    while S(d + 1) <= b:
        d += 1
    return d, d + (b - S(d))


@pytest.mark.parametrize("n", [1000, 517, 64, 33, 2000])
def test_small_path_blocks_cover_the_map_once(n):
    """corr2d_small_block_count (host code, no GPU needed) matches the
    enumeration, and every 64 x 64 output block is written exactly once
    (homo: directly or as the mirror of an upper block)."""
    lib = _abi.load()
    for homo in (1, 0):
        n2 = n if homo else max(1, n - 77)
        T1, T2 = (n + 63) // 64, (n2 + 63) // 64
        count = lib.corr2d_small_block_count(n, n2, homo)
        assert count == (T1 * (T1 + 1) // 2 if homo else T1 * T2)
        written = {}
        for b in range(count):
            I, J = _small_decode(b, T1, T2, homo)
            targets = [(I, J)] + ([(J, I)] if homo and J != I else [])
            for t in targets:
                written[t] = written.get(t, 0) + 1
        want = {(i, j) for i in range(T1) for j in range(T2)}
        assert set(written) == want and all(v == 1 for v in written.values())


def test_small_path_bad_arguments():
    lib = _abi.load()
    assert lib.corr2d_small_block_count(10, 12, 1) < 0        # homo needs n1 == n2
    assert lib.corr2d_small_block_count(0, 12, 0) < 0
