"""Result serialization: native shortest round-trip
formatting against Python's repr, and write_correlation / save_correlation
byte-for-byte against the reference's own payloads (tests/golden/ser_*.npz).
Host code only -- runs without a GPU."""

import ctypes

import numpy as np
import pytest

from conftest import golden, golden_names
import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import _abi
from paper_1808_00685_b200.serialize import (LONG_FORM, MATRIX_PAIR, correlation_paths, format_number,
                                             save_correlation, write_correlation)


def _repr_native(xs):
    lib = _abi.load()
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    n = xs.size
    out = ctypes.create_string_buffer(max(1, n) * 32)
    offs = np.zeros(n + 1, dtype=np.int64)
    assert lib.corr2d_format_repr(xs.ctypes.data, n, out, n * 32, offs.ctypes.data) == 0
    raw = out.raw
    return [raw[offs[i]:offs[i + 1]].decode() for i in range(n)]


def test_native_repr_matches_python_repr():
    rng = np.random.default_rng(11)
    bits = np.frombuffer(rng.integers(0, 2**63, 60000, dtype=np.uint64).tobytes(), dtype=np.float64)
    special = np.array([0.0, -0.0, 1e16, 1e15, 9.999999999999999e15, 0.0001, 0.00001, 1e-4, 5e-324,
                        2.0**-1074 * 3, 1.7976931348623157e308, 2.0**53, 1e22, 123.0, 0.1, 1 / 3,
                        np.inf, -np.inf, np.nan, -1e-7, 1234567.0, 1e100, -2.5e-300])
    xs = np.concatenate([rng.standard_normal(40000), rng.uniform(-1e20, 1e20, 20000), bits, special,
                         rng.integers(-10**12, 10**12, 20000).astype(float),
                         (rng.standard_normal(20000) * 1e-5).astype(np.float32).astype(np.float64)])
    got = _repr_native(xs)
    want = [repr(float(x)) for x in xs]
    bad = [(w, g) for w, g in zip(want, got) if w != g]
    assert not bad, bad[:5]
    assert format_number(np.float32(0.1)) == "0.10000000149011612"


def _result_for(g):
    src = golden(str(g["src"]))
    n1, n2 = src["sync"].shape
    homo = "nu" in src
    ax1 = src["nu"] if homo else src["nu1"]
    ax2 = src["nu"] if homo else src["nu2"]
    return P.CorrelationSpectra(axis1=ax1, axis2=ax2, sync=src["sync"], asyn=src["asyn"], ref1=g["ref1"],
                                ref2=g["ref2"], normalization=float(src["norm"]), engine="fourier",
                                is_homo=homo, scaling_exponent=0.0)


@pytest.mark.parametrize("name", golden_names("ser_"))
def test_write_correlation_bytes_match_reference(name, tmp_path):
    g = golden(name)
    res = _result_for(g)
    fmt, delim = str(g["fmt"]), str(g["delim"])
    payload = write_correlation(res, fmt, delim)
    keys = ["sync.csv", "async.csv"] if fmt == MATRIX_PAIR else ["corr.csv"]
    assert sorted(payload) == sorted(keys)
    for k in keys:
        assert payload[k] == g[k.replace(".", "_")].tobytes(), k
    paths = save_correlation(res, tmp_path / "out", fmt, delim)
    assert [p.name for p in paths] == [correlation_paths(tmp_path / "out", fmt)[k].name for k in keys]
    for k, p in zip(keys, paths):
        assert p.read_bytes() == g[k.replace(".", "_")].tobytes()


def test_streamed_blocks_and_float32_round_trip(tmp_path, monkeypatch):
    """Multi-block streaming (tiny block size) gives the same bytes; float32
    planes serialize as repr of their float64 value and parse back exactly."""
    import paper_1808_00685_b200.serialize as S
    rng = np.random.default_rng(5)
    n1, n2 = 37, 23
    s = rng.standard_normal((n1, n2)).astype(np.float32)
    a = rng.standard_normal((n1, n2)).astype(np.float32)
    res = P.CorrelationSpectra(axis1=np.linspace(1, 2, n1), axis2=np.linspace(3, 4, n2), sync=s, asyn=a,
                               ref1=np.zeros(n1), ref2=np.zeros(n2), normalization=0.5, engine="fourier",
                               is_homo=False, scaling_exponent=0.0)
    whole = write_correlation(res, LONG_FORM)
    monkeypatch.setattr(S, "_BLOCK_BYTES", 1)
    assert write_correlation(res, LONG_FORM) == whole
    lines = whole["corr.csv"].decode().splitlines()
    body = [l for l in lines if l and not l.startswith("#")][1:]
    vals = np.array([[float(x) for x in l.split(",")] for l in body])
    assert np.array_equal(vals[:, 2].reshape(n1, n2), np.asarray(res.sync, dtype=np.float64))
    assert np.array_equal(vals[:, 3].reshape(n1, n2), np.asarray(res.asyn, dtype=np.float64))
    with pytest.raises(P.DataError):
        write_correlation(res, "xml")
