"""Correlation-result serialization drop-in (reference: dataset.py:34-36,
:292-341, :480-504).

Byte-for-byte the reference's files: the metadata header lines, then every
value as ``repr(float(x))`` -- the shortest decimal that round-trips to the
same float64.  The O(n1 n2) table is formatted by native host code in
libcorr2d.so (``corr2d_format_rows``: std::to_chars shortest digits laid out
with CPython's repr rules, several threads) instead of one Python call per
value; ``save_correlation`` streams row blocks to the files, so memory stays
bounded for maps of any size.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from . import _abi
from .errors import DataError

MATRIX_PAIR = "matrix-pair"
LONG_FORM = "long-form"
_BLOCK_BYTES = 64 << 20          # target text per native call


def format_number(x: float) -> str:
    """Shortest decimal string that round-trips to the same float64 (dataset.py:34-36)."""
    return repr(float(x))


def _threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _meta_lines(result, fmt: str, section: str) -> list[str]:
    return [
        f"# corrtwo-correlation format={fmt} section={section}",
        f"# engine={result.engine} normalization={format_number(result.normalization)} "
        f"scaling_exponent={format_number(result.scaling_exponent)} "
        f"is_homo={'true' if result.is_homo else 'false'}",
        "# ref1=" + ",".join(format_number(v) for v in np.asarray(result.ref1)),
        "# ref2=" + ",".join(format_number(v) for v in np.asarray(result.ref2)),
    ]


def _plane(a):
    a = np.asarray(a)
    if a.dtype not in (np.float64, np.float32):
        a = a.astype(np.float64)
    if a.strides[1] != a.itemsize:
        a = np.ascontiguousarray(a)
    return a, (_abi.F32 if a.dtype == np.float32 else _abi.F64)


def _table_blocks(result, matrix, matrix2, delimiter: str, long_form: bool):
    """Yield the table text in row blocks (bytes)."""
    lib = _abi.load()
    if len(delimiter.encode()) != 1:
        raise DataError(f"delimiter must be one byte, got {delimiter!r}")
    ax1 = np.ascontiguousarray(result.axis1, dtype=np.float64)
    ax2 = np.ascontiguousarray(result.axis2, dtype=np.float64)
    m1, dt = _plane(matrix)
    m2 = None
    if long_form:
        m2, dt2 = _plane(matrix2)
        if dt2 != dt or m2.strides != m1.strides:
            m1, m2 = np.ascontiguousarray(m1, np.float64), np.ascontiguousarray(m2, np.float64)
            dt = _abi.F64
    n1, n2 = m1.shape
    ld = m1.strides[0] // m1.itemsize
    per_row = (n2 + 1) * 25 if not long_form else n2 * 100
    rows = max(1, _BLOCK_BYTES // per_row)
    threads = _threads()
    written = ctypes.c_int64(0)
    buf = np.empty(0, dtype=np.uint8)      # reused across blocks, never zero-filled
    for r0 in range(0, n1, rows):
        r1 = min(n1, r0 + rows)
        cap = (r1 - r0) * per_row + 64
        while True:
            if buf.size < cap:
                buf = np.empty(cap, dtype=np.uint8)
            code = lib.corr2d_format_rows(dt, ax1.ctypes.data, ax2.ctypes.data, m1.ctypes.data,
                                          None if m2 is None else m2.ctypes.data, ld, n2, r0, r1,
                                          delimiter.encode(), 1 if long_form else 0, threads, buf.ctypes.data,
                                          buf.size, ctypes.byref(written))
            if code == 0:
                break
            if written.value <= buf.size:
                _abi.check(code, lib)
            cap = written.value
        yield memoryview(buf)[:written.value]


def _payload_parts(result, fmt: str, delimiter: str):
    """{suffix: iterator of byte chunks} of write_correlation (dataset.py:311-341)."""
    if fmt == MATRIX_PAIR:
        out = {}
        for section, matrix in (("sync", result.sync), ("async", result.asyn)):
            head = _meta_lines(result, fmt, section)
            head.append(delimiter.join([""] + [format_number(v) for v in np.asarray(result.axis2)]))

            def gen(head=head, matrix=matrix):
                yield ("\n".join(head) + "\n").encode("utf-8")
                yield from _table_blocks(result, matrix, None, delimiter, False)
            out[f"{section}.csv"] = gen()
        return out
    if fmt == LONG_FORM:
        head = _meta_lines(result, fmt, "long") + ["nu1,nu2,sync,async"]

        def gen():
            yield ("\n".join(head) + "\n").encode("utf-8")
            yield from _table_blocks(result, result.sync, result.asyn, ",", True)
        return {"corr.csv": gen()}
    raise DataError(f"unknown correlation format {fmt!r}")


def write_correlation(result, fmt: str = MATRIX_PAIR, delimiter: str = ",") -> dict[str, bytes]:
    """Serialize a correlation result: ``{"sync.csv", "async.csv"}`` payloads
    (matrix-pair) or ``{"corr.csv"}`` (long-form), as dataset.py:311-341."""
    return {k: b"".join(bytes(c) for c in v) for k, v in _payload_parts(result, fmt, delimiter).items()}


def correlation_paths(stem, fmt: str = MATRIX_PAIR) -> dict[str, Path]:
    """dataset.py:480-489."""
    stem = Path(stem)
    if fmt == MATRIX_PAIR:
        return {"sync.csv": stem.with_name(stem.name + ".sync.csv"),
                "async.csv": stem.with_name(stem.name + ".async.csv")}
    if fmt == LONG_FORM:
        return {"corr.csv": stem.with_name(stem.name + ".corr.csv")}
    raise DataError(f"unknown correlation format {fmt!r}")


def save_correlation(result, stem, fmt: str = MATRIX_PAIR, delimiter: str = ",") -> list[Path]:
    """Write the files of ``write_correlation`` (dataset.py:492-504), streaming
    row blocks so the text never has to fit in memory at once."""
    parts = _payload_parts(result, fmt, delimiter)
    paths = correlation_paths(stem, fmt)
    written = []
    for key, chunks in parts.items():
        try:
            with open(paths[key], "wb") as fh:
                for c in chunks:
                    fh.write(c)
        except OSError as exc:
            raise DataError(f"cannot write {paths[key]}: {exc}") from None
        written.append(paths[key])
    return written
