"""Homo-map device -> host transfer that sends the upper triangle only
(corr2d_fetch_mirrored, csrc/fetch.cu): the host planes must equal a
full-plane copy bit for bit -- on exactly (anti)symmetric synthetic planes of
ragged sizes and host fill shares, and on maps the contractions wrote (fp64,
fp32 tcgen05) through the public corr2d() call against the full copy."""

import numpy as np
import pytest

import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import _abi, engine

pytestmark = pytest.mark.gpu


def _planes(n, dtype, seed=0):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn((n, n), generator=g, device="cuda", dtype=dtype)
    b = torch.randn((n, n), generator=g, device="cuda", dtype=dtype)
    return (a + a.T).contiguous(), (b - b.T).contiguous()


def _bits(x):
    x = np.asarray(x)
    return x.view(np.uint64 if x.dtype == np.float64 else np.uint32)


@pytest.mark.parametrize("n,band,fill,threads", [(4096, 1024, 100, 8), (5000, 1024, 45, 3), (1300, 256, 100, 1),
                                                  (1300, 256, 0, 2), (2304, 512, 37, 16), (257, 512, 100, 4)])
@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_mirrored_fetch_bit_identical(n, band, fill, threads, dt):
    import torch
    dtype = getattr(torch, dt)
    phi, psi = _planes(n, dtype, seed=n)
    hs = torch.full((n, n), float("nan"), dtype=dtype).pin_memory()
    ha = torch.full((n, n), float("nan"), dtype=dtype).pin_memory()
    engine.fetch_mirrored(_abi.load(), phi, psi, hs, ha, band=band, fill_pct=fill, threads=threads)
    assert np.array_equal(_bits(hs.numpy()), _bits(phi.cpu().numpy()))
    assert np.array_equal(_bits(ha.numpy()), _bits(psi.cpu().numpy()))
    nb = (n + band - 1) // band
    split = [(b * band * fill // 100) // 64 * 64 for b in range(nb)]
    sent = sum(2 * (min(n, b * band + band) - b * band) * (n - split[b]) for b in range(nb)) * hs.element_size()
    assert engine.last_fetch_bytes == sent
    if fill == 100 and n >= 4096:
        assert sent <= (1 + 1 / nb) / 2 * 2 * n * n * hs.element_size()


def test_mirrored_fetch_async_and_pageable_host():
    import torch
    phi, psi = _planes(2048, torch.float64, seed=7)
    hs = np.empty((2048, 2048))
    ha = np.empty((2048, 2048))
    done = engine.fetch_mirrored(_abi.load(), phi, psi, torch.from_numpy(hs), torch.from_numpy(ha), wait=False)
    done()
    assert np.array_equal(_bits(hs), _bits(phi.cpu().numpy()))
    assert np.array_equal(_bits(ha), _bits(psi.cpu().numpy()))


def test_mirrored_fetch_bad_arguments():
    import torch
    phi, psi = _planes(512, torch.float32)
    hs = torch.empty((512, 512)).pin_memory()
    ha = torch.empty((512, 512)).pin_memory()
    with pytest.raises(P.DataError, match="multiple of 256"):
        engine.fetch_mirrored(_abi.load(), phi, psi, hs, ha, band=100)
    with pytest.raises(P.DataError, match="multiple of 256"):
        engine.fetch_mirrored(_abi.load(), phi, psi, hs, ha, band=100, wait=False)()
    with pytest.raises(P.DataError, match="fill_pct"):
        engine.fetch_mirrored(_abi.load(), phi, psi, hs, ha, fill_pct=101)


@pytest.mark.parametrize("dt,m,n", [("float64", 24, 4352), ("float32", 64, 5120), ("float32", 32, 16384)])
def test_public_call_mirrored_equals_full_copy(monkeypatch, dt, m, n):
    rng = np.random.default_rng(m)
    x = rng.standard_normal((m, n)).cumsum(axis=1)
    ds = P.SpectralDataset(np.linspace(0.0, 1.0, n), np.arange(m, dtype=float), x,
                           dtype=np.float32 if dt == "float32" else np.float64)
    monkeypatch.setattr(engine, "MIRROR_FILL_PCT", 0)
    full = P.corr2d(ds, dtype=dt)      # the full-plane copy
    assert engine.last_fetch_bytes == 2 * n * n * full.sync.itemsize
    monkeypatch.setattr(engine, "MIRROR_FILL_PCT", 45)
    monkeypatch.setattr(engine, "MIRROR_MIN_N", 4096)
    half = P.corr2d(ds, dtype=dt)
    assert engine.last_fetch_bytes < 2 * n * n * full.sync.itemsize
    assert np.array_equal(_bits(half.sync), _bits(full.sync))
    assert np.array_equal(_bits(half.asyn), _bits(full.asyn))
