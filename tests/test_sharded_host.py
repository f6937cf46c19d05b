"""Host logic of the multi-GPU band ownership (paper_1808_00685_b200/sharded.py,
SURVEY.md 8e) on the CPU: the band partition, the per-rank contraction pieces,
the host assembly of the map from bands (mirror included), and the gloo
collectives of the spectra exchange and of ``gather`` at world size 2 and 3
(127.0.0.1).  Bands are produced by the CPU oracle here; the GPU tests run the
same code over the kernels (tests/test_gpu_sharded.py)."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import corr2d_oracle as O
from paper_1808_00685_b200.engine_core import BAND_UNIT, assemble_bands, band_partition, band_pieces

ROOT = Path(__file__).resolve().parent.parent


def _area(band, n):
    r0, r1 = band
    return sum(n - r for r in range(r0, r1))


@pytest.mark.parametrize("n", [32768, 16384, 8192, 1000, 300])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("homo", [True, False])
def test_band_partition_covers_rows_in_order(n, world, homo):
    bands = band_partition(n, world, homo)
    assert len(bands) == world
    assert bands[0][0] == 0 and bands[-1][1] == n
    for (a0, a1), (b0, b1) in zip(bands[:-1], bands[1:]):
        assert a1 == b0 and a0 <= a1
    for r0, r1 in bands:
        assert r0 % BAND_UNIT == 0 and (r1 % BAND_UNIT == 0 or r1 == n)


@pytest.mark.parametrize("n,world,slack", [(32768, 8, 1.04), (32768, 2, 1.01), (16384, 8, 1.04), (16384, 4, 1.025)])
def test_homo_bands_balanced_by_upper_triangle_area(n, world, slack):
    bands = band_partition(n, world, True)
    areas = [_area(b, n) for b in bands]
    assert sum(areas) == n * (n + 1) // 2
    assert max(areas) <= slack * sum(areas) / world
    # the bands thicken towards the bottom of the map
    widths = [r1 - r0 for r0, r1 in bands]
    assert widths == sorted(widths)


def test_band_memory_scales_as_one_over_world():
    n = 32768
    full = n * n
    for world in (2, 4, 8):
        per_rank = max((r1 - r0) * (n - r0) for r0, r1 in band_partition(n, world, True))
        assert per_rank <= 1.25 * full / world


@pytest.mark.parametrize("n1,n2,world", [(1000, 1000, 3), (2000, 1500, 3), (777, 777, 8), (4096, 4096, 4)])
def test_pieces_write_every_owned_element_once(n1, n2, world):
    homo = n1 == n2
    bands = band_partition(n1, world, homo)
    cols = None if homo else band_partition(n2, world, False)
    cover = np.zeros((n1, n2), dtype=np.int32)
    for rank in range(world):
        r0, r1 = bands[rank]
        for kind, owner, c0, c1 in band_pieces(bands, rank, homo, cols):
            if kind == "diag":
                assert owner == rank and (c0, c1) == (r0, r1)
                cover[r0:r1, c0:c1] += 1               # the square, both triangles (mirrored in-band)
            else:
                assert owner != rank or not homo
                cover[r0:r1, c0:c1] += 1
        if homo and r1 > r0:
            cover[r1:, r0:r1] += 1                     # implied mirror of the band's rectangle
    assert np.all(cover == 1)


def test_homo_pieces_wait_only_for_later_owners():
    bands = band_partition(32768, 8, True)
    for rank in range(8):
        pieces = band_pieces(bands, rank, True)
        assert pieces[0][0] == "diag"
        assert [p[1] for p in pieces[1:]] == list(range(rank + 1, 8))


def _oracle_bands(v1, v2, bands, homo):
    s, a, _ = O.correlate_ft(v1, None if homo else v2)
    out = []
    for r0, r1 in bands:
        c0 = r0 if homo else 0
        out.append((r0, r1, c0, s[r0:r1, c0:].copy(), a[r0:r1, c0:].copy()))
    return s, a, out


@pytest.mark.parametrize("homo", [True, False])
@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_assemble_bands_reproduces_the_map(homo, world):
    rng = np.random.default_rng(world)
    v1 = rng.normal(size=(12, 700))
    v2 = rng.normal(size=(12, 450))
    n1, n2 = 700, (700 if homo else 450)
    bands = band_partition(n1, world, homo)
    s, a, parts = _oracle_bands(v1, v2, bands, homo)
    gs, ga = assemble_bands(n1, n2, homo, parts)
    if homo:
        # the oracle map is symmetric only to rounding; the assembled one is
        # exactly symmetric, with the upper triangle the oracle's
        iu = np.triu_indices(n1)
        assert np.array_equal(gs[iu], s[iu]) and np.array_equal(ga[iu], a[iu])
        assert np.array_equal(gs, gs.T) and np.array_equal(ga, -ga.T)
    else:
        assert np.array_equal(gs, s) and np.array_equal(ga, a)


# ------------------------------------------------------------------ gloo ranks

def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, homo, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, str(ROOT))
        from paper_1808_00685_b200 import sharded
        n = 600
        bands = band_partition(n, world, homo)
        # spectra exchange: each owner fills its chunk, the broadcasts complete the buffer
        buf = torch.zeros((n, 5), dtype=torch.float64)
        r0, r1 = bands[rank]
        buf[r0:r1] = torch.arange(r0, r1, dtype=torch.float64)[:, None] + 0.25 * torch.arange(5)
        for owner, (q0, q1) in enumerate(bands):
            assert sharded._broadcast(buf[q0:q1], owner, None) is None     # gloo: synchronous
        want = torch.arange(n, dtype=torch.float64)[:, None] + 0.25 * torch.arange(5)
        exchange_ok = bool(torch.equal(buf, want))
        # gather: bands from the oracle, assembled on rank 0 through the real gather()
        rng = np.random.default_rng(11)
        v1 = rng.normal(size=(9, n))
        v2 = rng.normal(size=(9, 410))
        n2 = n if homo else 410
        s, a, parts = _oracle_bands(v1, v2, bands, homo)
        _, _, c0, bs, ba = parts[rank]

        class _Plan:            # the attributes gather() reads from a ShardedCorrelationPlan
            pass
        pl = _Plan()
        pl.group, pl.global_ranks, pl.n1, pl.n2 = None, list(range(world)), n, n2
        pl.dtype, pl.homo, pl.dev = np.dtype(np.float64), homo, torch.device("cpu")
        pl.phi, pl.psi = torch.from_numpy(bs), torch.from_numpy(ba)
        pl.r0, pl.r1, pl.c0, pl.rank, pl.world, pl.bands = r0, r1, c0, rank, world, bands
        meta = dict(axis1=np.arange(n, dtype=float), axis2=np.arange(n2, dtype=float), ref1=np.zeros(n),
                    ref2=np.zeros(n2), normalization=1.0, engine="fourier", is_homo=homo,
                    scaling_exponent=0.0)
        res = sharded.ShardedCorrelationSpectra(pl, meta).gather(root=0)
        if rank == 0:
            ref_s, ref_a = assemble_bands(n, n2, homo, parts)
            q.put((exchange_ok, bool(np.array_equal(res.sync, ref_s) and np.array_equal(res.asyn, ref_a)),
                   res.is_homo))
        else:
            q.put((exchange_ok, res is None, homo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("homo", [True, False])
def test_gloo_spectra_exchange_and_gather(world, homo):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, homo, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for exchange_ok, gather_ok, h in got:
        assert exchange_ok and gather_ok and h == homo
