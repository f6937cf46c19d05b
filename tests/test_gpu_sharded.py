"""Multi-GPU band ownership through the PUBLIC call (sharded.py):
``corr2d(..., distributed=True)`` on every rank, ``gather()`` on rank 0, equal
bit for bit to the one-GPU ``corr2d`` map.  The ranks run over gloo, all on
this one device (only one GPU is available): the code path -- K1 on the
rank's chunk, the owners' broadcasts, the diagonal square and the rectangle
pieces on pointer-offset operands, the status / stats reductions, the gather
-- is the one NCCL runs, with the broadcasts staged through the host."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CASES = {
    # name: (dtype, m, n1, n2 or None, resample, alpha)
    "f64_homo": ("float64", 64, 1000, None, None, 0.0),
    "f64_homo_resampled_scaled": ("float64", 37, 777, None, 64, 0.5),
    "f64_hetero": ("float64", 21, 900, 650, None, 0.0),
    "f32_homo": ("float32", 64, 1100, None, None, 0.0),
    "f32_hetero": ("float32", 64, 700, 520, None, 0.0),
}


def _datasets(name):
    import paper_1808_00685_b200 as P
    dtype, m, n1, n2, resample, alpha = CASES[name]
    rng = np.random.default_rng(sum(map(ord, name)))      # same data in every rank's process
    t = np.sort(rng.uniform(0.0, 50.0, m)) if resample else np.arange(m, dtype=float)
    dt = np.float32 if dtype == "float32" else np.float64
    ds1 = P.SpectralDataset(np.arange(n1, dtype=float), t, rng.normal(size=(m, n1)) + 1.0, dtype=dt)
    ds2 = None if n2 is None else P.SpectralDataset(np.arange(n2, dtype=float) + 0.5, t,
                                                    rng.normal(size=(m, n2)) - 1.0, dtype=dt)
    kw = dict(dtype=dtype, alpha=alpha)
    if resample:
        kw.update(resample=resample, interpolant="linear")
    return ds1, ds2, kw


def _worker(rank, world, port, name, spectra, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, str(ROOT))
        import paper_1808_00685_b200 as P
        torch.cuda.set_device(0)
        ds1, ds2, kw = _datasets(name)
        res = P.corr2d(ds1, ds2, distributed=True, spectra=spectra, **kw)
        band_ok = tuple(res.sync.shape) == (res.rows[1] - res.rows[0], res.cols[1] - res.cols[0])
        full = res.gather(root=0)
        if rank == 0:
            fused = P.corr2d(ds1, ds2, **kw)      # m <= 32 fp64: the one-kernel path (other rounding)
            os.environ["CORR2D_SMALL_FUSED"] = "0"
            one = P.corr2d(ds1, ds2, **kw)        # the two-kernel path the bands run
            del os.environ["CORR2D_SMALL_FUSED"]
            scale = max(float(np.abs(fused.sync).max()), float(np.abs(fused.asyn).max()))
            close = max(float(np.abs(full.sync - fused.sync).max()),
                        float(np.abs(full.asyn - fused.asyn).max())) <= 1e-12 * scale
            same = bool(np.array_equal(full.sync, one.sync) and np.array_equal(full.asyn, one.asyn))
            meta = (np.array_equal(full.ref1, one.ref1) and np.array_equal(full.ref2, one.ref2)
                    and full.normalization == one.normalization and full.is_homo == one.is_homo
                    and full.stats == one.stats)
            q.put((rank, band_ok, same and close, bool(meta), res.band_bytes))
        else:
            q.put((rank, band_ok, full is None, True, res.band_bytes))
    finally:
        dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("world,spectra", [(2, "broadcast"), (3, "broadcast"), (2, "recompute")])
def test_distributed_corr2d_bit_identical_to_one_gpu(name, world, spectra):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, spectra, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for rank, band_ok, same, meta, _ in got:
        assert band_ok and same and meta, (rank, band_ok, same, meta)
    dtype, m, n1, n2, *_ = CASES[name]
    elem = 4 if dtype == "float32" else 8
    full_bytes = 2 * elem * n1 * (n2 or n1)
    # bands, not whole maps: a homo rank holds its rows right of the diagonal
    # (plus its diagonal square's lower half)
    assert sum(b for *_, b in got) < full_bytes * (0.85 if n2 is None else 1.01)


def test_distributed_needs_a_process_group():
    import paper_1808_00685_b200 as P
    rng = np.random.default_rng(0)
    ds = P.SpectralDataset(np.arange(50.0), np.arange(8.0), rng.normal(size=(8, 50)))
    with pytest.raises(P.DataError, match="process group"):
        P.corr2d(ds, distributed=True)
