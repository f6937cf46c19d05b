"""Multi-rank logic on the CPU: the tile-range partition used by bench.py for
N GPUs (every output element written exactly once, by exactly one rank), the
row-shard partition of correlate_ft(rows=...), and the torch.distributed
plumbing (world_size 2, gloo, 127.0.0.1)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_00685_b200.engine_core import (DIAG, MIRROR, PLAIN, TRANS_ONLY, homo_tile_count,
                                               homo_tile_decode, tile_aligned_blocks, tile_range)

ROOT = Path(__file__).resolve().parent.parent


def coverage(n, tile, row0, row1, tiles):
    """Count how often each output element of rows [row0, row1) is written
    by the tiles `tiles` of the shard's enumeration (kernel semantics)."""
    cnt = np.zeros((n, n), dtype=np.int32)
    for b in tiles:
        I, J, mode = homo_tile_decode(b, n, tile, row0, row1)
        i0, j0 = I * tile, J * tile
        for r in range(tile):
            for c in range(tile):
                gi, gj = i0 + r, j0 + c
                if mode != TRANS_ONLY and gi < row1 and gj < n and (mode != DIAG or r <= c):
                    cnt[gi, gj] += 1
                if mode in (MIRROR, DIAG, TRANS_ONLY) and gj < row1 and gj >= row0 and gi < n and (mode != DIAG or r < c):
                    cnt[gj, gi] += 1
    return cnt


@pytest.mark.parametrize("n,tile", [(64, 16), (70, 16), (33, 8)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_tile_ranges_cover_map_exactly_once(n, tile, world):
    total = homo_tile_count(n, tile)
    acc = np.zeros((n, n), dtype=np.int32)
    for rank in range(world):
        t0, t1 = tile_range(total, world, rank)
        acc += coverage(n, tile, 0, n, range(t0, t1))
    assert np.all(acc == 1)


@pytest.mark.parametrize("n,tile,parts", [(70, 16, 2), (64, 16, 4), (33, 8, 3)])
def test_row_shards_cover_their_rows_exactly_once(n, tile, parts):
    for row0, row1 in tile_aligned_blocks(n, parts, tile):
        total = homo_tile_count(n, tile, row0, row1)
        cnt = coverage(n, tile, row0, row1, range(total))
        assert np.all(cnt[row0:row1] == 1)
        assert np.all(cnt[:row0] == 0) and np.all(cnt[row1:] == 0)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    sys.path.insert(0, str(ROOT))
    import bench
    total = homo_tile_count(32768, 128)
    t0, t1 = tile_range(total, world, rank)
    mine = torch.tensor([t1 - t0], dtype=torch.int64)
    dist.all_reduce(mine)
    mx = bench.allreduce_max(float(rank + 1) * 1.5, world)
    bench.barrier(world)
    if rank == 0:
        out.put((int(mine.item()), total, mx))
    dist.destroy_process_group()


def test_gloo_world2_partition_and_max_over_ranks():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    covered, total, mx = q.get(timeout=5)
    assert covered == total
    assert mx == 3.0


def test_reference_arm_under_torchrun_prints_one_line():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29617", str(ROOT / "bench.py"),
           "--impl", "reference", "--gpus", "2", "--config", "1", "--steps", "1", "--warmup", "0"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def pair_coverage(n1, n2, tile, homo, tiles, G, quad=False):
    from paper_1808_00685_b200.engine_core import SKIP, pair_tile_decode, quad_tile_decode
    T1, T2 = -(-n1 // tile), -(-n2 // tile)
    cnt = np.zeros((n1, n2), dtype=np.int32)
    for b in tiles:
        for rank in ((0, 1, 2, 3) if quad else (0, 1)):
            if quad:
                P, J, mode = quad_tile_decode(b, T1, T2, homo, rank, G)
            else:
                P, J, mode = pair_tile_decode(b, T1, T2, homo, rank, G)
            if mode == SKIP:
                continue
            i0, j0 = (2 * P + (rank & 1)) * tile, J * tile
            r, c = np.meshgrid(np.arange(tile), np.arange(tile), indexing="ij")
            gi, gj = i0 + r, j0 + c
            ok = (gi < n1) & (gj < n2)
            direct = ok & ((r <= c) if mode == DIAG else True)
            cnt[gi[direct], gj[direct]] += 1
            if mode in (MIRROR, DIAG):
                mir = ok & ((r < c) if mode == DIAG else True) & (gj < n1) & (gi < n2)
                cnt[gj[mir], gi[mir]] += 1
    return cnt


@pytest.mark.parametrize("n,tile,G", [(64, 8, 2), (72, 8, 3), (40, 8, 16), (130, 8, 4)])
@pytest.mark.parametrize("world", [1, 3])
def test_pair_tiles_cover_homo_map_once(n, tile, G, world):
    from paper_1808_00685_b200.engine_core import pair_tile_count
    T = -(-n // tile)
    total = pair_tile_count(T, T, True)
    acc = np.zeros((n, n), dtype=np.int32)
    for rank in range(world):
        t0, t1 = tile_range(total, world, rank)
        acc += pair_coverage(n, n, tile, True, range(t0, t1), G)
    assert np.all(acc == 1)


@pytest.mark.parametrize("n1,n2,G", [(64, 40, 2), (72, 24, 16), (24, 72, 3)])
def test_pair_tiles_cover_hetero_map_once(n1, n2, G):
    from paper_1808_00685_b200.engine_core import pair_tile_count
    T1, T2 = -(-n1 // 8), -(-n2 // 8)
    acc = pair_coverage(n1, n2, 8, False, range(pair_tile_count(T1, T2, False)), G)
    assert np.all(acc == 1)


@pytest.mark.parametrize("n,G", [(64, 2), (72, 3), (40, 16), (130, 4), (88, 1)])
@pytest.mark.parametrize("world", [1, 3])
def test_quad_tiles_cover_homo_map_once(n, G, world):
    from paper_1808_00685_b200.engine_core import quad_tile_count
    T = -(-n // 8)
    total = quad_tile_count(T, T, True)
    acc = np.zeros((n, n), dtype=np.int32)
    for rank in range(world):
        t0, t1 = tile_range(total, world, rank)
        acc += pair_coverage(n, n, 8, True, range(t0, t1), G, quad=True)
    assert np.all(acc == 1)


@pytest.mark.parametrize("n1,n2,G", [(64, 40, 2), (72, 24, 16), (24, 72, 3), (40, 56, 1)])
def test_quad_tiles_cover_hetero_map_once(n1, n2, G):
    from paper_1808_00685_b200.engine_core import quad_tile_count
    T1, T2 = -(-n1 // 8), -(-n2 // 8)
    acc = pair_coverage(n1, n2, 8, False, range(quad_tile_count(T1, T2, False)), G, quad=True)
    assert np.all(acc == 1)


def _gather_worker(rank, world, port, n, out):
    """Each rank fills only its channel chunk of a (world*chunk) x L buffer (as
    K1 does with spectra_shard) plus its status word; after gather_rows and the
    status all-reduce every rank holds the full buffer and the combined status."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_1808_00685_b200.engine_core import channel_chunk, gather_rows
    c0, c1, chunk = channel_chunk(n, world, rank)
    buf = torch.zeros(world * chunk, 5, dtype=torch.float64)
    for c in range(c0, c1):
        buf[c] = torch.arange(5, dtype=torch.float64) + 10.0 * c
    gather_rows(buf, chunk, world, rank)
    status = torch.tensor([rank, 1 if rank == 1 else 0, 2**31 - 1 - 7 * (rank + 1), 0], dtype=torch.int32)
    dist.all_reduce(status[:2], op=dist.ReduceOp.SUM)
    dist.all_reduce(status[2:3], op=dist.ReduceOp.MAX)
    out.put((rank, buf.numpy().copy(), status.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 10), (3, 10), (3, 2)])
def test_gloo_sharded_spectra_allgather(world, n):
    import socket
    from paper_1808_00685_b200.engine_core import channel_chunk
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    chunk = channel_chunk(n, world, 0)[2]
    want = np.zeros((world * chunk, 5))
    for c in range(n):
        want[c] = np.arange(5) + 10.0 * c
    for rank, buf, st in res:
        assert np.array_equal(buf, want)
        assert st[0] == sum(range(world)) and st[1] == 1 and st[2] == 2**31 - 1 - 7
    # chunks tile the channels exactly once
    seen = np.zeros(n, dtype=int)
    for r in range(world):
        c0, c1, _ = channel_chunk(n, world, r)
        seen[c0:c1] += 1
    assert np.all(seen == 1)
