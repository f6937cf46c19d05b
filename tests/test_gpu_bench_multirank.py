"""bench.py's multi-rank path (torchrun, row bands through the public
distributed plan, both spectra schemes) end to end on one GPU: BENCH_ONE_DEVICE=1 puts both ranks on cuda:0
over gloo, so the launch / partition / reduction / JSON contract is exercised
even where only one device exists (the timings mean nothing there)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("spectra,port,config", [("recompute", 29531, 2), ("broadcast", 29532, 2),
                                                 ("broadcast", 29533, 4)])
def test_bench_two_ranks_one_device(spectra, port, config):
    env = dict(os.environ, BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--config", str(config), "--steps", "2", "--warmup", "3", "--spectra", spectra]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]          # rank 0 prints one line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["scaling"] == "strong"
    assert d["value"] > 0 and d["gpu_launches"] > 0
    if d.get("parity"):                                  # gated on rank 0 when present
        assert d["parity"]["max_rel_err"] <= d["parity"]["tol"]
    assert spectra in d["config"]["parallelism"]
