"""The small-m fp64 path (csrc/small_path.cu, corr2d_correlate_small_f64) in
both variants: K1 + the streamed contraction (the default) and the one-kernel
variant (CORR2D_SMALL_ONEKERNEL=1: each CTA builds its blocks' operand rows in
shared memory).  Parity against the CPU oracle (1e-10 of max|sync|,
BASELINE.json north_star) for every m it serves, exact homo symmetry,
agreement with the generic K1 + fp64 contraction, row shards (generic path)
bit-identical to that path's whole map, and the self-resetting status / stat
words (an error call must not leak into the next call)."""

import warnings

import numpy as np
import pytest

from conftest import rel_err
from oracle import corr2d_oracle as O
import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import engine
from paper_1808_00685_b200.errors import NumericError

pytestmark = pytest.mark.gpu
TOL64 = 1e-10


@pytest.fixture(params=["two-kernel", "one-kernel"])
def variant(request, monkeypatch):
    if request.param == "one-kernel":
        monkeypatch.setenv("CORR2D_SMALL_ONEKERNEL", "1")
    else:
        monkeypatch.delenv("CORR2D_SMALL_ONEKERNEL", raising=False)
    return request.param


def pipe_idle(plan):
    """The plan's pipeline words after a synchronise: no contraction CTA
    mid-release, every call's contraction completed (completed calls == the
    two slots' completed uses == contraction launches)."""
    w = plan.pipe.cpu().numpy()
    gen, planes, arrive = w[2:4], w[9], w[10:12]
    return not arrive.any() and planes == gen.sum()


def dyn(values, alpha=0.0):
    values = np.asarray(values, dtype=float)
    m, n = values.shape
    return P.DynamicSpectra(np.arange(n, dtype=float) + 1.0, np.arange(m, dtype=float), values,
                            np.zeros(n), scaling_exponent=alpha)


def scale_of(s, a):
    return max(float(np.abs(s).max()), float(np.abs(a).max()), 1e-300)


def _plan_is_small(n1, n2, m, homo=True):
    recipe = engine.PrepRecipe(m_in=m, m=m, ref_mode=P._abi.REF_NONE)
    plan = engine.CorrelationPlan(n1=n1, n2=n2, m=m, recipe1=recipe, recipe2=None if homo else recipe,
                                  norm=1.0, want_ref=False)
    return plan.small


def test_small_plans_take_the_fused_path():
    assert _plan_is_small(1000, 1000, 11) and _plan_is_small(2000, 1500, 21, homo=False)
    assert _plan_is_small(5, 5, 2) and _plan_is_small(64, 64, 32)
    assert not _plan_is_small(64, 64, 33)


@pytest.mark.parametrize("n1,n2,m", [(1, 1, 2), (3, 5, 3), (31, 33, 8), (63, 65, 5), (64, 64, 12),
                                     (65, 130, 21), (517, 300, 32), (1000, 999, 11)])
def test_fused_matches_oracle_homo_and_hetero(n1, n2, m, variant):
    rng = np.random.default_rng(n1 * 7 + n2 + m)
    v1 = rng.normal(size=(m, n1))
    v2 = rng.normal(size=(m, n2))
    res = P.correlate_ft(dyn(v1), dyn(v2))
    s, a, _ = O.correlate_ft(v1, v2)
    sc = scale_of(s, a)
    assert rel_err(res.sync, s, sc) <= TOL64 and rel_err(res.asyn, a, sc) <= TOL64
    homo = P.correlate_ft(dyn(v1))
    s, a, _ = O.correlate_ft(v1)
    sc = scale_of(s, a)
    assert rel_err(homo.sync, s, sc) <= TOL64 and rel_err(homo.asyn, a, sc) <= TOL64
    assert np.array_equal(homo.sync, homo.sync.T) and np.array_equal(homo.asyn, -homo.asyn.T)
    assert np.all(np.diag(homo.asyn) == 0)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_fused_full_pipeline_inputs(dtype):
    """Raw intensities (mean reference, alpha scaling, float32 storage) through corr2d()."""
    rng = np.random.default_rng(5)
    m, n = 21, 777
    t = np.linspace(0, 100, m)
    x = (rng.normal(size=(m, n)) + np.outer(np.sin(t / 9.0), rng.uniform(1, 3, n))).astype(dtype)
    ds = P.SpectralDataset(np.arange(n, dtype=float), t, x, dtype=x.dtype)
    for alpha in (0.0, 0.5):
        res = P.corr2d(ds, alpha=alpha)
        vals = np.asarray(x, dtype=np.float64)
        ref = vals.mean(axis=0)
        y = vals - ref
        if alpha:
            y = y / (np.sqrt(((vals - ref) ** 2).sum(axis=0) / (m - 1)) ** alpha)
        s, a, _ = O.correlate_ft(y)
        sc = scale_of(s, a)
        assert rel_err(res.sync, s, sc) <= TOL64 and rel_err(res.asyn, a, sc) <= TOL64
        assert np.array_equal(res.ref1, ref) or rel_err(res.ref1, ref) <= 1e-15


def test_row_shards_bit_identical_to_two_kernel_map(monkeypatch):
    """Row shards run the two-kernel path (the fused kernel serves whole maps):
    every shard equals the rows of that path's whole map bit for bit."""
    from paper_1808_00685_b200.engine_core import tile_aligned_blocks
    v = np.random.default_rng(3).normal(size=(11, 517))
    d = dyn(v)
    monkeypatch.setenv("CORR2D_SMALL_FUSED", "0")
    full = P.correlate_ft(d)
    monkeypatch.delenv("CORR2D_SMALL_FUSED")
    for parts in (2, 3, 8):
        for r0, r1 in tile_aligned_blocks(517, parts):
            sh = P.correlate_ft(d, rows=(r0, r1), return_device=True)
            assert np.array_equal(sh.sync.cpu().numpy(), full.sync[r0:r1])
            assert np.array_equal(sh.asyn.cpu().numpy(), full.asyn[r0:r1])


@pytest.mark.parametrize("m", list(range(2, 33)))
def test_fused_every_m(m, variant):
    rng = np.random.default_rng(100 + m)
    v1 = rng.normal(size=(m, 150)) * np.linspace(0.1, 10.0, 150)
    v2 = rng.normal(size=(m, 97))
    res = P.correlate_ft(dyn(v1), dyn(v2))
    s, a, _ = O.correlate_ft(v1, v2)
    sc = scale_of(s, a)
    assert rel_err(res.sync, s, sc) <= TOL64 and rel_err(res.asyn, a, sc) <= TOL64
    homo = P.correlate_ft(dyn(v1))
    s, a, _ = O.correlate_ft(v1)
    sc = scale_of(s, a)
    assert rel_err(homo.sync, s, sc) <= TOL64 and rel_err(homo.asyn, a, sc) <= TOL64
    assert np.array_equal(homo.sync, homo.sync.T) and np.array_equal(homo.asyn, -homo.asyn.T)


def test_fused_status_words_reset_between_calls(variant):
    """A call that flags non-finite input / zero variance must not leak its
    counters into the next call on the same plan (self-resetting accumulators)."""
    rng = np.random.default_rng(2)
    m, n = 11, 300
    t = np.arange(m, dtype=float)
    x = rng.normal(size=(m, n))
    bad = x.copy()
    bad[3, 17] = np.nan
    with pytest.raises(Exception):
        P.corr2d(P.SpectralDataset(np.arange(n, dtype=float), t, bad))
    good = P.corr2d(P.SpectralDataset(np.arange(n, dtype=float), t, x))
    assert np.isfinite(good.sync).all()
    # one plan, launched repeatedly: identical bits, clean status every time
    from paper_1808_00685_b200 import api
    ds = P.SpectralDataset(np.arange(n, dtype=float), t, x)
    plan, _ = api.build_plan(ds, None, P.PreprocessSpec(), dtype="float64")
    assert plan.small
    outs = []
    for _ in range(3):
        plan.launch()
        engine.sync()
        plan.check()
        outs.append(plan.phi.cpu().numpy().copy())
        assert not plan.work.cpu().numpy().any()      # accumulators / arrival counter left zero
        assert pipe_idle(plan)                        # pipelined calls: every slot released
    assert all(np.array_equal(o, outs[0]) for o in outs)
    # zero variance with alpha > 0: the error policy raises, the substitute policy warns
    flat = x.copy()
    flat[:, 40] = 2.5
    dsf = P.SpectralDataset(np.arange(n, dtype=float), t, flat)
    with pytest.raises(NumericError, match="zero-variance"):
        P.corr2d(dsf, alpha=0.5)
    res = P.corr2d(P.SpectralDataset(np.arange(n, dtype=float), t, x), alpha=0.5)
    assert np.isfinite(res.sync).all()


def test_fused_and_two_kernel_paths_agree(monkeypatch):
    rng = np.random.default_rng(4)
    v = rng.normal(size=(21, 1500))
    fused = P.correlate_ft(dyn(v))
    monkeypatch.setenv("CORR2D_SMALL_FUSED", "0")
    two = P.correlate_ft(dyn(v))
    sc = scale_of(two.sync, two.asyn)
    assert rel_err(fused.sync, two.sync, sc) <= 1e-13 and rel_err(fused.asyn, two.asyn, sc) <= 1e-13


# maps with more 64 x 64 blocks than SMs: K1 + the streamed contraction
# (small_stream_kernel: persistent CTAs, double-buffered operand rows, TMA
# tensor stores from one or two staging slots; m = 29..32 has one slot, so a
# mirrored block stores twice through it)
@pytest.mark.parametrize("n1,n2,m", [(1100, 1100, 21), (1090, 1090, 32), (1000, 1023, 11), (2000, 1500, 21),
                                     (1153, 700, 5), (700, 1153, 30), (1201, 1201, 2), (9000, 130, 13)])
def test_streamed_contraction_matches_oracle(n1, n2, m):
    from paper_1808_00685_b200 import _abi
    lib = _abi.load()
    homo = n1 == n2
    assert lib.corr2d_small_launches(n1, n2, 1 if homo else 0) == 2
    rng = np.random.default_rng(n1 + 3 * n2 + m)
    v1 = rng.normal(size=(m, n1)) * np.linspace(0.5, 4.0, n1)
    if homo:
        res = P.correlate_ft(dyn(v1))
        s, a, _ = O.correlate_ft(v1)
    else:
        v2 = rng.normal(size=(m, n2))
        res = P.correlate_ft(dyn(v1), dyn(v2))
        s, a, _ = O.correlate_ft(v1, v2)
    sc = scale_of(s, a)
    assert rel_err(res.sync, s, sc) <= TOL64 and rel_err(res.asyn, a, sc) <= TOL64
    if homo:
        assert np.array_equal(res.sync, res.sync.T) and np.array_equal(res.asyn, -res.asyn.T)
        assert np.all(np.diag(res.asyn) == 0)


def test_streamed_contraction_flags_nonfinite_and_resets():
    """The streamed contraction's stats: a non-finite input is reported, and the
    next call on the same plan is clean (K1 zeroes, the contraction publishes)."""
    from paper_1808_00685_b200 import api
    rng = np.random.default_rng(8)
    m, n = 21, 1300
    t = np.arange(m, dtype=float)
    x = rng.normal(size=(m, n))
    bad = x.copy()
    bad[5, 1234] = np.inf
    with pytest.raises(Exception):
        P.corr2d(P.SpectralDataset(np.arange(n, dtype=float), t, bad))
    ds = P.SpectralDataset(np.arange(n, dtype=float), t, x)
    plan, _ = api.build_plan(ds, None, P.PreprocessSpec(), dtype="float64")
    assert plan.small and plan.launches_per_step == 2
    outs = []
    for _ in range(3):
        plan.launch()
        engine.sync()
        plan.check()
        outs.append(plan.phi.cpu().numpy().copy())
        assert not plan.work.cpu().numpy().any()
    assert all(np.array_equal(o, outs[0]) for o in outs)


@pytest.mark.parametrize("n1,n2", [(1300, 1300), (1000, 1100), (400, 400)])
def test_back_to_back_launches_with_rebound_inputs(n1, n2, variant):
    """Programmatic dependent launch lets K1 of the next call start (reading
    its inputs) while the previous call's contraction runs; its writes wait.
    Back-to-back launches of ONE plan on alternating inputs -- without a host
    sync or any copy in between -- must each produce their own map, status and
    statistics: a non-finite input in call k flags call k only."""
    import torch
    from paper_1808_00685_b200 import api
    rng = np.random.default_rng(n1 + n2)
    m = 21
    t = np.arange(m, dtype=float)
    homo = n1 == n2
    xs = [rng.normal(size=(m, n1)) * np.linspace(1.0, 3.0, n1) for _ in range(2)]
    ys = [None, None] if homo else [rng.normal(size=(m, n2)) for _ in range(2)]
    bad = xs[0].copy()
    bad[4, 7] = np.nan
    mk = lambda x, n: P.SpectralDataset(np.arange(n, dtype=float), t, x)
    plan, _ = api.build_plan(mk(xs[0], n1), None if homo else mk(ys[0], n2), P.PreprocessSpec(), dtype="float64")
    assert plan.small
    dev = plan.phi.device
    raws = [torch.from_numpy(x).to(dev) for x in (xs[0], xs[1], bad)]
    raws2 = [None, None] if homo else [torch.from_numpy(y).to(dev) for y in ys]
    oracle = []
    for k in range(2):
        if homo:
            s, a, _ = O.correlate_ft(xs[k] - xs[k].mean(axis=0))
        else:
            s, a, _ = O.correlate_ft(xs[k] - xs[k].mean(axis=0), ys[k] - ys[k].mean(axis=0))
        oracle.append((s, a))
    # A, B, A, B back to back; the last call's outputs are B's
    for k in (0, 1, 0, 1):
        plan.bind(raws[k], raws2[k])
        plan.launch()
    engine.sync()
    plan.check()
    s, a = oracle[1]
    sc = scale_of(s, a)
    assert rel_err(plan.phi.cpu().numpy(), s, sc) <= TOL64 and rel_err(plan.psi.cpu().numpy(), a, sc) <= TOL64
    # a bad call followed at once by a clean one: the clean call's status is clean
    plan.bind(raws[2], raws2[0])
    plan.launch()
    plan.bind(raws[0], raws2[0])
    plan.launch()
    engine.sync()
    plan.check()
    s, a = oracle[0]
    assert rel_err(plan.phi.cpu().numpy(), s, sc) <= TOL64 * 10
    # and the other way round: the bad call is reported
    plan.bind(raws[0], raws2[0])
    plan.launch()
    plan.bind(raws[2], raws2[0])
    plan.launch()
    engine.sync()
    with pytest.raises(NumericError, match="non-finite"):
        plan.check()
    assert not plan.work.cpu().numpy().any() and pipe_idle(plan)
    # a longer back-to-back chain (graph-captured, as bench.py replays it):
    # A, B alternating, the last launch's map is B's
    s_, stream = torch.cuda.current_stream(), torch.cuda.Stream()
    stream.wait_stream(s_)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            for k in range(9):
                plan.bind(raws[k % 2], raws2[k % 2])
                plan.launch()
    s_.wait_stream(stream)
    for _ in range(3):
        g.replay()
    engine.sync()
    s, a = oracle[0]                                   # k = 8: input A
    sc = scale_of(s, a)
    assert rel_err(plan.phi.cpu().numpy(), s, sc) <= TOL64 and rel_err(plan.psi.cpu().numpy(), a, sc) <= TOL64
    assert pipe_idle(plan)
