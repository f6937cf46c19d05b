"""GPU parity: the sm_100a path (through the C ABI) against the golden fixtures
made by the reference and against the CPU oracle.  Tolerances (BASELINE.json
north_star): max |delta| / max|sync_ref| <= 1e-10 in fp64, <= 1e-4 in fp32."""

import warnings

import numpy as np
import pytest

from conftest import golden, golden_names, rel_err
from oracle import corr2d_oracle as O
import paper_1808_00685_b200 as P

pytestmark = pytest.mark.gpu
TOL64 = 1e-10
TOL32 = 1e-4


def dyn_from_values(values, alpha=0.0):
    values = np.asarray(values, dtype=float)
    m, n = values.shape
    return P.DynamicSpectra(np.arange(n, dtype=float) + 1.0, np.arange(m, dtype=float), values,
                            np.zeros(n), scaling_exponent=alpha)


def scale_of(sync, asyn):
    return max(float(np.abs(sync).max()), float(np.abs(asyn).max()), 1e-300)


@pytest.mark.parametrize("name", golden_names("homo_"))
def test_homo_pipeline_matches_reference(name):
    g = golden(name)
    ds = P.SpectralDataset(g["nu"], g["t"], g["raw"])
    dyn = P.preprocess_dataset(ds)
    if ds.m <= 128:   # left-to-right mean over the axis: bitwise equal to numpy
        assert np.array_equal(dyn.reference_used, g["ref"])
        assert np.array_equal(dyn.values, g["values"])
    else:             # warp-parallel sums for long axes: a few ulp
        assert rel_err(dyn.reference_used, g["ref"]) <= 1e-14
        assert rel_err(dyn.values, g["values"]) <= 1e-14
    ws = P.dft_channels(dyn)
    assert rel_err(ws.half_spectrum1, g["half"]) <= 1e-13
    assert np.all(ws.half_spectrum1[0].imag == 0)
    res = P.correlate_ft(dyn)
    sc = scale_of(g["sync"], g["asyn"])
    assert rel_err(res.sync, g["sync"], sc) <= TOL64
    assert rel_err(res.asyn, g["asyn"], sc) <= TOL64
    assert res.normalization == float(g["norm"]) and res.is_homo and res.engine == "fourier"
    # exact symmetry by construction (dataset.py:159-170 at tolerance 0)
    assert np.array_equal(res.sync, res.sync.T)
    assert np.array_equal(res.asyn, -res.asyn.T)
    assert np.all(np.diag(res.asyn) == 0)


@pytest.mark.parametrize("name", golden_names("hetero_"))
def test_hetero_matches_reference(name):
    g = golden(name)
    d1 = P.preprocess_dataset(P.SpectralDataset(g["nu1"], g["t"], g["raw1"]))
    d2 = P.preprocess_dataset(P.SpectralDataset(g["nu2"], g["t"], g["raw2"]))
    res = P.correlate_ft(d1, d2)
    assert not res.is_homo
    sc = scale_of(g["sync"], g["asyn"])
    assert rel_err(res.sync, g["sync"], sc) <= TOL64
    assert rel_err(res.asyn, g["asyn"], sc) <= TOL64


@pytest.mark.parametrize("name", golden_names("pre_"))
def test_preprocess_variants(name):
    g = golden(name)
    import json
    from conftest import GOLDEN
    spec_txt = json.loads((GOLDEN / "manifest.json").read_text())["cases"][name].get("spec", {})
    resample = None
    if "resample" in spec_txt:
        txt = spec_txt["resample"]
        kind = P.InterpolantKind.LINEAR if "LINEAR" in txt else P.InterpolantKind.CUBIC_SPLINE
        resample = P.ResampleSpec(int(txt.split("target_count=")[1].split(",")[0]), kind)
    alpha = float(spec_txt.get("scaling_exponent", 0.5 if "zero_variance" in name else 0.0))
    ref = P.ReferenceSpec.provided(g["provided"]) if "provided" in g else P.ReferenceSpec.mean()
    spec = P.PreprocessSpec(reference=ref, resample=resample, scaling_exponent=alpha)
    ds = P.SpectralDataset(g["nu"], g["t"], g["raw"])
    policy = "substitute" if "zero_variance" in name else "error"
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dyn = P.preprocess_dataset(ds, spec, on_zero_variance=policy)
    spline = resample is not None and resample.interpolant is P.InterpolantKind.CUBIC_SPLINE and g["t"].size > 2
    if "t_used" in g:
        assert np.array_equal(dyn.perturbation_axis, g["t_used"])
    if alpha not in (0.0, 0.5, 1.0):  # CUDA pow vs libm pow: last-ulp differences
        assert rel_err(dyn.values, g["values"]) <= 1e-14
        assert np.array_equal(dyn.reference_used, g["ref"]) and np.array_equal(dyn.sigma, g["sigma"])
    elif spline:   # dense spline matrix vs scipy's banded solve: rounding-level
        assert rel_err(dyn.values, g["values"]) <= 1e-12
        assert rel_err(dyn.reference_used, g["ref"]) <= 1e-12
    else:        # same operations, same order: bitwise
        assert np.array_equal(dyn.values, g["values"])
        assert np.array_equal(dyn.reference_used, g["ref"])
        if "sigma" in g:
            assert np.array_equal(dyn.sigma, g["sigma"])
    res = P.correlate_ft(dyn)
    sc = scale_of(g["sync"], g["asyn"])
    assert rel_err(res.sync, g["sync"], sc) <= TOL64
    assert rel_err(res.asyn, g["asyn"], sc) <= TOL64
    # the fused one-call pipeline gives the same planes
    kw = dict(alpha=alpha, on_zero_variance=policy)
    if resample is not None:
        kw.update(resample=resample.target_count, interpolant=resample.interpolant.value)
    if "provided" in g:
        kw["reference"] = g["provided"]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        fused = P.corr2d(ds, **kw)
    assert rel_err(fused.sync, g["sync"], sc) <= TOL64
    assert rel_err(fused.asyn, g["asyn"], sc) <= TOL64


def test_norm_variants():
    g = golden("norm_unit_custom")
    dyn = dyn_from_values(g["values"])
    r1 = P.correlate_ft(dyn, norm=P.NormalizationSpec.unit())
    r2 = P.correlate_ft(dyn, norm=P.NormalizationSpec.custom(0.4))
    assert r2.normalization == 0.4
    assert rel_err(r1.sync, g["sync_unit"]) <= TOL64
    assert rel_err(r2.asyn, g["asyn_custom"], np.abs(g["sync_custom"]).max()) <= TOL64


def test_zero_variance_error_and_warning():
    raw = np.random.default_rng(0).normal(size=(6, 5))
    raw[:, 2] = 1.25
    ds = P.SpectralDataset(np.arange(5.0), np.arange(6.0), raw)
    with pytest.raises(P.NumericError, match="zero-variance spectral channel"):
        P.preprocess_dataset(ds, P.PreprocessSpec(scaling_exponent=0.5))
    with pytest.warns(RuntimeWarning, match="substituting sigma = 1"):
        dyn = P.preprocess_dataset(ds, P.PreprocessSpec(scaling_exponent=0.5), on_zero_variance="substitute")
    assert dyn.sigma[2] == 1.0
    with pytest.raises(P.DataError, match="unknown zero-variance policy"):
        P.preprocess_dataset(ds, P.PreprocessSpec(scaling_exponent=0.5), on_zero_variance="bogus")


def test_non_finite_rejected():
    values = np.zeros((4, 2))
    values[1, 1] = np.nan
    with pytest.raises(P.NumericError, match="non-finite"):
        P.dft_channels(dyn_from_values(values))
    with pytest.raises(P.NumericError, match="first dynamic-spectra matrix contains non-finite"):
        P.correlate_ft(dyn_from_values(values))


def test_errors_match_reference():
    rng = np.random.default_rng(7)
    d1 = dyn_from_values(rng.normal(size=(8, 4)))
    d2 = dyn_from_values(rng.normal(size=(9, 4)))
    with pytest.raises(P.DataError, match="perturbation axes differ"):
        P.correlate_ft(d1, d2)
    d3 = dyn_from_values(np.zeros((8, 4)), alpha=0.5)
    with pytest.raises(P.DataError, match="scaling regimes differ"):
        P.correlate_ft(d1, d3)


def test_cosine_bin_one():
    m = 8
    col = np.cos(2 * np.pi * np.arange(m) / m)
    ws = P.dft_channels(dyn_from_values(np.column_stack([col, col])))
    mag = np.abs(ws.half_spectrum1[:, 0])
    assert mag[1] == pytest.approx(m / 2, rel=1e-12)
    assert np.all(np.delete(mag, 1) < 1e-12)


@pytest.mark.parametrize("m", list(range(2, 65)) + [96, 100, 127, 128, 255, 256, 257, 509, 512, 1000, 1024])
def test_dft_matches_oracle_any_m(m):
    rng = np.random.default_rng(m)
    v = rng.normal(size=(m, 37))
    ws = P.dft_channels(dyn_from_values(v))
    ref = O.dft_channels(v)
    assert rel_err(ws.half_spectrum1, ref) <= 1e-12
    res = P.correlate_ft(dyn_from_values(v))
    s, a, _ = O.correlate_ft(v)
    sc = scale_of(s, a)
    assert rel_err(res.sync, s, sc) <= TOL64 and rel_err(res.asyn, a, sc) <= TOL64


@pytest.mark.parametrize("n1,n2,m", [(1, 1, 2), (63, 65, 5), (64, 64, 12), (65, 130, 21), (200, 3, 64), (129, 257, 33)])
def test_ragged_shapes(n1, n2, m):
    rng = np.random.default_rng(n1 * 1000 + n2)
    v1 = rng.normal(size=(m, n1))
    v2 = rng.normal(size=(m, n2))
    d1 = P.DynamicSpectra(np.arange(n1, dtype=float), np.arange(m, dtype=float), v1, np.zeros(n1))
    d2 = P.DynamicSpectra(np.arange(n2, dtype=float) + .5, np.arange(m, dtype=float), v2, np.zeros(n2))
    res = P.correlate_ft(d1, d2)
    s, a, _ = O.correlate_ft(v1, v2)
    sc = scale_of(s, a)
    assert rel_err(res.sync, s, sc) <= TOL64 and rel_err(res.asyn, a, sc) <= TOL64
    homo = P.correlate_ft(d1)
    s, a, _ = O.correlate_ft(v1)
    sc = scale_of(s, a)
    assert rel_err(homo.sync, s, sc) <= TOL64 and rel_err(homo.asyn, a, sc) <= TOL64


def test_repeat_bit_identical_and_workers_invariant():
    v = np.random.default_rng(6).normal(size=(10, 300))
    d = dyn_from_values(v)
    r1 = P.correlate_ft(d, workers=1)
    r2 = P.correlate_ft(d, workers=3)
    assert np.array_equal(r1.sync, r2.sync) and np.array_equal(r1.asyn, r2.asyn)


def test_row_shards_bit_identical_to_full():
    """Row ownership (multi-GPU partition) reproduces the full map exactly."""
    from paper_1808_00685_b200.engine_core import tile_aligned_blocks
    v = np.random.default_rng(3).normal(size=(33, 517))
    d = dyn_from_values(v)
    full = P.correlate_ft(d)
    for parts in (2, 3, 8):
        for r0, r1 in tile_aligned_blocks(517, parts):
            sh = P.correlate_ft(d, rows=(r0, r1), return_device=True)
            assert np.array_equal(sh.sync.cpu().numpy(), full.sync[r0:r1])
            assert np.array_equal(sh.asyn.cpu().numpy(), full.asyn[r0:r1])


FP32_FORMATS = ("f16f8", "bf16x3")     # CORR2D_FP32_FORMAT: operand formats of the tensor-core path


@pytest.mark.parametrize("fmt", FP32_FORMATS)
def test_fp32_path_small(fmt, monkeypatch):
    monkeypatch.setenv("CORR2D_FP32_FORMAT", fmt)
    rng = np.random.default_rng(11)
    for m, n in [(64, 300), (512, 200), (37, 129)]:
        v = rng.normal(size=(m, n))
        res = P.correlate_ft(dyn_from_values(v), dtype="float32")
        assert res.sync.dtype == np.float32
        s, a, _ = O.correlate_ft(v)
        sc = scale_of(s, a)
        assert rel_err(res.sync, s, sc) <= TOL32 and rel_err(res.asyn, a, sc) <= TOL32
        assert np.array_equal(res.sync, res.sync.T) and np.array_equal(res.asyn, -res.asyn.T)


@pytest.mark.parametrize("fmt", FP32_FORMATS)
def test_fp32_tile_ranges_and_both_tensor_core_kernels(fmt, monkeypatch):
    """Tile-range partition (multi-GPU unit) is bit-identical to the whole map,
    for the 2-SM (CTA pair) kernel and the 1-SM kernel; both match the oracle."""
    monkeypatch.setenv("CORR2D_FP32_FORMAT", fmt)
    from paper_1808_00685_b200 import engine
    from paper_1808_00685_b200.engine_core import tile_range
    rng = np.random.default_rng(21)
    v = rng.normal(size=(64, 700))
    s, a, _ = O.correlate_ft(v)
    sc = scale_of(s, a)
    for one_sm, quads in (("0", "0"), ("0", "1"), ("1", "0")):   # pairs, A-multicast quads, 1-SM
        monkeypatch.setenv("CORR2D_BF16_1SM", one_sm)
        monkeypatch.setenv("CORR2D_BF16_QUADS", quads)
        d = dyn_from_values(v)
        full = P.correlate_ft(d, dtype="float32")
        assert rel_err(full.sync, s, sc) <= TOL32 and rel_err(full.asyn, a, sc) <= TOL32
        assert np.array_equal(full.sync, full.sync.T) and np.array_equal(full.asyn, -full.asyn.T)
        recipe = engine.PrepRecipe(m_in=64, m=64, ref_mode=P._abi.REF_NONE)
        plan = engine.CorrelationPlan(n1=700, n2=700, m=64, recipe1=recipe, recipe2=None,
                                      norm=1.0 / (np.pi * 63), dtype="float32", want_ref=False)
        plan.bind(d.device_values(plan.dev))
        plan.launch_prep_only()
        total = plan.tile_count()
        plan.phi.zero_()
        plan.psi.zero_()
        for rank in range(3):
            plan.tile0, plan.tile1 = tile_range(total, 3, rank)
            plan.launch_contract()
        engine.sync()
        assert np.array_equal(plan.phi.cpu().numpy(), full.sync)
        assert np.array_equal(plan.psi.cpu().numpy(), full.asyn)


@pytest.mark.parametrize("fmt", FP32_FORMATS)
@pytest.mark.parametrize("n1,n2,m", [(300, 257, 64), (129, 1000, 37), (700, 65, 512), (5, 3, 2), (1025, 511, 21)])
def test_fp32_hetero_ragged(n1, n2, m, fmt, monkeypatch):
    """Tensor-core path, hetero: CTA-pair kernel for aligned planes, the register-store
    epilogue for n2 % 4 != 0, odd / even m, tiny and ragged shapes."""
    monkeypatch.setenv("CORR2D_FP32_FORMAT", fmt)
    rng = np.random.default_rng(n1 * 7 + n2 * 13 + m)
    v1 = rng.normal(size=(m, n1))
    v2 = rng.normal(size=(m, n2))
    d1 = P.DynamicSpectra(np.arange(n1, dtype=float), np.arange(m, dtype=float), v1, np.zeros(n1))
    d2 = P.DynamicSpectra(np.arange(n2, dtype=float) + .5, np.arange(m, dtype=float), v2, np.zeros(n2))
    res = P.correlate_ft(d1, d2, dtype="float32")
    s, a, _ = O.correlate_ft(v1, v2)
    sc = scale_of(s, a)
    assert res.sync.shape == (n1, n2)
    assert rel_err(res.sync, s, sc) <= TOL32 and rel_err(res.asyn, a, sc) <= TOL32


@pytest.mark.parametrize("fmt", FP32_FORMATS)
def test_fp32_row_shards_match_whole_map(fmt, monkeypatch):
    """Row shards (the 1-SM kernel with transpose-only tiles) reproduce the
    whole fp32 map bit for bit."""
    monkeypatch.setenv("CORR2D_FP32_FORMAT", fmt)
    from paper_1808_00685_b200.engine_core import tile_aligned_blocks
    v = np.random.default_rng(8).normal(size=(96, 600))
    d = dyn_from_values(v)
    full = P.correlate_ft(d, dtype="float32", return_device=True)
    whole1 = None
    import os
    os.environ["CORR2D_BF16_1SM"] = "1"
    try:
        whole1 = P.correlate_ft(d, dtype="float32").sync
        for r0, r1 in tile_aligned_blocks(600, 3, 128):
            sh = P.correlate_ft(d, dtype="float32", rows=(r0, r1), return_device=True)
            assert np.array_equal(sh.sync.cpu().numpy(), whole1[r0:r1])
    finally:
        del os.environ["CORR2D_BF16_1SM"]
    s, a, _ = O.correlate_ft(v)
    sc = scale_of(s, a)
    assert rel_err(full.sync.cpu().numpy(), s, sc) <= TOL32 and rel_err(whole1, s, sc) <= TOL32


@pytest.mark.parametrize("fmt", FP32_FORMATS)
@pytest.mark.parametrize("m", [64, 96, 512])
def test_fp32_channel_dynamic_range(fmt, m, monkeypatch):
    """Channels spanning 24 decades plus an all-zero pair: the per-channel
    power-of-two operand scale (F16F8) keeps every block of the map accurate
    relative to its OWN magnitude, not only to max|sync|; zero channels give
    exact zeros.  Magnitudes are shared by channel pairs (2k, 2k+1): K1's fp32
    path transforms a pair as one complex FFT, so a channel's error floor is
    ~2^-24 of its partner's magnitude."""
    monkeypatch.setenv("CORR2D_FP32_FORMAT", fmt)
    rng = np.random.default_rng(m)
    n = 300
    v = rng.normal(size=(m, n))
    mag = np.repeat(10.0 ** rng.uniform(-12, 12, size=n // 2), 2)
    v *= mag
    v[:, 6:8] = 0.0
    res = P.correlate_ft(dyn_from_values(v), dtype="float32")
    s, a, _ = O.correlate_ft(v)
    sc = scale_of(s, a)
    assert rel_err(res.sync, s, sc) <= TOL32 and rel_err(res.asyn, a, sc) <= TOL32
    assert not res.sync[7].any() and not res.asyn[7].any()
    # every element against the product of its two channels' own scales
    own = np.sqrt(np.abs(np.diag(s)))
    denom = np.outer(own, own)
    denom[denom == 0] = 1.0
    assert np.max(np.abs(res.sync - s) / denom) <= TOL32
    assert np.max(np.abs(res.asyn - a) / denom) <= TOL32


@pytest.mark.parametrize("fmt", FP32_FORMATS)
def test_fp32_errors_and_edge_inputs(fmt, monkeypatch):
    """The tensor-core path raises the reference's errors (non-finite input,
    zero-variance channel under alpha > 0, through the fast and the generic K1)
    and maps all-zero / constant data to exact zeros; fp32 overflow of the
    planes is reported as a non-finite output, never returned silently."""
    monkeypatch.setenv("CORR2D_FP32_FORMAT", fmt)
    for m in (64, 37):                       # fast K1 (m = 32 R) and generic K1
        v = np.random.default_rng(m).normal(size=(m, 300))
        v[3, 17] = np.inf
        with pytest.raises(P.NumericError, match="non-finite"):
            P.correlate_ft(dyn_from_values(v), dtype="float32")
        raw = np.random.default_rng(m + 1).normal(size=(m, 200)).astype(np.float32)
        raw[:, 5] = 2.5
        ds = P.SpectralDataset(np.arange(200.0), np.arange(float(m)), raw, dtype=np.float32)
        with pytest.raises(P.NumericError, match="zero-variance spectral channel"):
            P.corr2d(ds, alpha=0.5, dtype="float32")
        zero = P.correlate_ft(dyn_from_values(np.zeros((m, 150))), dtype="float32")
        assert not zero.sync.any() and not zero.asyn.any()
        const = P.corr2d(P.SpectralDataset(np.arange(150.0), np.arange(float(m)),
                                           np.full((m, 150), 3.0, np.float32), dtype=np.float32), dtype="float32")
        assert not const.sync.any() and not const.asyn.any()
        big = np.random.default_rng(m + 2).normal(size=(m, 140)) * 1e25
        with pytest.raises(P.NumericError, match="non-finite"):
            P.correlate_ft(dyn_from_values(big), dtype="float32")
