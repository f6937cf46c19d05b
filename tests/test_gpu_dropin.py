"""Drop-in fidelity on the GPU: the reference's dataclass semantics for
DynamicSpectra / CorrelationSpectra (preprocess.py:90-120, dataset.py:111-131),
no stale device copy of ``values`` (the reference re-reads dyn.values on every
call, fourier.py:106), ``device=`` on an explicit device, and streaming with a
budget derived from real free memory (engine.run_streamed)."""

import dataclasses

import numpy as np
import pytest

from oracle import corr2d_oracle as O
import paper_1808_00685_b200 as P

pytestmark = pytest.mark.gpu


def _dyn(values, shift=0.0):
    m, n = values.shape
    return P.DynamicSpectra(np.arange(n, dtype=float) + shift, np.arange(m, dtype=float), values, np.zeros(n))


def _err(res, s, a):
    scale = max(float(np.abs(s).max()), float(np.abs(a).max()))
    return max(float(np.abs(res.sync - s).max()), float(np.abs(res.asyn - a).max())) / scale


@pytest.mark.parametrize("m", [11, 64])
def test_in_place_mutation_of_values_is_honoured(m):
    rng = np.random.default_rng(m)
    v = rng.normal(size=(m, 150))
    dyn = _dyn(v)                          # np.asarray aliases v, as in the reference
    first = P.correlate_ft(dyn)
    v[3] *= -2.0                           # mutate the caller's array in place
    dyn.values[5, 7] = 9.0                 # and the field itself (same array)
    second = P.correlate_ft(dyn)
    s, a, _ = O.correlate_ft(v)
    assert _err(second, s, a) <= 1e-10
    assert not np.array_equal(first.sync, second.sync)
    ws = P.dft_channels(dyn)
    assert np.allclose(ws.half_spectrum1, np.fft.rfft(v, axis=0), rtol=0, atol=1e-12 * np.abs(v).max() * m)


def test_preprocessed_values_then_mutated():
    rng = np.random.default_rng(3)
    ds = P.SpectralDataset(np.arange(200.0), np.arange(16.0), rng.normal(size=(16, 200)) + 1.0)
    dyn = P.preprocess_dataset(ds)          # values live in HBM (K1 output)
    base = P.correlate_ft(dyn)
    vals = dyn.values                        # first host read: host becomes authoritative
    vals[:, 10] = 0.0
    again = P.correlate_ft(dyn)
    s, a, _ = O.correlate_ft(vals)
    assert _err(again, s, a) <= 1e-10
    assert np.all(again.sync[10] == 0) and not np.all(base.sync[10] == 0)
    dyn.values = vals * 2.0                  # reassignment
    third = P.correlate_ft(dyn)
    assert np.allclose(third.sync, 4.0 * again.sync, rtol=1e-12, atol=0)


def test_dataclass_semantics():
    rng = np.random.default_rng(4)
    dyn = _dyn(rng.normal(size=(8, 40)))
    assert [f.name for f in dataclasses.fields(P.DynamicSpectra)] == [
        "spectral_axis", "perturbation_axis", "values", "reference_used", "scaling_exponent", "sigma"]
    d2 = dataclasses.replace(dyn, values=dyn.values[::-1].copy())
    assert not P.is_same_dynamic(dyn, d2)
    res = P.correlate_ft(dyn, d2)
    assert [f.name for f in dataclasses.fields(res)] == [
        "axis1", "axis2", "sync", "asyn", "ref1", "ref2", "normalization", "engine", "is_homo",
        "scaling_exponent"]
    assert set(dataclasses.asdict(res)) >= {"sync", "asyn", "is_homo"}
    again = dataclasses.replace(res, scaling_exponent=0.0)     # re-validates like the reference
    assert np.array_equal(again.sync, res.sync)
    homo = P.correlate_ft(dyn)
    bad = homo.sync.copy()
    bad[0, 1] += 1.0
    with pytest.raises(P.DataError, match="not symmetric"):
        dataclasses.replace(homo, sync=bad)


def test_explicit_device_argument():
    import torch
    rng = np.random.default_rng(7)
    v = rng.normal(size=(21, 300))
    dyn = _dyn(v)
    dev = torch.device("cuda", torch.cuda.current_device())
    r1 = P.correlate_ft(dyn, device=dev)
    r2 = P.correlate_ft(dyn, device=dev.index)
    assert np.array_equal(r1.sync, r2.sync) and np.array_equal(r1.asyn, r2.asyn)
    ds = P.SpectralDataset(np.arange(300.0), np.arange(21.0), v + 3.0)
    r3 = P.corr2d(ds, device=dev)
    s, a, _ = O.correlate_ft(O.preprocess(np.arange(21.0), v + 3.0)[1])
    assert _err(r3, s, a) <= 1e-10


@pytest.mark.slow
def test_streaming_with_budget_from_free_memory():
    """Fill the device so the default budget (85 % of free memory) forces row
    blocks, then run a map through the public call: every block must fit while
    the previous block's plan is released (engine.run_streamed)."""
    import torch
    from paper_1808_00685_b200 import engine
    n = 6000
    rng = np.random.default_rng(8)
    v = rng.normal(size=(40, n))                # m > 32: whole map and blocks take the same kernels
    dyn = _dyn(v)
    whole = P.correlate_ft(dyn)
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    plane_bytes = 2 * 8 * n * n                 # 576 MB
    keep = int(plane_bytes * 0.7)               # room for ~70 % of the map's planes
    filler = torch.empty(max(0, free - keep), dtype=torch.uint8, device="cuda")
    try:
        budget = engine.device_budget(torch.device("cuda", torch.cuda.current_device()))
        blocks = engine.stream_blocks(n, n, 8, budget)
        assert blocks is not None and len(blocks) >= 2
        part = P.correlate_ft(dyn)
    finally:
        del filler
        torch.cuda.empty_cache()
    assert np.array_equal(part.sync, whole.sync) and np.array_equal(part.asyn, whole.asyn)


def test_corr2d_plan_cache_rebinds_every_input():
    """corr2d() reuses a cached plan for repeated shapes (host-returning
    calls): every call must see its own intensities and provided reference."""
    from paper_1808_00685_b200 import api
    rng = np.random.default_rng(12)
    t = np.arange(11.0)
    outs = []
    for k in range(3):
        raw1 = rng.normal(size=(11, 257)) + k
        raw2 = rng.normal(size=(11, 130)) - k
        ref = rng.normal(size=257)
        ds1 = P.SpectralDataset(np.arange(257.0), t, raw1)
        ds2 = P.SpectralDataset(np.arange(130.0), t, raw2)
        homo = P.corr2d(ds1)
        s, a, _ = O.correlate_ft(O.preprocess(t, raw1)[1])
        assert _err(homo, s, a) <= 1e-10
        het = P.corr2d(ds1, ds2)
        s, a, _ = O.correlate_ft(O.preprocess(t, raw1)[1], O.preprocess(t, raw2)[1])
        assert _err(het, s, a) <= 1e-10
        prov = P.corr2d(ds1, reference=ref)
        v = raw1 - ref[None, :]
        s, a, _ = O.correlate_ft(v)
        assert _err(prov, s, a) <= 1e-10 and np.array_equal(prov.ref1, ref)
        outs.append(homo.sync)
    assert len(api._PLAN_CACHE) <= api.PLAN_CACHE_SIZE
    assert not np.array_equal(outs[0], outs[1])      # results never alias the cached planes


def test_standalone_preprocess_functions_match_reference():
    """Every standalone preprocessing function against the outputs the
    reference produced on the same inputs (tests/golden/dropin_functions.npz,
    make_golden_dropin.py): preprocess.py:123-259."""
    import json
    from conftest import GOLDEN, golden
    g = golden("dropin_functions")
    msgs = json.loads((GOLDEN / "dropin_messages.json").read_text())
    ds = P.SpectralDataset(g["nu"], g["t"], g["raw"])
    for kind, tag in ((P.InterpolantKind.LINEAR, "lin"), (P.InterpolantKind.CUBIC_SPLINE, "spl")):
        tol = 0 if tag == "lin" else 1e-12               # linear: the reference's own idx / frac arithmetic
        got = P.resample_to_axis(ds, g["new_axis"], kind)
        assert np.array_equal(got.perturbation_axis, g["new_axis"])
        assert np.max(np.abs(got.intensities - g[f"to_axis_{tag}"])) <= tol * np.abs(g["raw"]).max()
        eq = P.resample_equidistant(ds, 16, kind)
        assert np.array_equal(eq.perturbation_axis, g[f"equi_axis_{tag}"])
        assert np.max(np.abs(eq.intensities - g[f"equi_{tag}"])) <= tol * np.abs(g["raw"]).max()
    assert np.array_equal(P.mean_reference(ds), g["mean_ref"])
    assert np.array_equal(P.dynamic_spectra(ds).values, g["dyn_values"])
    prov = P.ReferenceSpec.provided(g["provided_ref"])
    assert np.array_equal(P.dynamic_spectra(ds, prov).values, g["dyn_values_provided"])
    assert np.allclose(P.stddev_spectrum(ds), g["sigma_mean"], rtol=1e-14, atol=0)
    assert np.allclose(P.stddev_spectrum(ds, prov), g["sigma_provided"], rtol=1e-14, atol=0)
    dyn = P.dynamic_spectra(ds)
    for alpha in (0.5, 1.0, 0.25):
        sc = P.apply_scaling(dyn, g["sigma_mean"], alpha)
        assert sc.scaling_exponent == alpha
        assert np.allclose(sc.values, g[f"scaled_{alpha}"], rtol=1e-14, atol=0)
    dsf = P.SpectralDataset(g["nu"], g["t"], g["flat_raw"])
    dynf = P.dynamic_spectra(dsf)
    sig = P.stddev_spectrum(dsf)
    assert sig[7] == 0.0 and np.allclose(sig, g["flat_sigma"], rtol=1e-14, atol=0)
    with pytest.warns(RuntimeWarning) as w:
        sub = P.apply_scaling(dynf, sig, 0.5, on_zero_variance="substitute")
    assert str(w[0].message) == msgs["substitute_warning"]
    assert np.allclose(sub.values, g["flat_scaled_substitute"], rtol=1e-14, atol=0)
    with pytest.raises(P.NumericError) as e:
        P.apply_scaling(dynf, sig, 0.5)
    assert str(e.value) == msgs["zero_variance_error"]
    with pytest.raises(P.DataError) as e:
        P.resample_to_axis(ds, np.linspace(-1.0, 5.0, 4))
    assert str(e.value) == msgs["target_beyond"][1]


def test_corr2d_resample_to_common_matches_reference_cli_pipeline():
    """corr2d(ds1, ds2, resample_to_common=N) = the reference CLI's common-axis
    pipeline (cli.py:313-343) on the same inputs."""
    from conftest import golden
    g = golden("dropin_functions")
    ds1 = P.SpectralDataset(g["nu"], g["t"], g["raw"])
    ds2 = P.SpectralDataset(g["common_nu2"], g["common_t2"], g["common_raw2"])
    res = P.corr2d(ds1, ds2, resample_to_common=20, interpolant="linear", alpha=0.5)
    s, a = g["common_sync"], g["common_asyn"]
    assert _err(res, s, a) <= 1e-10
    assert res.normalization == float(g["common_norm"]) and not res.is_homo
    assert np.allclose(res.ref1, g["common_ref1"], rtol=1e-14, atol=0)
    assert np.allclose(res.ref2, g["common_ref2"], rtol=1e-14, atol=0)
