"""Pin the CPU oracle (oracle/corr2d_oracle.py) against fixtures produced by the
reference package itself (tests/golden/make_golden.py).  CPU only."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, golden, golden_names, rel_err
from oracle import corr2d_oracle as O
from paper_1808_00685_b200 import configs

MANIFEST = json.loads((GOLDEN / "manifest.json").read_text())


@pytest.mark.parametrize("name", golden_names("homo_"))
def test_oracle_homo_bitwise(name):
    g = golden(name)
    t, values, ref, sigma = O.preprocess(g["t"], g["raw"])
    assert np.array_equal(ref, g["ref"])
    assert np.array_equal(values, g["values"])
    half = O.dft_channels(values)
    assert np.array_equal(half, g["half"])
    sync, asyn, c = O.correlate_ft(values)
    assert c == float(g["norm"])
    assert np.array_equal(sync, g["sync"]) and np.array_equal(asyn, g["asyn"])


@pytest.mark.parametrize("name", golden_names("hetero_"))
def test_oracle_hetero_bitwise(name):
    g = golden(name)
    _, v1, _, _ = O.preprocess(g["t"], g["raw1"])
    _, v2, _, _ = O.preprocess(g["t"], g["raw2"])
    sync, asyn, _ = O.correlate_ft(v1, v2)
    assert np.array_equal(sync, g["sync"]) and np.array_equal(asyn, g["asyn"])


@pytest.mark.parametrize("name", golden_names("pre_"))
def test_oracle_preprocess(name):
    g = golden(name)
    spec = MANIFEST["cases"][name].get("spec", {})
    resample = None
    kind = "spline"
    if "resample" in spec:
        txt = spec["resample"]
        resample = int(txt.split("target_count=")[1].split(",")[0])
        kind = "linear" if "LINEAR" in txt else "spline"
    alpha = float(spec.get("scaling_exponent", 0.5 if "zero_variance" in name else 0.0))
    provided = g.get("provided")
    policy = "substitute" if "zero_variance" in name else "error"
    t, values, ref, sigma = O.preprocess(g["t"], g["raw"], resample=resample, kind=kind,
                                         reference=provided, alpha=alpha, on_zero_variance=policy)
    if "t_used" in g:
        assert np.array_equal(t, g["t_used"])
    assert np.array_equal(ref, g["ref"])
    assert np.array_equal(values, g["values"])
    if "sigma" in g:
        assert np.array_equal(sigma, g["sigma"])
    sync, asyn, _ = O.correlate_ft(values)
    assert np.array_equal(sync, g["sync"]) and np.array_equal(asyn, g["asyn"])


def test_oracle_spline_matrix_matches_scipy():
    """The restated natural spline (as a matrix) agrees with scipy's CubicSpline."""
    g = golden("pre_spline_37to64_a1")
    t_new, vals = O.resample_equidistant(g["t"], g["raw"], 64, "spline")
    S = O.natural_spline_matrix(g["t"], t_new)
    assert rel_err(S @ g["raw"], vals) < 1e-12


def test_oracle_norm_variants():
    g = golden("norm_unit_custom")
    s, a, c = O.correlate_ft(g["values"], norm=O.unit_constant(6))
    assert np.array_equal(s, g["sync_unit"]) and np.array_equal(a, g["asyn_unit"])
    s, a, c = O.correlate_ft(g["values"], norm=0.4)
    assert np.array_equal(s, g["sync_custom"]) and np.array_equal(a, g["asyn_custom"])


def test_weights_and_constants():
    for m in (2, 3, 4, 5, 8, 9, 16, 17):
        w = O.half_spectrum_weights(m)
        assert w.size == m // 2 + 1 and w[0] == 1.0
        assert (w[-1] == 1.0) == (m % 2 == 0 or m == 1)
    assert O.noda_constant(6) == pytest.approx(1 / (5 * np.pi), rel=1e-15)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_config_generators_pinned(k):
    """Seeded generators reproduce the inputs the golden rows were made from."""
    import hashlib
    meta = MANIFEST["cases"][f"config{k}"]
    case = configs.make(k)
    assert hashlib.sha256(np.ascontiguousarray(case.set1.intensities).tobytes()).hexdigest() == meta["raw1_sha256"]
    if case.set2 is not None:
        assert hashlib.sha256(np.ascontiguousarray(case.set2.intensities).tobytes()).hexdigest() == meta["raw2_sha256"]


@pytest.mark.parametrize("k", [1, 2, 4])
def test_oracle_config_rows(k):
    """Row-block oracle reproduces the reference's rows bit-for-bit."""
    g = golden(f"config{k}")
    case = configs.make(k)
    t, v1, ref1, sig1 = O.preprocess(case.set1.perturbation_axis, case.set1.intensities,
                                     resample=case.resample, kind=case.interpolant, alpha=case.alpha)
    assert np.array_equal(ref1, g["ref1"])
    v2 = v1
    if case.set2 is not None:
        _, v2, ref2, _ = O.preprocess(case.set2.perturbation_axis, case.set2.intensities)
        assert np.array_equal(ref2, g["ref2"])
    for i, r in enumerate(g["rows"]):
        s, a, _ = O.correlate_ft(v1[:, r:r + 1], v2, rows=None)
        assert np.array_equal(s[0], g["sync_rows"][i])
        assert np.array_equal(a[0], g["asyn_rows"][i])


@pytest.mark.parametrize("name", golden_names("hilbert_"))
def test_oracle_hilbert(name):
    """oracle.correlate_ht against the reference's correlate_ht (hilbert.py:92-115)."""
    g = golden(name)
    sync, asyn, c = O.correlate_ht(g["values1"], g["values2"])
    assert c == float(g["norm"])
    scale = float(np.abs(g["sync"]).max())
    assert rel_err(sync, g["sync"], scale) <= 1e-15
    assert rel_err(asyn, g["asyn"], scale) <= 1e-15
    # the reference's own cross-engine identity (test_cross_engine.py:26-43)
    m = g["values1"].shape[0]
    assert rel_err(g["ft_sync"], (m / np.pi) * g["sync"], scale * m / np.pi) <= 1e-10
