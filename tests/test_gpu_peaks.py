"""find_peaks on the GPU against the reference's own
reports (tests/golden/peaks_*.npz): identical peak lists, verdicts, table and
long-form output, for host results and for device-resident results."""

import numpy as np
import pytest

from conftest import golden, golden_names
from oracle import corr2d_oracle as O
import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import configs

pytestmark = pytest.mark.gpu


def _reference_map(name):
    """The reference's correlate_ft map for the fixture's config, rebuilt with
    the oracle (bit-identical to the reference, test_oracle_golden.py)."""
    k = 1 if "cfg1" in name else 2
    case = configs.make(k)
    s1 = case.set1
    _, v1, _, _ = O.preprocess(s1.perturbation_axis, s1.intensities)
    v2, ax2 = None, s1.spectral_axis
    if k == 2:
        _, v2, _, _ = O.preprocess(case.set2.perturbation_axis, case.set2.intensities)
        ax2 = case.set2.spectral_axis
    sync, asyn, _ = O.correlate_ft(v1, v2)
    return P.CorrelationSpectra(axis1=s1.spectral_axis, axis2=ax2, sync=sync, asyn=asyn,
                                ref1=np.zeros(sync.shape[0]), ref2=np.zeros(sync.shape[1]),
                                normalization=1.0, engine="fourier", is_homo=v2 is None)


def _check(rep, g):
    assert np.array_equal([p.nu for p in rep.auto_peaks], g["auto_nu"])
    assert np.array_equal([p.phi for p in rep.auto_peaks], g["auto_phi"])
    cross = np.array([[p.nu1, p.nu2, p.phi, p.psi] for p in rep.cross_peaks], dtype=float).reshape(-1, 4)
    assert np.array_equal(cross, g["cross"])
    assert [str(p.verdict) for p in rep.cross_peaks] == list(g["verdicts"])
    assert rep.eps == float(g["eps"])
    assert rep.to_table() == str(g["table"])
    assert rep.to_long_form() == g["long_form"].tobytes()


@pytest.mark.parametrize("name", golden_names("peaks_"))
def test_find_peaks_matches_reference_on_reference_maps(name):
    g = golden(name)
    rep = P.find_peaks(_reference_map(name), float(g["threshold"]))
    _check(rep, g)


def test_find_peaks_on_device_result_cfg1():
    """The GPU-computed cfg1 map, left in HBM: same peaks as the reference found
    on its own map (cfg1 is fp64 and within 1e-10, far from any tie)."""
    g = golden("peaks_cfg1_homo")
    case = configs.make(1)
    s1 = case.set1
    ds = P.SpectralDataset(s1.spectral_axis, s1.perturbation_axis, s1.intensities)
    dev = P.corr2d(ds, return_device=True)
    rep = P.find_peaks(dev, float(g["threshold"]))
    assert [p.nu for p in rep.auto_peaks] == list(g["auto_nu"])
    got = np.array([[p.nu1, p.nu2] for p in rep.cross_peaks]).reshape(-1, 2)
    assert np.array_equal(got, g["cross"][:, :2])
    assert [str(p.verdict) for p in rep.cross_peaks] == list(g["verdicts"])
    scale = float(np.abs(_reference_map("cfg1").sync).max())
    vals = np.array([[p.phi, p.psi] for p in rep.cross_peaks]).reshape(-1, 2)
    assert np.abs(vals - g["cross"][:, 2:]).max() <= 1e-10 * scale


def test_find_peaks_edge_cases():
    axis = np.linspace(0.0, 4.0, 5)
    sync = np.zeros((5, 5))
    sync[2, 2] = 5.0
    res = P.CorrelationSpectra(axis1=axis, axis2=axis, sync=sync, asyn=np.zeros((5, 5)), ref1=np.zeros(5),
                               ref2=np.zeros(5), normalization=1.0, engine="fourier", is_homo=True)
    rep = P.find_peaks(res)
    assert [(p.nu, p.phi) for p in rep.auto_peaks] == [(2.0, 5.0)]
    assert rep.cross_peaks == []                       # (2, 2) is not in the strict upper triangle
    zero = P.CorrelationSpectra(axis1=axis, axis2=axis, sync=np.zeros((5, 5)), asyn=np.zeros((5, 5)),
                                ref1=np.zeros(5), ref2=np.zeros(5), normalization=1.0, engine="fourier",
                                is_homo=True)
    rep = P.find_peaks(zero)
    assert rep.auto_peaks == [] and rep.cross_peaks == []
    with pytest.raises(P.DataError, match="threshold_fraction"):
        P.find_peaks(res, 1.5)
    # plateaus are not strict maxima; a lone corner maximum is (-inf padding)
    s = np.zeros((6, 6))
    s[0, 5] = 3.0
    s[1, 3] = s[1, 4] = 2.0
    a = np.zeros((6, 6))
    res = P.CorrelationSpectra(axis1=np.arange(6.0), axis2=np.arange(6.0), sync=s + s.T, asyn=a,
                               ref1=np.zeros(6), ref2=np.zeros(6), normalization=1.0, engine="fourier",
                               is_homo=True)
    rep = P.find_peaks(res, 0.1)
    assert [(p.nu1, p.nu2) for p in rep.cross_peaks] == [(0.0, 5.0)]
