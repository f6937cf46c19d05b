"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports ``corrtwo`` (the reference, /root/reference/pkg/src/corrtwo) and
records inputs + outputs of ``preprocess_dataset``, ``dft_channels`` and
``correlate_ft`` for small seeded cases and for the five BASELINE configs
(config outputs are stored as a fixed sample of rows / a strided sub-grid plus
whole-matrix statistics, so the fixtures stay small).  Nothing at test or
bench time reads /root/reference; tests read these .npz files only.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import corrtwo  # noqa: E402  (the reference)
from corrtwo import (  # noqa: E402
    DynamicSpectra, InterpolantKind, NormalizationSpec, PreprocessSpec, ReferenceSpec,
    ResampleSpec, SpectralDataset, correlate_ft, correlate_ht, dft_channels, preprocess_dataset,
)

from paper_1808_00685_b200 import configs  # noqa: E402  (seeded generators only)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)


def small_cases(manifest):
    rng = np.random.default_rng(20240601)
    # homo random, many m (odd/even, prime, power of two) -- test_fourier.py:238-245, :266-274
    for m, n in [(2, 5), (3, 4), (4, 7), (5, 3), (7, 9), (8, 6), (11, 13), (13, 8), (16, 10),
                 (21, 17), (33, 12), (37, 9), (64, 20), (100, 7), (128, 9), (257, 5), (512, 6)]:
        ds = SpectralDataset(np.linspace(1000.0, 2000.0, n), np.linspace(0.0, 10.0, m),
                             rng.normal(size=(m, n)))
        dyn = preprocess_dataset(ds)
        res = correlate_ft(dyn)
        ws = dft_channels(dyn)
        name = f"homo_m{m}_n{n}"
        save(name, t=ds.perturbation_axis, nu=ds.spectral_axis, raw=ds.intensities,
             values=dyn.values, ref=dyn.reference_used, half=ws.half_spectrum1,
             sync=res.sync, asyn=res.asyn, norm=np.float64(res.normalization))
        manifest[name] = {"kind": "homo", "m": m, "n": n}
    # hetero -- test_fourier.py:331-342
    for m, n1, n2 in [(8, 4, 6), (21, 37, 29), (64, 33, 65)]:
        t = np.linspace(0.0, 5.0, m)
        ds1 = SpectralDataset(np.arange(n1, dtype=float), t, rng.normal(size=(m, n1)))
        ds2 = SpectralDataset(np.arange(n2, dtype=float) + 0.5, t.copy(), rng.normal(size=(m, n2)))
        d1, d2 = preprocess_dataset(ds1), preprocess_dataset(ds2)
        res = correlate_ft(d1, d2)
        name = f"hetero_m{m}_{n1}x{n2}"
        save(name, t=t, nu1=ds1.spectral_axis, nu2=ds2.spectral_axis, raw1=ds1.intensities,
             raw2=ds2.intensities, sync=res.sync, asyn=res.asyn, norm=np.float64(res.normalization))
        manifest[name] = {"kind": "hetero", "m": m, "n1": n1, "n2": n2}
    # preprocessing variants -- test_preprocess.py, test_cross_engine.py:103-118
    variants = [
        ("pre_linear_37to64_a0.5", dict(resample=ResampleSpec(64, InterpolantKind.LINEAR), scaling_exponent=0.5), 37, 23, True),
        ("pre_spline_8to21_a0", dict(resample=ResampleSpec(21, InterpolantKind.CUBIC_SPLINE)), 8, 11, True),
        ("pre_spline_37to64_a1", dict(resample=ResampleSpec(64, InterpolantKind.CUBIC_SPLINE), scaling_exponent=1.0), 37, 15, True),
        ("pre_spline_m2to8", dict(resample=ResampleSpec(8, InterpolantKind.CUBIC_SPLINE)), 2, 5, True),
        ("pre_alpha0.25", dict(scaling_exponent=0.25), 12, 19, False),
        ("pre_alpha1", dict(scaling_exponent=1.0), 9, 14, False),
        ("pre_provided_ref_a0.5", dict(scaling_exponent=0.5, reference="provided"), 10, 13, False),
    ]
    for name, kw, m, n, random_t in variants:
        if random_t:
            t = np.sort(rng.uniform(0.0, 100.0, m))
        else:
            t = np.linspace(0.0, 9.0, m)
        raw = rng.normal(size=(m, n)) + 3.0
        ds = SpectralDataset(np.linspace(10.0, 20.0, n), t, raw)
        provided = None
        if kw.get("reference") == "provided":
            provided = rng.normal(size=n)
            kw = dict(kw, reference=ReferenceSpec.provided(provided))
        spec = PreprocessSpec(**kw)
        dyn = preprocess_dataset(ds, spec)
        res = correlate_ft(dyn)
        arrays = dict(t=t, nu=ds.spectral_axis, raw=raw, t_used=dyn.perturbation_axis,
                      values=dyn.values, ref=dyn.reference_used, sync=res.sync, asyn=res.asyn,
                      norm=np.float64(res.normalization))
        if dyn.sigma is not None:
            arrays["sigma"] = dyn.sigma
        if provided is not None:
            arrays["provided"] = provided
        save(name, **arrays)
        manifest[name] = {"kind": "preprocess", "m_in": m, "n": n,
                          "spec": {k: (str(v) if not isinstance(v, (int, float)) else v) for k, v in kw.items()}}
    # zero-variance substitution (preprocess.py:248-254)
    raw = rng.normal(size=(6, 5))
    raw[:, 2] = 1.25
    ds = SpectralDataset(np.arange(5.0), np.arange(6.0), raw)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        dyn = preprocess_dataset(ds, PreprocessSpec(scaling_exponent=0.5), on_zero_variance="substitute")
    res = correlate_ft(dyn)
    save("pre_zero_variance_substitute", t=ds.perturbation_axis, nu=ds.spectral_axis, raw=raw,
         values=dyn.values, sigma=dyn.sigma, ref=dyn.reference_used, sync=res.sync, asyn=res.asyn)
    manifest["pre_zero_variance_substitute"] = {"kind": "preprocess", "m_in": 6, "n": 5}
    # custom / unit normalisation (engine_core.py:24-72)
    vals = rng.normal(size=(6, 4))
    dyn = DynamicSpectra(np.arange(4.0) + 1.0, np.arange(6.0), vals, np.zeros(4))
    r1 = correlate_ft(dyn, norm=NormalizationSpec.unit())
    r2 = correlate_ft(dyn, norm=NormalizationSpec.custom(0.4))
    save("norm_unit_custom", values=vals, sync_unit=r1.sync, asyn_unit=r1.asyn,
         sync_custom=r2.sync, asyn_custom=r2.asyn)
    manifest["norm_unit_custom"] = {"kind": "norm"}
    # Hilbert route -- hilbert.py:92-115, test_cross_engine.py:26-65
    for m, n1, n2 in [(2, 5, 5), (11, 13, 13), (21, 17, 17), (64, 20, 20), (128, 9, 9),
                      (8, 4, 6), (37, 21, 29)]:
        t = np.linspace(0.0, 7.0, m)
        ds1 = SpectralDataset(np.arange(n1, dtype=float), t, rng.normal(size=(m, n1)))
        homo = n1 == n2
        ds2 = None if homo else SpectralDataset(np.arange(n2, dtype=float) + 0.25, t.copy(),
                                                rng.normal(size=(m, n2)))
        d1 = preprocess_dataset(ds1)
        d2 = None if homo else preprocess_dataset(ds2)
        res = correlate_ht(d1, d2)
        ft = correlate_ft(d1, d2)
        name = f"hilbert_m{m}_{n1}x{n2}"
        save(name, t=t, nu1=ds1.spectral_axis, raw1=ds1.intensities,
             raw2=ds1.intensities if homo else ds2.intensities,
             nu2=ds1.spectral_axis if homo else ds2.spectral_axis,
             values1=d1.values, values2=d1.values if homo else d2.values,
             sync=res.sync, asyn=res.asyn, norm=np.float64(res.normalization),
             ft_sync=ft.sync, ft_norm=np.float64(ft.normalization))
        manifest[name] = {"kind": "hilbert", "m": m, "n1": n1, "n2": n2, "homo": homo}
    # find_peaks -- analysis.py:152-201 on banded data
    from corrtwo import find_peaks
    cases = [("peaks_cfg1_homo", configs.make(1), None, 0.05),
             ("peaks_cfg2_hetero", configs.make(2), "set2", 0.1)]
    for name, case, other, thr in cases:
        s1 = case.set1
        ds1 = SpectralDataset(s1.spectral_axis, s1.perturbation_axis, s1.intensities)
        d1 = preprocess_dataset(ds1)
        d2 = None
        if other:
            s2 = case.set2
            d2 = preprocess_dataset(SpectralDataset(s2.spectral_axis, s2.perturbation_axis, s2.intensities))
        res = correlate_ft(d1, d2)
        rep = find_peaks(res, thr)
        # the maps themselves are not stored: tests rebuild them bit-for-bit with the
        # oracle from the seeded config inputs (pinned by test_oracle_golden.py)
        save(name, threshold=np.float64(thr), eps=np.float64(rep.eps), homo=np.bool_(res.is_homo),
             auto_nu=np.array([p.nu for p in rep.auto_peaks], dtype=float),
             auto_phi=np.array([p.phi for p in rep.auto_peaks], dtype=float),
             cross=np.array([[p.nu1, p.nu2, p.phi, p.psi] for p in rep.cross_peaks], dtype=float).reshape(-1, 4),
             verdicts=np.array([str(p.verdict) for p in rep.cross_peaks]),
             table=np.array(rep.to_table()), long_form=np.frombuffer(rep.to_long_form(), dtype=np.uint8))
        manifest[name] = {"kind": "peaks", "auto": len(rep.auto_peaks), "cross": len(rep.cross_peaks)}
    # serialization -- dataset.py:292-341 byte for byte
    from corrtwo.dataset import write_correlation
    ser = [("ser_homo_m64", "homo_m64_n20", "matrix-pair", ","),
           ("ser_hetero_m21", "hetero_m21_37x29", "matrix-pair", ";"),
           ("ser_long_m11", "homo_m11_n13", "long-form", ",")]
    for name, src, fmt, delim in ser:
        g = np.load(HERE / f"{src}.npz")
        n1, n2 = g["sync"].shape
        t = g["t"]
        ax1 = g["nu"] if "nu" in g else g["nu1"]
        ax2 = g["nu"] if "nu" in g else g["nu2"]
        d1 = DynamicSpectra(ax1, t, np.zeros((t.size, n1)), np.linspace(-1.0, 1.0, n1) / 3.0)
        d2 = DynamicSpectra(ax2, t, np.zeros((t.size, n2)), np.linspace(2.0, 5.0, n2) / 7.0)
        from corrtwo import CorrelationSpectra
        res = CorrelationSpectra(axis1=ax1, axis2=ax2, sync=g["sync"], asyn=g["asyn"], ref1=d1.reference_used,
                                 ref2=d2.reference_used if n1 != n2 or "nu1" in g else d1.reference_used,
                                 normalization=float(g["norm"]), engine="fourier", is_homo="nu" in g,
                                 scaling_exponent=0.0)
        payload = write_correlation(res, fmt, delim)
        save(name, src=np.array(src), fmt=np.array(fmt), delim=np.array(delim),
             ref1=res.ref1, ref2=res.ref2,
             **{k.replace(".", "_"): np.frombuffer(v, dtype=np.uint8) for k, v in payload.items()})
        manifest[name] = {"kind": "serialize", "src": src, "fmt": fmt}


def config_cases(manifest):
    for k in (1, 2, 3, 4, 5):
        case = configs.make(k)
        s1 = case.set1
        ds1 = SpectralDataset(s1.spectral_axis, s1.perturbation_axis, s1.intensities.astype(np.float64))
        spec = PreprocessSpec(
            resample=None if case.resample is None else ResampleSpec(
                case.resample, InterpolantKind.from_name(case.interpolant)),
            scaling_exponent=case.alpha)
        dyn1 = preprocess_dataset(ds1, spec)
        if case.set2 is not None:
            s2 = case.set2
            ds2 = SpectralDataset(s2.spectral_axis, s2.perturbation_axis, s2.intensities)
            dyn2 = preprocess_dataset(ds2, spec)
        else:
            dyn2 = dyn1
        n1, n2 = dyn1.n, dyn2.n
        # fixed sample of output rows (row-block oracle) + strided grid
        rows = np.unique(np.linspace(0, n1 - 1, 12 if n1 <= 2000 else 5).astype(int))
        col_stride = max(1, n2 // 512)
        rr = []
        for r in rows:
            sub = DynamicSpectra(dyn1.spectral_axis[r:r + 1], dyn1.perturbation_axis,
                                 dyn1.values[:, r:r + 1], dyn1.reference_used[r:r + 1],
                                 dyn1.scaling_exponent, None if dyn1.sigma is None else dyn1.sigma[r:r + 1])
            res = correlate_ft(sub, dyn2)
            rr.append((res.sync[0], res.asyn[0]))
        sync_rows = np.stack([a for a, _ in rr])
        asyn_rows = np.stack([b for _, b in rr])
        arrays = dict(rows=rows, sync_rows=sync_rows, asyn_rows=asyn_rows,
                      ref1=dyn1.reference_used, norm=np.float64(1.0 / (np.pi * (dyn1.m - 1))),
                      values_head=dyn1.values[:, :64])
        meta = {"kind": "config", "cfg": k, "m": dyn1.m, "n1": n1, "n2": n2,
                "raw1_sha256": sha(s1.intensities), "dtype": case.dtype}
        if dyn1.sigma is not None:
            arrays["sigma1"] = dyn1.sigma
        if case.set2 is not None:
            arrays["ref2"] = dyn2.reference_used
            meta["raw2_sha256"] = sha(case.set2.intensities)
        if k in (1, 2):  # full result is small enough to summarise exactly
            res = correlate_ft(dyn1, None if case.set2 is None else dyn2)
            arrays["sync_grid"] = res.sync[::7, ::7]
            arrays["asyn_grid"] = res.asyn[::7, ::7]
            arrays["sync_absmax"] = np.float64(np.abs(res.sync).max())
            arrays["asyn_absmax"] = np.float64(np.abs(res.asyn).max())
            arrays["sync_sum"] = np.float64(res.sync.sum())
            arrays["asyn_sum"] = np.float64(res.asyn.sum())
        save(f"config{k}", **arrays)
        manifest[f"config{k}"] = meta
        print("config", k, "done", flush=True)


def main():
    manifest = {"reference": "corrtwo " + corrtwo.__version__,
                "numpy": np.__version__}
    import scipy
    manifest["scipy"] = scipy.__version__
    cases = {}
    small_cases(cases)
    config_cases(cases)
    manifest["cases"] = cases
    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
