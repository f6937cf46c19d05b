"""Golden fixtures for the standalone drop-in functions, made by running the
REFERENCE itself (run in the build container, where it is importable):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_dropin.py

Records, for seeded inputs, the outputs of corrtwo's resample_to_axis /
resample_equidistant (linear and natural spline), mean_reference,
dynamic_spectra (mean and provided reference), stddev_spectrum, apply_scaling
(alpha 0.5 / 1 / 0.25, the zero-variance substitution and its warning), the
CLI's common-axis hetero pipeline (cli.py:313-343: resample both sets onto
linspace(max t0, min t_end, N), preprocess, correlate_ft) and the exception
messages of SpectralDataset / the preprocessing functions
(dataset.py:77-100, preprocess.py:155-259).  Tests read the .npz / .json only.
"""

from __future__ import annotations

import json
import sys
import warnings
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import corrtwo as R  # noqa: E402  (the reference)
from corrtwo.preprocess import (  # noqa: E402
    apply_scaling, dynamic_spectra, mean_reference, resample_equidistant, resample_to_axis, stddev_spectrum,
)


def main():
    rng = np.random.default_rng(808)
    out = {}
    t = np.sort(rng.uniform(0.0, 30.0, 13))
    t[0], t[-1] = 0.0, 30.0
    nu = np.linspace(900.0, 1300.0, 41)
    raw = rng.normal(size=(13, 41)) + 0.5 * np.sin(t)[:, None] + 2.0
    ds = R.SpectralDataset(nu, t, raw)
    out.update(t=t, nu=nu, raw=raw)
    new_axis = np.linspace(1.5, 27.25, 9)
    out["new_axis"] = new_axis
    for kind, tag in ((R.InterpolantKind.LINEAR, "lin"), (R.InterpolantKind.CUBIC_SPLINE, "spl")):
        out[f"to_axis_{tag}"] = resample_to_axis(ds, new_axis, kind).intensities
        eq = resample_equidistant(ds, 16, kind)
        out[f"equi_{tag}"] = eq.intensities
        out[f"equi_axis_{tag}"] = eq.perturbation_axis
    out["mean_ref"] = mean_reference(ds)
    dyn = dynamic_spectra(ds)
    out["dyn_values"] = dyn.values
    prov = rng.normal(size=41) + 2.0
    out["provided_ref"] = prov
    dynp = dynamic_spectra(ds, R.ReferenceSpec.provided(prov))
    out["dyn_values_provided"] = dynp.values
    out["sigma_mean"] = stddev_spectrum(ds)
    out["sigma_provided"] = stddev_spectrum(ds, R.ReferenceSpec.provided(prov))
    for alpha in (0.5, 1.0, 0.25):
        sc = apply_scaling(dyn, out["sigma_mean"], alpha)
        out[f"scaled_{alpha}"] = sc.values
    # zero-variance channel: substitution (with its warning) and the error text
    flat = raw.copy()
    flat[:, 7] = 3.0
    dsf = R.SpectralDataset(nu, t, flat)
    dynf = dynamic_spectra(dsf)
    sig = stddev_spectrum(dsf)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        sub = apply_scaling(dynf, sig, 0.5, on_zero_variance="substitute")
    out["flat_raw"] = flat
    out["flat_sigma"] = sig
    out["flat_scaled_substitute"] = sub.values
    messages = {"substitute_warning": str(w[0].message)}
    try:
        apply_scaling(dynf, sig, 0.5)
    except R.NumericError as e:
        messages["zero_variance_error"] = str(e)
    # the CLI's common-axis hetero pipeline (cli.py:313-343)
    t2 = np.sort(rng.uniform(2.0, 35.0, 11))
    raw2 = rng.normal(size=(11, 29)) - 1.0
    nu2 = np.linspace(0.0, 280.0, 29)
    ds2 = R.SpectralDataset(nu2, t2, raw2)
    lo, hi = max(t[0], t2[0]), min(t[-1], t2[-1])
    axis = np.linspace(lo, hi, 20)
    a1 = resample_to_axis(ds, axis, R.InterpolantKind.LINEAR)
    a2 = resample_to_axis(ds2, axis, R.InterpolantKind.LINEAR)
    d1 = R.preprocess_dataset(a1, R.PreprocessSpec(scaling_exponent=0.5))
    d2 = R.preprocess_dataset(a2, R.PreprocessSpec(scaling_exponent=0.5))
    res = R.correlate_ft(d1, d2)
    out.update(common_t2=t2, common_raw2=raw2, common_nu2=nu2, common_axis=axis, common_sync=res.sync,
               common_asyn=res.asyn, common_norm=np.float64(res.normalization), common_ref1=res.ref1,
               common_ref2=res.ref2)
    # exception messages of the data model and of the preprocessing functions
    cases = {
        "m_lt_2": lambda: R.SpectralDataset(nu, t[:1], raw[:1]),
        "n_lt_2": lambda: R.SpectralDataset(nu[:1], t, raw[:, :1]),
        "shape": lambda: R.SpectralDataset(nu, t, raw[:, :40]),
        "nonfinite_axis": lambda: R.SpectralDataset(np.where(np.arange(41) == 3, np.nan, nu), t, raw),
        "nonfinite_pert": lambda: R.SpectralDataset(nu, np.where(np.arange(13) == 2, np.inf, t), raw),
        "nonfinite_intensity": lambda: R.SpectralDataset(nu, t, np.where(
            (np.arange(13)[:, None] == 4) & (np.arange(41)[None, :] == 6), np.nan, raw)),
        "duplicate_spectral": lambda: R.SpectralDataset(np.concatenate([nu[:5], nu[4:40]]), t, raw),
        "nonmonotonic_spectral": lambda: R.SpectralDataset(np.concatenate([nu[:10], nu[10:][::-1]]), t, raw),
        "pert_not_increasing": lambda: R.SpectralDataset(nu, np.concatenate([t[:6], [t[5] - 1.0], t[7:]]), raw),
        "target_beyond": lambda: resample_to_axis(ds, np.linspace(-1.0, 5.0, 4)),
        "target_count": lambda: resample_equidistant(ds, 3),
        "already_scaled": lambda: apply_scaling(apply_scaling(dyn, out["sigma_mean"], 0.5), out["sigma_mean"], 0.5),
        "alpha_range": lambda: apply_scaling(dyn, out["sigma_mean"], 1.5),
        "sigma_length": lambda: apply_scaling(dyn, out["sigma_mean"][:40], 0.5),
        "provided_length": lambda: dynamic_spectra(ds, R.ReferenceSpec.provided(prov[:40])),
    }
    for name, fn in cases.items():
        try:
            fn()
        except R.CorrtwoError as e:
            messages[name] = [type(e).__name__, str(e)]
        else:
            raise AssertionError(f"{name}: the reference raised nothing")
    np.savez_compressed(HERE / "dropin_functions.npz", **out)
    (HERE / "dropin_messages.json").write_text(json.dumps(messages, indent=1, sort_keys=True))
    print(f"wrote dropin_functions.npz ({len(out)} arrays), dropin_messages.json ({len(messages)} messages)")


if __name__ == "__main__":
    main()
