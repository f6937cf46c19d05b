"""One small invocation of every libcorr2d kernel, for compute-sanitizer
(memcheck / racecheck / synccheck).  Run as

    compute-sanitizer --tool memcheck --target-processes all python tools/sanitize.py [which]

`which` selects a subset (all, small, f64, tc, prep, peaks, hilbert); shapes are
ragged on purpose (partial tiles, odd m, hetero).  Not part of the product."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_00685_b200 as P  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(0)


def dyn(v, shift=0.0):
    m, n = v.shape
    return P.DynamicSpectra(np.arange(n, dtype=float) + shift, np.arange(m, dtype=float), v, np.zeros(n))


def run(name, fn):
    if which not in ("all", name):
        return
    fn()
    print(f"sanitize: {name} ok", flush=True)


def small():
    # one-kernel small-m path: homo + hetero, ragged blocks, f32 input, alpha
    v1, v2 = rng.normal(size=(11, 150)), rng.normal(size=(11, 97))
    P.correlate_ft(dyn(v1))
    P.correlate_ft(dyn(v1), dyn(v2, 0.5))
    ds = P.SpectralDataset(np.arange(130.0), np.arange(21.0), rng.normal(size=(21, 130)).astype(np.float32),
                           dtype=np.float32)
    P.corr2d(ds, alpha=0.5)
    P.corr2d(P.SpectralDataset(np.arange(70.0), np.arange(32.0), rng.normal(size=(32, 70))))


def f64():
    v1, v2 = rng.normal(size=(64, 200)), rng.normal(size=(64, 77))
    P.correlate_ft(dyn(v1))                           # Gauss contraction, homo (diag / mirror / ragged tiles)
    P.correlate_ft(dyn(v1), dyn(v2, 0.5))
    P.correlate_ft(dyn(v1), rows=(64, 192), return_device=True)
    os.environ["CORR2D_F64_FORMAT"] = "four"
    P.correlate_ft(dyn(v1))
    del os.environ["CORR2D_F64_FORMAT"]


def tc():
    v = rng.normal(size=(64, 300))
    P.correlate_ft(dyn(v), dtype="float32")           # CTA-pair kernel
    P.correlate_ft(dyn(v), dyn(rng.normal(size=(64, 130)), 0.5), dtype="float32")
    P.correlate_ft(dyn(v), dtype="float32", rows=(128, 256), return_device=True)   # 1-SM kernel
    os.environ["CORR2D_FP32_FORMAT"] = "bf16x3"
    P.correlate_ft(dyn(v), dtype="float32")
    del os.environ["CORR2D_FP32_FORMAT"]


def prep():
    t = np.sort(rng.uniform(0, 10, 37))
    ds = P.SpectralDataset(np.arange(250.0), t, rng.normal(size=(37, 250)) + 1.0)
    P.preprocess_dataset(ds, P.PreprocessSpec(resample=P.ResampleSpec(64, P.InterpolantKind.LINEAR),
                                              scaling_exponent=0.5))
    P.corr2d(ds, resample=40, interpolant="spline")
    P.dft_channels(dyn(rng.normal(size=(45, 90))))
    P.corr2d(P.SpectralDataset(np.arange(300.0), np.arange(512.0), rng.normal(size=(512, 300)).astype(np.float32),
                               dtype=np.float32), dtype="float32")


def peaks():
    v = rng.normal(size=(16, 180))
    res = P.correlate_ft(dyn(v))
    P.find_peaks(res, 0.2)


def hilbert():
    v = rng.normal(size=(20, 140))
    P.correlate_ht(dyn(v))
    P.correlate_ht(dyn(v), dyn(rng.normal(size=(20, 60)), 0.5))


for name, fn in (("small", small), ("f64", f64), ("tc", tc), ("prep", prep), ("peaks", peaks),
                 ("hilbert", hilbert)):
    run(name, fn)
print("sanitize: done")
