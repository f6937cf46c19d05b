"""Out-of-bounds guards for every kernel family (compute-sanitizer is not
available on this pool, so the memory-safety evidence is built in): each
device buffer a kernel touches is placed inside an allocation whose guard
bands -- 4 KiB before and after, plus the pad columns of every padded row
(ld > row length) -- are filled with 0xFF bytes, a NaN in every format the
kernels read (f64, f32, fp16 / bf16, e4m3).

After the launch:
* every guard byte must still be 0xFF (no stray store, row overrun or mirror
  write outside the row band);
* the results inside must be BIT-identical to the same plan run on buffers of
  the same geometry with zero-filled surroundings (same kernel variants; a
  stray READ of a guard would bring a NaN in, or trip the non-finite input /
  output checks).

Shapes are ragged (no multiple of any tile size), inputs are padded views
(ld_raw > n), outputs use ld_out > n2 both 16-byte aligned (vector / TMA
stores) and odd (scalar fallbacks)."""

import numpy as np
import pytest

import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import api, engine, _abi

pytestmark = pytest.mark.gpu

GUARD = 4096
FILL = 0xFF


class Guarded:
    """A rows x cols view (row pitch cols + pad) inside a 0xFF-filled allocation."""

    def __init__(self, like, pad=0, zero=False, copy=None, fill=FILL):
        import torch
        self.shape = tuple(like.shape)
        rows, cols = (self.shape[0], self.shape[1]) if like.dim() == 2 else (1, self.shape[0])
        es = like.element_size()
        self.ld = cols + pad
        self.body = rows * self.ld * es
        self.fill = fill
        self.buf = torch.full((GUARD + self.body + GUARD,), fill, dtype=torch.uint8, device=like.device)
        flat = self.buf[GUARD:GUARD + self.body].view(like.dtype).view(rows, self.ld)
        self.view = flat[:, :cols] if like.dim() == 2 else flat[0, :cols]
        self.rows, self.cols, self.es = rows, cols, es
        if zero:
            self.view.zero_()
        if copy is not None:
            self.view.copy_(copy)

    def intact(self):
        """Every guard byte still 0xFF."""
        b = self.buf
        ok = bool((b[:GUARD] == self.fill).all()) and bool((b[GUARD + self.body:] == self.fill).all())
        if self.ld > self.cols:
            rows = b[GUARD:GUARD + self.body].view(self.rows, self.ld * self.es)
            ok = ok and bool((rows[:, self.cols * self.es:] == self.fill).all())
        return ok


def _dataset(n, m, seed, dtype=np.float64):
    rng = np.random.default_rng(seed)
    t = np.linspace(0.0, 1.0, m)
    v = rng.normal(size=(m, n)) + np.sin(np.outer(7 * t, np.arange(n) / n))
    return P.SpectralDataset(np.arange(float(n)), t, v.astype(dtype), dtype=dtype)


def _plan(ds1, ds2, dtype, engine_name="fourier", rows=None, spec=None):
    plan, _ = api.build_plan(ds1, ds2, spec or P.PreprocessSpec(), dtype=dtype, rows=rows,
                             engine_name=engine_name)
    return plan


def _results(plan):
    import torch
    plan.launch()
    torch.cuda.synchronize()
    plan.check()
    out = {"phi": plan.phi.clone(), "psi": plan.psi.clone(), "ref1": plan.ref1.clone(),
           "stats": plan.stats.clone()}
    if plan.ref2 is not None:
        out["ref2"] = plan.ref2.clone()
    return out


def _guard_plan(plan, out_pad, raw_pad, fill):
    """Move every buffer of `plan` into guarded allocations; returns the guards."""
    g = {}
    shared_b = plan.b_homo is not None and plan.b_homo is plan.a_phi   # tensor-core homo: one array
    for name in ("a_phi", "a_psi", "b", "b_homo", "noda_scratch", "ref1", "ref2", "sigma1", "sigma2"):
        t = getattr(plan, name, None)
        if t is None:
            continue
        if name == "b_homo" and shared_b:
            plan.b_homo = g["a_phi"].view
            continue
        # a_psi of the Hilbert route must keep its zero padding columns
        g[name] = Guarded(t, copy=t if name == "a_psi" else None, fill=fill)
        setattr(plan, name, g[name].view)
    for name in ("stats", "status1", "status2", "work"):
        t = getattr(plan, name, None)
        if t is not None:
            g[name] = Guarded(t, zero=True, fill=fill)
            setattr(plan, name, g[name].view)
    for name in ("phi", "psi"):
        t = getattr(plan, name)
        g[name] = Guarded(t, pad=out_pad, fill=fill)
        setattr(plan, name, g[name].view)
    raws = [plan.raw1, plan.raw2]
    for i, r in enumerate(raws):
        if r is not None:
            g[f"raw{i + 1}"] = Guarded(r, pad=raw_pad, copy=r, fill=fill)
    plan.bind(g["raw1"].view, g["raw2"].view if "raw2" in g else None)
    return g


def _run_guarded(make, out_pad, raw_pad=3):
    """The same plan twice with the same buffer geometry (so the same kernel
    variants run): zero-filled surroundings, then 0xFF (NaN) guards."""
    import torch
    plan = make()
    _guard_plan(plan, out_pad, raw_pad, 0)
    ref = _results(plan)
    plan = make()
    g = _guard_plan(plan, out_pad, raw_pad, FILL)
    got = _results(plan)
    bad = [k for k, v in g.items() if not v.intact()]
    assert not bad, f"guard bytes overwritten in {bad}"
    for k, v in ref.items():
        assert torch.equal(v.view(torch.uint8) if v.dtype != torch.int64 else v,
                           got[k].view(torch.uint8) if got[k].dtype != torch.int64 else got[k]), k
    return plan


CASES = [
    # (label, n1, n2 or None, m, dtype, fp32 format, f64 format, engine)
    ("f64-gauss-fastK1", 1000, None, 64, "float64", None, "gauss", "fourier"),
    ("f64-four-genericK1", 777, None, 100, "float64", None, "four", "fourier"),
    ("f64-gauss-hetero", 515, 301, 64, "float64", None, "gauss", "fourier"),
    ("f64-gauss-hetero-wide", 130, 1100, 200, "float64", None, "gauss", "fourier"),
    ("f32-f16f8-fastK1", 1000, None, 64, "float32", "f16f8", None, "fourier"),
    ("f32-bf16x3", 600, None, 128, "float32", "bf16x3", None, "fourier"),
    ("f32-f16f8-hetero", 300, 1100, 512, "float32", "f16f8", None, "fourier"),
    ("f32-f16f8-genericK1", 300, None, 1000, "float32", "f16f8", None, "fourier"),
    ("hilbert", 300, None, 50, "float64", None, None, "hilbert"),
    ("small-homo", 500, None, 16, "float64", None, None, "fourier"),
    ("small-hetero", 200, 333, 31, "float64", None, None, "fourier"),
    # the one-kernel variant (no operand scratch: CORR2D_SMALL_ONEKERNEL=1)
    ("small-1k-homo", 500, None, 16, "float64", None, None, "fourier"),
    ("small-1k-hetero", 200, 333, 31, "float64", None, None, "fourier"),
    # more 64 x 64 blocks than SMs: K1 + the streamed (persistent, TMA-store) contraction
    ("small-stream-homo", 1100, None, 21, "float64", None, None, "fourier"),
    ("small-stream-homo-1slot", 1090, None, 32, "float64", None, None, "fourier"),
    ("small-stream-hetero", 1000, 1023, 11, "float64", None, None, "fourier"),
]


@pytest.mark.parametrize("out_pad", [4, 1])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_guard_bands_intact_and_results_bit_identical(case, out_pad, monkeypatch):
    label, n1, n2, m, dtype, f32fmt, f64fmt, eng = case
    if f32fmt:
        monkeypatch.setenv("CORR2D_FP32_FORMAT", f32fmt)
    if f64fmt:
        monkeypatch.setenv("CORR2D_F64_FORMAT", f64fmt)
    if "-1k-" in label:
        monkeypatch.setenv("CORR2D_SMALL_ONEKERNEL", "1")
    ds1 = _dataset(n1, m, 1)
    ds2 = _dataset(n2, m, 2) if n2 else None
    plan = _run_guarded(lambda: _plan(ds1, ds2, dtype, eng), out_pad)
    if label.startswith("small"):
        assert plan.small
    elif eng == "fourier":
        assert not plan.small


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_guard_bands_row_band(dtype):
    """A row band [128, 640) of a homo map: the mirrored (transposed) stores
    must stay inside the band's rows."""
    ds = _dataset(1000, 64, 3)
    _run_guarded(lambda: _plan(ds, None, dtype, rows=(128, 640)), 2)


def test_guard_bands_resampled_input():
    ds = _dataset(411, 90, 4)
    spec = P.PreprocessSpec(resample=P.ResampleSpec(64, P.InterpolantKind.LINEAR), scaling_exponent=0.5)
    _run_guarded(lambda: _plan(ds, None, "float64", spec=spec), 2)


def test_find_peaks_index_buffer_guarded():
    """corr2d_find_peaks with more candidates than capacity: the index buffer's
    guard stays intact and the count reports every candidate."""
    import torch
    lib, dev = engine.require_device(None)
    n = 300
    g = torch.Generator(device="cpu").manual_seed(5)
    s = torch.randn(n, n, generator=g, dtype=torch.float64)
    s = (s + s.T).to(dev)
    a = torch.randn(n, n, generator=g, dtype=torch.float64)
    a = (a - a.T).to(dev)
    cap = 17
    idx = Guarded(torch.empty(cap, dtype=torch.int64, device=dev))
    count = Guarded(torch.zeros(1, dtype=torch.int64, device=dev), zero=True)
    code = lib.corr2d_find_peaks(_abi.F64, engine.ptr(s), engine.ptr(a), n, n, n, 1, 0.5, 0.5,
                                 engine.ptr(idx.view), cap, engine.ptr(count.view), engine.stream_handle())
    _abi.check(code, lib)
    torch.cuda.synchronize()
    assert idx.intact() and count.intact()
    assert int(count.view[0]) > cap
