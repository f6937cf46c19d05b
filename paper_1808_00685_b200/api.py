"""``corr2d()`` -- the one-call pipeline of the paper's R function, mirroring the
reference CLI's correlate pipeline (cli.py:299-343): optional resampling of two
datasets onto a common axis (:313-321) -> preprocess each with one spec
(:323-330) -> Fourier-route correlation (:332-344).

GPU execution is fused: each raw dataset goes through ONE K1 launch
(resample -> reference -> sigma -> scale -> DFT -> operand packing), the
dynamic values are never materialised, then ONE K2 launch writes the planes.
"""

from __future__ import annotations

import numpy as np

from . import _abi, engine
from . import engine as _engine_mod
from .dataset import CorrelationSpectra, SpectralDataset
from .engine_core import NormalizationSpec
from .errors import DataError, NumericError
from .fourier import DeviceCorrelationSpectra
from .preprocess import (InterpolantKind, PreprocessSpec, ReferenceSpec, ResampleSpec,
                         resample_to_axis)


def _reference_spec(reference) -> ReferenceSpec:
    if reference is None or (isinstance(reference, str) and reference == "mean"):
        return ReferenceSpec.mean()
    if isinstance(reference, ReferenceSpec):
        return reference
    if isinstance(reference, str):
        raise DataError(f"unknown reference {reference!r} (use 'mean' or a vector)")
    return ReferenceSpec.provided(reference)


def _norm_spec(norm, engine_name="fourier") -> NormalizationSpec:
    if norm is None:  # cli.py:334-340: noda for the Fourier route, unit for Hilbert
        return NormalizationSpec.noda() if engine_name == "fourier" else NormalizationSpec.unit()
    if isinstance(norm, NormalizationSpec):
        return norm
    if isinstance(norm, str):
        return NormalizationSpec.parse(norm)
    return NormalizationSpec.custom(float(norm))


def build_plan(ds1: SpectralDataset, ds2: SpectralDataset | None, spec: PreprocessSpec, *,
               norm=None, on_zero_variance="error", dtype="float64", rows=None, device=None,
               engine_name="fourier", distributed=None):
    """A bound :class:`engine.CorrelationPlan` for the fused raw -> planes pipeline."""
    from .preprocess import _raw_device, _recipe_for
    _, dev = engine.require_device(device)
    homo = ds2 is None or ds2 is ds1 or ds1.equals(ds2)
    r1, plan1 = _recipe_for(ds1, spec, on_zero_variance, dev)
    r2 = None
    if not homo:
        r2, plan2 = _recipe_for(ds2, spec, on_zero_variance, dev)
        t1 = plan1.t_new if plan1 is not None else ds1.perturbation_axis
        t2 = plan2.t_new if plan2 is not None else ds2.perturbation_axis
        if not np.array_equal(t1, t2):
            raise DataError("perturbation axes differ between the two inputs; resample both "
                            "onto a common axis before correlating")
    m = r1.m
    if engine_name not in ("fourier", "hilbert"):
        raise DataError(f"unknown engine {engine_name!r} (use 'fourier' or 'hilbert')")
    constant = _norm_spec(norm, engine_name).constant(m)
    if distributed is not None:
        # one band of a multi-GPU map (sharded.py); distributed = dict(group=, spectra=)
        from .sharded import ShardedCorrelationPlan
        if engine_name != "fourier":
            raise DataError("distributed=True supports the Fourier route")
        plan = ShardedCorrelationPlan(n1=ds1.n, n2=(ds1 if homo else ds2).n, m=m, recipe1=r1, recipe2=r2,
                                      norm=constant, dtype=dtype, device=dev, **distributed)
        plan.bind(_raw_device(ds1, dev), None if homo else _raw_device(ds2, dev))
        plan.constant = constant
        plan.t_axis = plan1.t_new if plan1 is not None else ds1.perturbation_axis
        return plan, homo
    plan = engine.CorrelationPlan(
        n1=ds1.n, n2=(ds1 if homo else ds2).n, m=m, recipe1=r1, recipe2=r2, norm=constant,
        dtype=dtype, rows=rows, device=dev, want_ref=True, want_sigma=r1.alpha > 0.0,
        route=engine_name)
    plan.bind(_raw_device(ds1, dev), None if homo else _raw_device(ds2, dev))
    plan.constant = constant
    plan.t_axis = plan1.t_new if plan1 is not None else ds1.perturbation_axis
    return plan, homo


_PLAN_CACHE: "OrderedDict[tuple, object]" = None
PLAN_CACHE_SIZE = 2                    # plans kept per process (LRU)
PLAN_CACHE_MAX_BYTES = 1 << 30         # only maps whose two planes fit in 1 GB are kept


def _axis_key(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return (a.size, hash(a.tobytes()))


def _cached_plan(ds1, ds2, spec, *, norm, on_zero_variance, dtype, device, engine_name):
    """A bound plan for a host-returning corr2d() call, reused across calls of
    the same shape / recipe (its device buffers and launch configuration),
    rebound to this call's inputs.  Maps larger than PLAN_CACHE_MAX_BYTES are
    never kept.  Results never alias a cached plan: the planes are copied out
    before the call returns."""
    global _PLAN_CACHE
    from collections import OrderedDict

    from .preprocess import _raw_device
    if _PLAN_CACHE is None:
        _PLAN_CACHE = OrderedDict()
    _, dev = engine.require_device(device)
    homo = ds2 is None or ds2 is ds1 or ds1.equals(ds2)
    dsb = ds1 if homo else ds2
    odt = np.dtype(dtype)
    if 2 * ds1.n * dsb.n * odt.itemsize > PLAN_CACHE_MAX_BYTES:
        return build_plan(ds1, ds2, spec, norm=norm, on_zero_variance=on_zero_variance, dtype=dtype,
                          device=device, engine_name=engine_name)
    nkey = norm if isinstance(norm, (str, float, int, type(None))) else (norm.kind, norm.value)
    rs = spec.resample
    key = (str(dev), dtype, engine_name, on_zero_variance, nkey, spec.reference.kind, float(spec.scaling_exponent),
           None if rs is None else (rs.target_count, rs.interpolant.value), homo,
           ds1.n, ds1.intensities.dtype.str, _axis_key(ds1.perturbation_axis),
           None if homo else (ds2.n, ds2.intensities.dtype.str, _axis_key(ds2.perturbation_axis)),
           engine.f64_pack_kind() if odt == np.float64 else engine.fp32_pack_kind(),
           engine.small_fused_enabled())
    hit = _PLAN_CACHE.get(key)
    if hit is None:
        plan, homo = build_plan(ds1, ds2, spec, norm=norm, on_zero_variance=on_zero_variance, dtype=dtype,
                                device=device, engine_name=engine_name)
        _PLAN_CACHE[key] = plan
        while len(_PLAN_CACHE) > PLAN_CACHE_SIZE:
            _PLAN_CACHE.popitem(last=False)
        return plan, homo
    _PLAN_CACHE.move_to_end(key)
    plan = hit
    if spec.reference.kind == "provided":            # this call's reference vector
        spec.reference.check_length(ds1.n)
        plan.recipe1.ref_in = engine.to_device(spec.reference.spectrum, dev)
        if plan.recipe2 is not None:
            spec.reference.check_length(ds2.n)
            plan.recipe2.ref_in = plan.recipe1.ref_in
    plan.bind(_raw_device(ds1, dev), None if homo else _raw_device(ds2, dev))
    return plan, homo


@engine.on_device
def corr2d(ds1: SpectralDataset, ds2: SpectralDataset | None = None, *, reference="mean",
           resample: int | None = None, resample_to_common: int | None = None,
           interpolant: str = "spline", alpha: float = 0.0, norm=None, workers: int = 1,
           on_zero_variance: str = "error", dtype="float64", out=None,
           return_device: bool = False, device=None, engine: str = "fourier",
           distributed: bool = False, group=None, spectra: str = "broadcast") -> CorrelationSpectra:
    """Generalised 2D correlation of one (homo) or two (hetero) spectral series.

    Keyword arguments follow the reference CLI (`corrtwo correlate`): reference
    ("mean" or a vector), resample (target count), resample_to_common,
    interpolant ("spline" | "linear"), alpha (scaling exponent), norm
    (NormalizationSpec, "noda" | "unit" | "custom:c", or a float; default noda
    for the Fourier route, unit for the Hilbert route), engine ("fourier" |
    "hilbert", cli.py:332-344; the Hilbert route computes in float64).

    ``distributed=True`` (one process per GPU, torch.distributed initialised,
    e.g. under torchrun): every rank calls ``corr2d`` with the same inputs and
    gets a :class:`~.sharded.ShardedCorrelationSpectra` holding ITS band of
    the map in HBM (``.gather(root)`` assembles the whole map on one rank);
    ``group`` selects the process group, ``spectra`` the K1 scheme
    ("broadcast": each rank transforms its chunk, owners NCCL-broadcast;
    "recompute": every rank transforms every channel).
    """
    if workers < 1:
        raise DataError("correlate: --workers must be >= 1")
    kind = InterpolantKind.from_name(interpolant)
    if resample_to_common is not None and ds2 is not None:
        lo = max(ds1.perturbation_axis[0], ds2.perturbation_axis[0])
        hi = min(ds1.perturbation_axis[-1], ds2.perturbation_axis[-1])
        if not lo < hi:
            raise DataError("preprocess: perturbation ranges do not overlap")
        axis = np.linspace(lo, hi, int(resample_to_common))
        ds1 = resample_to_axis(ds1, axis, kind)
        ds2 = resample_to_axis(ds2, axis, kind)
    spec = PreprocessSpec(reference=_reference_spec(reference),
                          resample=None if resample is None else ResampleSpec(int(resample), kind),
                          scaling_exponent=float(alpha))
    homo = ds2 is None or ds2 is ds1 or ds1.equals(ds2)
    dsb = ds1 if homo else ds2
    if distributed:
        from . import sharded
        plan, homo = build_plan(ds1, ds2, spec, norm=norm, on_zero_variance=on_zero_variance, dtype=dtype,
                                device=device, engine_name=engine,
                                distributed=dict(group=group, spectra=spectra))
        meta = dict(axis1=ds1.spectral_axis, axis2=dsb.spectral_axis, normalization=plan.constant,
                    engine=engine, is_homo=homo, scaling_exponent=float(alpha) if alpha > 0 else 0.0)
        return sharded.run(plan, meta, axes=(ds1.spectral_axis, dsb.spectral_axis))
    blocks = None
    plan = None
    if not return_device:
        _, dev = _engine_mod.require_device(device)
        odt = np.dtype(dtype)
        blocks = _engine_mod.maybe_stream_blocks(ds1.n, dsb.n, odt.itemsize, dev)
        if blocks is None:
            try:
                plan, homo = _cached_plan(ds1, ds2, spec, norm=norm, on_zero_variance=on_zero_variance,
                                          dtype=dtype, device=device, engine_name=engine)
            except NumericError as e:            # the device is fuller than the size check assumed
                if "out of memory" not in str(e):
                    raise
                blocks = _engine_mod.stream_blocks(ds1.n, dsb.n, odt.itemsize, _engine_mod.device_budget(dev))
        if blocks is not None:        # planes larger than device memory: stream row blocks
            def make_plan(rws):
                return build_plan(ds1, ds2, spec, norm=norm, on_zero_variance=on_zero_variance, dtype=dtype,
                                  device=device, engine_name=engine, rows=rws)[0]
            s, a, info, first = _engine_mod.run_streamed(
                make_plan, ds1.n, dsb.n, odt, blocks, out,
                check=lambda pl: pl.check(axes=(ds1.spectral_axis, dsb.spectral_axis), labels=("first", "second")))
            constant = _norm_spec(norm, engine).constant(spec.resample.target_count if spec.resample
                                                         else ds1.perturbation_axis.size)
            return CorrelationSpectra._trusted(
                sync=s, asyn=a, axis1=ds1.spectral_axis, axis2=dsb.spectral_axis, ref1=first[0], ref2=first[1],
                normalization=constant, engine=engine, is_homo=homo,
                scaling_exponent=float(alpha) if alpha > 0 else 0.0, stats=info)
    if not return_device:
        # planes' D2H queued right behind the kernels; status checks overlap it
        s, a, (ref1, ref2, _, _, info) = plan.run_to_host(out, axes=(ds1.spectral_axis, dsb.spectral_axis))
        return CorrelationSpectra._trusted(
            sync=s, asyn=a, axis1=ds1.spectral_axis, axis2=dsb.spectral_axis, ref1=ref1, ref2=ref2,
            normalization=plan.constant, engine=engine, is_homo=homo,
            scaling_exponent=float(alpha) if alpha > 0 else 0.0, stats=info)
    plan, homo = build_plan(ds1, ds2, spec, norm=norm, on_zero_variance=on_zero_variance,
                            dtype=dtype, device=device, engine_name=engine)
    plan.launch()
    _engine_mod.sync()
    ref1, ref2, _, _, info = plan.check(axes=(ds1.spectral_axis, dsb.spectral_axis),
                                        labels=("first", "second"))
    meta = dict(axis1=ds1.spectral_axis, axis2=dsb.spectral_axis, ref1=ref1, ref2=ref2,
                normalization=plan.constant, engine=engine, is_homo=homo,
                scaling_exponent=float(alpha) if alpha > 0 else 0.0, stats=info)
    if return_device:
        return DeviceCorrelationSpectra(plan, meta)
    s, a = plan.fetch(out)
    return CorrelationSpectra._trusted(sync=s, asyn=a, **meta)
