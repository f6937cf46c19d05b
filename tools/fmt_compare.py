"""Accuracy and K2 time of the two float32 operand formats (bf16x3, f16f8)
against the fp64 DMMA planes of the same plan (tools only, GPU box).

usage: python tools/fmt_compare.py [config ...]     (default: 5 1 2 4)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import api, configs, engine


def planes(case, dtype, fmt=None):
    if fmt:
        os.environ["CORR2D_FP32_FORMAT"] = fmt
    dt = np.float32 if case.dtype == "float32" else np.float64
    s1 = case.set1
    ds1 = P.SpectralDataset(s1.spectral_axis, s1.perturbation_axis, s1.intensities, dtype=dt)
    ds2 = None
    if case.set2 is not None:
        ds2 = P.SpectralDataset(case.set2.spectral_axis, case.set2.perturbation_axis, case.set2.intensities, dtype=dt)
    spec = P.PreprocessSpec(
        resample=None if case.resample is None else P.ResampleSpec(case.resample, P.InterpolantKind.from_name(case.interpolant)),
        scaling_exponent=case.alpha)
    plan, _ = api.build_plan(ds1, ds2, spec, dtype=dtype)
    plan.launch_prep_only()
    plan.launch_contract()
    torch.cuda.synchronize()
    ms = None
    if dtype == "float32":
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        plan.launch_contract()
        e0.record()
        for _ in range(5):
            plan.launch_contract()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
    return plan, ms


def main():
    cfgs = [int(c) for c in sys.argv[1:]] or [5, 1, 2, 4]
    for c in cfgs:
        case = configs.make(c)
        ref, _ = planes(case, "float64")
        rphi, rpsi = ref.phi, ref.psi
        sphi, spsi = rphi.abs().max().item(), rpsi.abs().max().item()
        out = {"config": c, "n1": ref.n1, "n2": ref.n2, "m": ref.m}
        for fmt in ("bf16x3", "f16f8"):
            pl, ms = planes(case, "float32", fmt)
            ephi = max((pl.phi[i:i + 2048].double() - rphi[i:i + 2048]).abs().max().item()
                       for i in range(0, ref.n1, 2048))
            epsi = max((pl.psi[i:i + 2048].double() - rpsi[i:i + 2048]).abs().max().item()
                       for i in range(0, ref.n1, 2048))
            out[fmt] = {"k2_ms": ms, "rel_err_sync": ephi / sphi, "rel_err_async": epsi / max(spsi, 1e-300)}
            del pl
            torch.cuda.empty_cache()
        del ref, rphi, rpsi
        torch.cuda.empty_cache()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
