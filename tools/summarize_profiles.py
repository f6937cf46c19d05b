#!/usr/bin/env python3
"""Turn a tools/profile_round.sh run (gpurun_out/prof/) into the tracked
evidence under profiles/:

  profiles/<round>_bench_cfg{1..5}.json        bench lines (our arm)
  profiles/<round>_bench_reference_cfg5.json   reference arm line
  profiles/<round>_launches_cfg5.csv           ncu launch list (gpu__time_duration)
  profiles/<round>_launch_shares_cfg5.json     per-kernel mean time and share of the step
  profiles/<round>_ncu_cfg{5,3}.json           selected metrics of the --set full capture
  profiles/traffic.json                         dram read+write bytes per launch of the
                                                dominant kernel, keyed by config (bench.py
                                                reads it for roofline.traffic)

Usage: python tools/summarize_profiles.py r1 [gpurun_out/prof]
"""
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__cluster_size",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
              "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1, "nsecond": 1e-6}


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = r[i].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                k[m] = v
                continue
            u = units[i]
            if m.startswith("dram__bytes"):
                v *= UNIT_SCALE.get(u, 1)
                u = "byte"
            elif m == "gpu__time_duration.sum":
                v *= UNIT_SCALE.get(u, 1)
                u = "ms"
            k[m] = v
            k[m + ".unit"] = u
        kernels.append(k)
    return kernels


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = {}
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        ms = float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1)
        per.setdefault(r[ki], []).append(ms)
    mine = {k: v for k, v in per.items() if "corr2d::" in k or "tc::" in k}
    means = {k: sum(v) / len(v) for k, v in mine.items()}
    step = sum(means.values())
    return {"step_ms_sum_of_kernel_means": step,
            "kernels": {k: {"launches": len(per[k]), "mean_ms": means[k], "share": means[k] / step}
                        for k in means},
            "note": "ncu launch list: cold-cache, serialised per-launch times; shares, not absolutes, "
                    "are compared with the bench's live CUDA-event timing"}


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
    src = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "gpurun_out" / "prof"
    dst = ROOT / "profiles"
    dst.mkdir(exist_ok=True)
    for f in sorted(src.glob("bench_*.json")):
        text = f.read_text().strip()
        if text:
            (dst / f"{rnd}_{f.name}").write_text(json.dumps(json.loads(text.splitlines()[-1]), indent=1) + "\n")
    if (src / "launches_cfg5.csv").exists():
        shutil.copy(src / "launches_cfg5.csv", dst / f"{rnd}_launches_cfg5.csv")
        (dst / f"{rnd}_launch_shares_cfg5.json").write_text(
            json.dumps(launch_shares(src / "launches_cfg5.csv"), indent=1) + "\n")
    tpath = dst / "traffic.json"
    traffic = json.loads(tpath.read_text()) if tpath.exists() else {}
    for rep in sorted(src.glob("full_cfg*.ncu-rep")):
        cfg = rep.stem.split("cfg")[1]
        ks = ncu_raw(rep)
        (dst / f"{rnd}_ncu_cfg{cfg}.json").write_text(json.dumps(ks, indent=1) + "\n")
        con = [k for k in ks if "contract" in k["kernel"]]
        if con:
            k = con[-1]
            traffic[cfg] = k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
    tpath.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")
    for rep in sorted(src.glob("full_peaks*.ncu-rep")):
        (dst / f"{rnd}_ncu_{rep.stem[5:]}.json").write_text(json.dumps(ncu_raw(rep), indent=1) + "\n")
    ex = src / "extras.json"
    if ex.exists():
        lines = [json.loads(l) for l in ex.read_text().splitlines() if l.startswith("{")]
        (dst / f"{rnd}_extras.json").write_text(json.dumps(lines, indent=1) + "\n")
    print("wrote", sorted(p.name for p in dst.iterdir()))


if __name__ == "__main__":
    main()
