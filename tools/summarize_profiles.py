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
    for c in (5, 1, 2):
        if (src / f"launches_cfg{c}.csv").exists():
            shutil.copy(src / f"launches_cfg{c}.csv", dst / f"{rnd}_launches_cfg{c}.csv")
            (dst / f"{rnd}_launch_shares_cfg{c}.json").write_text(
                json.dumps(launch_shares(src / f"launches_cfg{c}.csv"), indent=1) + "\n")
    tpath = dst / "traffic.json"
    traffic = json.loads(tpath.read_text()) if tpath.exists() else {}
    for rep in sorted(src.glob("full_cfg*.ncu-rep")):
        cfg = rep.stem.split("cfg")[1]
        ks = ncu_raw(rep)
        (dst / f"{rnd}_ncu_cfg{cfg}.json").write_text(json.dumps(ks, indent=1) + "\n")
        con = [k for k in ks if "contract" in k["kernel"] or "small_fused" in k["kernel"]]
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
    readme(rnd, dst)
    print("wrote", sorted(p.name for p in dst.iterdir()))


def _load(path):
    return json.loads(path.read_text()) if path.exists() else None


def readme(rnd, dst):
    """profiles/README.md from the round's JSON files (no hand-edited numbers)."""
    L = [f"# profiles/ -- round {rnd[1:]} evidence (B200, 1 GPU)", "",
         f"Produced by `tools/profile_round.sh` under gpurun and summarised by "
         f"`tools/summarize_profiles.py {rnd}`; every number below is read from the JSON files here.", "",
         f"Files: `{rnd}_bench_cfg{{1..5}}.json` (bench.py lines), `{rnd}_bench_reference_cfg5.json` "
         f"(reference arm), `{rnd}_launches_cfg{{5,1,2}}.csv` + `{rnd}_launch_shares_cfg{{5,1,2}}.json` (ncu launch "
         f"lists of the bench commands), `{rnd}_ncu_cfg{{5,3,1,2}}.json`, `{rnd}_ncu_peaks5.json` (selected metrics of "
         f"`ncu --set full` captures), `{rnd}_extras.json` (tools/bench_extras.py: Hilbert route, find_peaks, "
         f"serialization), `traffic.json` (dram bytes per K2 launch, read by bench.py for `roofline.traffic`).",
         "", "## Headline (bench.py: CUDA events around a graph of K steps -- per-step event pairs for cfg3-5, "
         "event-free rotation over independent buffers for cfg1 / cfg2; clocks sampled during the timed region)",
         "", "| config | ms/step | GElem/s | K2 ms | roofline frac | executed frac | e2e GElem/s | SM MHz (reasons) |",
         "|---|---|---|---|---|---|---|---|"]
    b5 = None
    for c in range(1, 6):
        b = _load(dst / f"{rnd}_bench_cfg{c}.json")
        if b is None:
            continue
        if c == 5:
            b5 = b
        r, ck = b["roofline"], b["clocks"]
        ex = r.get("executed", {}).get("frac_of_peak")
        L.append(f"| {b['config']['workload']} | {b['ms_per_step']:.4f} | {b['value']:.1f} | "
                 f"{r.get('kernel_ms', float('nan')):.4f} | {r['frac']:.3f} ({r['bound']}, {r['peak']:g} {r['unit']}) | "
                 f"{'-' if ex is None else f'{ex:.3f}'} | {b['e2e']['value']:.2f} | "
                 f"{ck['sm_mhz']:.0f} {','.join(ck['reasons']) or '-'} |")
    L.append("")
    L.append("* roofline frac = algorithmic work / K2 time / measured peak (MEASURED_PEAKS.json). fp64 configs "
             "exceed 1.0 because the homo map is computed once per mirrored tile pair (algorithmic flops count "
             "the full map); executed frac counts the flops the kernel actually issues, in fp16-equivalents (F16F8: the "
             "fp16 hi.hi product + two e4m3 cross products at twice the rate = 2; bf16x3: 3). cfg1 / cfg2 run as ONE "
             "kernel (small_fused_kernel: K1 + contraction), so their 'K2 ms' is the whole step, timed as an "
             "event-free graph rotating over independent buffers (> 4x L2); the two-kernel path's K2-only "
             "fraction is not comparable.")
    ref = _load(dst / f"{rnd}_bench_reference_cfg5.json")
    if ref and b5:
        L.append(f"* Reference arm ({ref['cpu_baseline']['kind']} on {ref['cpu_baseline']['cores']} host threads, "
                 f"{ref['cpu_baseline']['sample'][:60]}...): {ref['value']:.4f} GElem/s -> e2e speed-up "
                 f"{b5['e2e']['value'] / ref['value']:.0f}x (the e2e step is PCIe-bound: "
                 f"{b5['e2e']['d2h_bytes_per_step'] / 1e9:.1f} GB of planes D2H per step); device-resident "
                 f"value / reference = {b5['value'] / ref['value']:.0f}x.")
    if b5:
        cb = b5["cpu_baseline"]
        L.append(f"* cpu_baseline in the cfg5 line: {cb['value']:.4f} GElem/s ({cb['cores']} threads, {cb['sample']}).")
    L += ["", "## ncu (cold, serialised launches; per-launch numbers)", "",
          "| kernel | config | duration ms | DRAM read MB | DRAM write MB | tensor pipe active % | SM MHz |",
          "|---|---|---|---|---|---|---|"]
    for tag in ("cfg5", "cfg3", "cfg1", "cfg2", "peaks5"):
        ks = _load(dst / f"{rnd}_ncu_{tag}.json") or []
        for k in ks:
            tp = k.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
            hz = k.get("sm__cycles_elapsed.avg.per_second", 0.0)
            hz_mhz = hz * (1e3 if k.get("sm__cycles_elapsed.avg.per_second.unit") == "Ghz" else
                           1e-6 if k.get("sm__cycles_elapsed.avg.per_second.unit") == "hz" else 1)
            L.append(f"| `{k['kernel'][:60]}` | {tag} | {k['gpu__time_duration.sum']:.4f} | "
                     f"{k['dram__bytes_read.sum'] / 1e6:.1f} | {k['dram__bytes_write.sum'] / 1e6:.1f} | "
                     f"{tp if isinstance(tp, str) else f'{tp:.1f}'} | {hz_mhz:.0f} |")
    sh = _load(dst / f"{rnd}_launch_shares_cfg5.json")
    if sh:
        L += ["", "* Launch shares of the cfg5 step (ncu launch list): " + ", ".join(
            f"{k.split('(')[0].replace('void ', '')} {v['share'] * 100:.1f}%" for k, v in sh["kernels"].items())]
    ex = _load(dst / f"{rnd}_extras.json")
    if ex:
        L += ["", "## SURVEY 8f rows (tools/bench_extras.py)", ""] + [f"* `{json.dumps(e)}`" for e in ex]
    (dst / "README.md").write_text("\n".join(L) + "\n")


if __name__ == "__main__":
    main()
