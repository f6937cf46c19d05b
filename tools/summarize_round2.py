#!/usr/bin/env python3
"""Turn a tools/profile_round2.sh run (gpurun_out/prof2/) into the tracked
evidence under profiles/ (r2_* files) and regenerate profiles/README.md from
them -- no hand-edited numbers.

Usage: python tools/summarize_round2.py [gpurun_out/prof2]
"""
import json
import re
import shutil
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from summarize_profiles import launch_shares, ncu_raw  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
RND = "r2"


def last_json(path):
    if not path.exists():
        return None
    lines = [ln for ln in path.read_text().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main():
    src = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out" / "prof2"
    dst = ROOT / "profiles"
    dst.mkdir(exist_ok=True)
    for name in [f"bench_cfg{c}.json" for c in range(1, 6)] + ["bench_reference_cfg5.json"]:
        d = last_json(src / name)
        if d is not None:
            (dst / f"{RND}_{name}").write_text(json.dumps(d, indent=1) + "\n")
    for name in ("peaks.json", "floor.json"):
        d = last_json(src / name)
        if d is not None:
            (dst / f"{RND}_{name}").write_text(json.dumps(d, indent=1) + "\n")
    ex = src / "extras.json"
    if ex.exists():
        lines = [json.loads(ln) for ln in ex.read_text().splitlines() if ln.startswith("{")]
        (dst / f"{RND}_extras.json").write_text(json.dumps(lines, indent=1) + "\n")
    for f in sorted((src / "evidence").glob("*.json")):
        shutil.copy(f, dst / f.name)
    # fp64 contraction bound decomposition (profiling build)
    dec = {}
    for c in (3, 4):
        row = {}
        for skip, label in ((0, "full"), (1, "no_stores"), (2, "no_mma"), (3, "neither")):
            d = last_json(src / f"decomp_cfg{c}_skip{skip}.json")
            if d:
                row[label + "_ms"] = d["kernel_ms"]
        if row:
            dec[f"cfg{c}"] = row
    if dec:
        dec["how"] = ("tools/time_contract.py: 30 back-to-back K2 launches after one K1, CUDA events; "
                      "profiling build (-DCORR2D_PROFILING) with CORR2D_DEBUG_SKIP=1 (no output stores), "
                      "2 (no MMAs), 3 (neither: operand loads + epilogue arithmetic only)")
        (dst / f"{RND}_f64_decomposition.json").write_text(json.dumps(dec, indent=1) + "\n")
    for name in ("small_trace.txt", "power_cfg5.txt", "small_decomp.txt"):
        if (src / name).exists():
            shutil.copy(src / name, dst / f"{RND}_{name}")
    for name in ("gpu_tests.log", "wholemap_tests.log", "guards.log"):
        if (src / name).exists():
            text = (src / name).read_text(errors="replace").splitlines()
            (dst / f"{RND}_{name.replace('.log', '.txt')}").write_text("\n".join(text[-15:]) + "\n")
    for c in (5, 1, 2, 3):
        p = src / f"launches_cfg{c}.csv"
        if p.exists():
            shutil.copy(p, dst / f"{RND}_launches_cfg{c}.csv")
            (dst / f"{RND}_launch_shares_cfg{c}.json").write_text(json.dumps(launch_shares(p), indent=1) + "\n")
    tpath = dst / "traffic.json"
    traffic = json.loads(tpath.read_text()) if tpath.exists() else {}
    for rep in sorted(src.glob("full_cfg*.ncu-rep")):
        cfg = rep.stem.split("cfg")[1]
        ks = ncu_raw(rep)
        (dst / f"{RND}_ncu_cfg{cfg}.json").write_text(json.dumps(ks, indent=1) + "\n")
        con = [k for k in ks if "contract" in k["kernel"]]
        small = [k for k in ks if "small_" in k["kernel"]]
        if small and not con:        # small-m path: the step's two kernels together
            traffic[cfg] = sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in small[-2:])
        elif con:
            k = con[-1]
            traffic[cfg] = k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
    # small-m path: single-pass DRAM counters of the step's two kernels late in
    # the bench's rotation (--cache-control none: the steady state's evictions),
    # averaged over the captured steps
    import csv
    for c in (1, 2):
        p = src / f"traffic_cfg{c}.csv"
        if not p.exists():
            continue
        rows = [r for r in csv.reader(ln for ln in p.read_text().splitlines() if ln.startswith('"'))]
        hdr = rows[0]
        ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
        per = {}
        for r in rows[1:]:
            if r[ix["Metric Name"]] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                per[r[ix["ID"]]] = per.get(r[ix["ID"]], 0.0) + float(r[ix["Metric Value"]].replace(",", ""))
        if per:
            steps = max(1, len(per) // 2)
            traffic[str(c)] = sum(per.values()) / steps
            shutil.copy(p, dst / f"{RND}_traffic_cfg{c}.csv")
    tpath.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")
    for rep in sorted(src.glob("full_peaks*.ncu-rep")):
        (dst / f"{RND}_ncu_{rep.stem[5:]}.json").write_text(json.dumps(ncu_raw(rep), indent=1) + "\n")
    readme(dst)
    print("wrote", sorted(p.name for p in dst.iterdir() if p.name.startswith(RND) or p.name == "README.md"))


def _load(p):
    return json.loads(p.read_text()) if p.exists() else None


def readme(dst):
    R = RND
    L = ["# profiles/ -- evidence (B200, 1 GPU)", "",
         f"Round 2 files are `{R}_*` (produced by `tools/profile_round2.sh` under gpurun and summarised by "
         f"`tools/summarize_round2.py`; every number below is read from them).  Round 1's `r1_*` files are kept "
         "for comparison.", ""]
    L += ["## Headline (bench.py)", "",
          "CUDA events around a graph of K steps (per-step event pairs for cfg3-5; an event-free graph rotating "
          "over independent buffers larger than 4x L2 for cfg1 / cfg2); clocks sampled during the timed region; "
          "`e2e` = the public `corr2d()` call with pinned host inputs and pinned host output planes.", "",
          "| config | ms/step | GElem/s | K2 ms | roofline frac | executed frac | e2e GElem/s (ms/call) | SM MHz (reasons) | r1 ms/step |",
          "|---|---|---|---|---|---|---|---|---|"]
    b5 = None
    for c in range(1, 6):
        b = _load(dst / f"{R}_bench_cfg{c}.json")
        if b is None:
            continue
        if c == 5:
            b5 = b
        r, ck = b["roofline"], b["clocks"]
        old = _load(dst / f"r1_bench_cfg{c}.json")
        ex = r.get("executed", {}).get("frac_of_peak")
        L.append(f"| {b['config']['workload']} | {b['ms_per_step']:.4f} | {b['value']:.1f} | "
                 f"{r.get('kernel_ms', float('nan')):.4f} | {r['frac']:.3f} ({r['bound']}, {r['peak']:g} {r['unit']}) | "
                 f"{'-' if ex is None else f'{ex:.3f}'} | {b['e2e']['value']:.2f} ({b['e2e']['ms_per_step']:.3f}) | "
                 f"{ck['sm_mhz']:.0f} {','.join(ck['reasons']) or '-'} | "
                 f"{'-' if old is None else format(old['ms_per_step'], '.4f')} |")
    L += ["",
          "* roofline frac = algorithmic work (8K flops per complex element) / K2 time / measured peak. The fp64 "
          "homo configs exceed 1.0: the map is computed once per mirrored tile pair and, with the Gauss form, "
          "with 3 instead of 4 real products per bin; `executed frac` counts the DMMA / tensor-core flops the "
          "kernel actually issues against the same peak. cfg1 / cfg2 run the small-m path (two PDL-chained "
          "kernels: K1 + contraction), so their 'K2 ms' is the whole step.",
          "* roofline `traffic` (profiles/traffic.json): ncu DRAM bytes of the dominant kernel per launch; for "
          "cfg1 / cfg2 the step's two kernels late in the bench's rotation, single-pass counters with "
          "`--cache-control none` (`r2_traffic_cfg*.csv`: the steady state's write-backs, ~15 / 48 MB against "
          "16 / 48 MB of planes).  Bench lines record the file as it was when they ran."]
    ref = _load(dst / f"{R}_bench_reference_cfg5.json")
    if ref and b5:
        L.append(f"* Reference arm ({ref['cpu_baseline']['kind']} on {ref['cpu_baseline']['cores']} host threads): "
                 f"{ref['value']:.4f} GElem/s -> e2e / reference = {b5['e2e']['value'] / ref['value']:.0f}x "
                 f"(the e2e step is bound by the PCIe link and the host's memory: "
                 f"{b5['e2e']['d2h_bytes_per_step'] / 1e9:.1f} GB of the 8.6 GB of planes cross the link, host threads "
                 f"fill the rest as the mirror), device-resident value / reference = {b5['value'] / ref['value']:.0f}x.")
    if b5 and "cpu_baseline" in b5:
        cb = b5["cpu_baseline"]
        L.append(f"* cpu_baseline in the cfg5 line: {cb['value']:.4f} GElem/s ({cb['cores']} threads; {cb['sample']}).")
    pk, fl = _load(dst / f"{R}_peaks.json"), _load(dst / f"{R}_floor.json")
    if pk or fl:
        L += ["", "## Measured peaks and floors (this pool)", ""]
        if pk:
            L.append(f"* `tools/microbench/peaks.cu` ({R}_peaks.json): FP64 DMMA {pk['dmma_m16n8k16_tflops']} TFLOP/s, "
                     f"DFMA {pk['dfma_tflops']} TFLOP/s, HBM copy {pk['hbm_copy_gbs']} GB/s, pinned H2D "
                     f"{pk['h2d_pinned_gbs']} / D2H {pk['d2h_pinned_gbs']} GB/s.  bench.py's FP64 denominator "
                     f"(37.03) is this DMMA figure.")
        if fl:
            L.append(f"* `tools/microbench/floor.cu` ({R}_floor.json), graphs of {fl['graph_steps']} steps rotating over "
                     f"buffers > 4x L2: empty kernel {fl['empty_kernel_us']} us, two PDL-chained empty kernels "
                     f"{fl['two_empty_kernels_pdl_us']} us, a 16 MB store (cfg1's planes) {fl['store_16MB_us']} us "
                     f"({fl['store_16MB_GBs']} GB/s), 48 MB (cfg2) {fl['store_48MB_us']} us.  Against these floors: "
                     + ", ".join(f"cfg{c} {(_load(dst / f'{R}_bench_cfg{c}.json') or {}).get('ms_per_step', float('nan')) * 1e3:.1f} us"
                                 for c in (1, 2)) + ".")
    dec = _load(dst / f"{R}_f64_decomposition.json")
    if dec:
        L += ["", "## fp64 contraction: where the time goes (profiling build, K2 alone)", "",
              "| config | full ms | no stores | no MMAs | neither (loads + epilogue math) |", "|---|---|---|---|---|"]
        for c in ("cfg3", "cfg4"):
            if c in dec:
                d = dec[c]
                L.append(f"| {c} | {d.get('full_ms', 0):.3f} | {d.get('no_stores_ms', 0):.3f} | "
                         f"{d.get('no_mma_ms', 0):.3f} | {d.get('neither_ms', 0):.3f} |")
        L.append("")
        L.append("* " + dec["how"] + ".  MMA-only and store-only each run near their own ceilings (DMMA ~84 % "
                 "of peak; stores at the tile + mirror pattern's ~5.6 TB/s); the full kernel is their "
                 "imperfect overlap.")
    sd = dst / f"{R}_small_decomp.txt"
    if sd.exists():
        L += ["", "## Small-m path: step decomposition (tools/dev/small_rot.py, the bench's rotation graph, us/step)",
              "", "```"] + sd.read_text().strip().splitlines() + ["```"]
    tr = dst / f"{R}_small_trace.txt"
    if tr.exists():
        L += ["", "## Small-m path timeline (profiling build, one cold-ish step, ns)", "",
              "Eager launches: the gap between K1's last stamp and the contraction's `after wait` includes the "
              "host's encoding / launch of the second kernel (a graph replay has none); the steady state is the "
              "decomposition above.", "", "```"] + \
             tr.read_text().strip().splitlines() + ["```"]
    L += ["", "## Parity beyond sampled rows", ""]
    for f in sorted(dst.glob("r2_wholemap_*.json")) + sorted(dst.glob("r2_*_adversarial_*.json")):
        L.append(f"* `{f.name}`: `{json.dumps(json.loads(f.read_text()))}`")
    for name in (f"{R}_wholemap_tests.txt", f"{R}_gpu_tests.txt"):
        p = dst / name
        if p.exists():
            L.append(f"* `{name}`: " + (p.read_text().strip().splitlines() or [""])[-1])
    p = dst / f"{R}_guards.txt"
    if p.exists():
        L += ["", "## Memory safety (tests/test_gpu_guards.py; compute-sanitizer is closed on this pool)", "",
              "Every kernel family runs with its buffers inside 0xFF (NaN) guard bands and padded rows; "
              "guards must be untouched and results bit-identical to tight buffers.", "",
              "* `" + p.name + "`: " + (p.read_text().strip().splitlines() or [""])[-1]]
    L += ["", "## ncu (cold, serialised launches; per-launch numbers)", "",
          "| kernel | config | duration ms | DRAM read MB | DRAM write MB | tensor pipe active % | SM MHz |",
          "|---|---|---|---|---|---|---|"]
    for tag in ("cfg5", "cfg3", "cfg1", "cfg2", "peaks5"):
        for k in _load(dst / f"{R}_ncu_{tag}.json") or []:
            tp = k.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
            hz = k.get("sm__cycles_elapsed.avg.per_second", 0.0)
            unit = k.get("sm__cycles_elapsed.avg.per_second.unit")
            hz_mhz = hz * (1e3 if unit == "Ghz" else 1e-6 if unit == "hz" else 1)
            L.append(f"| `{k['kernel'][:60]}` | {tag} | {k['gpu__time_duration.sum']:.4f} | "
                     f"{k['dram__bytes_read.sum'] / 1e6:.1f} | {k['dram__bytes_write.sum'] / 1e6:.1f} | "
                     f"{tp if isinstance(tp, str) else f'{tp:.1f}'} | {hz_mhz:.0f} |")
    for c in (5, 3, 1, 2):
        sh = _load(dst / f"{R}_launch_shares_cfg{c}.json")
        if sh:
            L.append(f"* Launch shares of the cfg{c} step (ncu launch list): " + ", ".join(
                f"{k.split('(')[0].replace('void ', '')} {v['share'] * 100:.1f}%" for k, v in sh["kernels"].items()))
    ex = _load(dst / f"{R}_extras.json")
    if ex:
        L += ["", "## SURVEY 8f rows (tools/bench_extras.py)", ""] + [f"* `{json.dumps(e)}`" for e in ex]
    (dst / "README.md").write_text("\n".join(L) + "\n")


if __name__ == "__main__":
    main()
