"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python tools/make_profile_summary.py --config c4 --round r01 \
        --launches gpurun_out/launches_c4_default.csv \
        --reports gpurun_out/prof_c4_r1.ncu-rep [more.ncu-rep ...]

Writes / updates
  profiles/ncu_summary.json         {config: {kernel: {...}}}  (bench.py reads dram_bytes_per_launch)
  profiles/<round>_<config>.md      launch-list shares + per-kernel counters
and copies the launch list to profiles/<round>_<config>_launches.csv.
For k_smooth the steady-state iteration (the longest captured launch, i.e. one
that gathers neighbour offsets) is the representative launch.
"""
import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
METRICS = {
    "duration_ms": ("gpu__time_duration.sum", "ms"),
    "dram_read_bytes": ("dram__bytes_read.sum", "byte"),
    "dram_write_bytes": ("dram__bytes_write.sum", "byte"),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    "sm_pct_peak": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%"),
    "registers": ("launch__registers_per_thread", ""),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", "%"),
    "warp_instructions": ("smsp__inst_executed.sum", ""),
    "stall_long_scoreboard": ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", ""),
    "stall_barrier": ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", ""),
    "stall_short_scoreboard": ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", ""),
    "stall_wait": ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", ""),
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0, "us": 1e-3, "ns": 1e-6}


def kernel_key(name):
    n = name.split("(")[0].replace("void ", "").replace("psn::", "").strip()
    return n.split("<")[0]


def read_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = {"kernel": kernel_key(r[hdr.index("Kernel Name")]), "full_name": r[hdr.index("Kernel Name")]}
        for k, (m, _) in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
        recs.append(d)
    return recs


def read_launches(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    agg = collections.defaultdict(list)
    for r in csv.DictReader(io.StringIO(txt)):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"])
            unit = r.get("Metric Unit", "ns")
            agg[kernel_key(r["Kernel Name"])].append(v * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1e-6))
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--round", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--reports", nargs="*", default=[])
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    js_path = os.path.join(PROF, "ncu_summary.json")
    summary = json.load(open(js_path)) if os.path.exists(js_path) else {}
    cfg = summary.setdefault(args.config, {})
    for rep in args.reports:
        best = {}
        for d in read_report(rep):   # keep the longest launch of each kernel in this report
            if d["kernel"] not in best or d.get("duration_ms", 0) > best[d["kernel"]].get("duration_ms", 0):
                best[d["kernel"]] = d
        for k, d in best.items():
            d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
            d["source"] = os.path.basename(rep)
            d["round"] = args.round
            cfg[k] = d
    md = [f"# {args.round} — ncu summary, config {args.config}", ""]
    if args.note:
        md += [args.note, ""]
    if args.launches:
        la = read_launches(args.launches)
        shutil.copy(args.launches, os.path.join(PROF, f"{args.round}_{args.config}_launches.csv"))
        # shares of the last full step: take per-kernel means weighted by launches per step
        md += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`; cold-cache, serialised)", "",
               "| kernel | launches | mean (us) | min (us) | total (ms) |", "|---|---|---|---|---|"]
        for k, v in sorted(la.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| {k} | {len(v)} | {1e3 * sum(v) / len(v):.1f} | {1e3 * min(v):.1f} | {sum(v):.3f} |")
        cfg["_launch_means_ms"] = {k: sum(v) / len(v) for k, v in la.items()}
        md.append("")
    md += ["## Per-kernel counters (`ncu --set full`, one representative launch each)", "",
           "| kernel | ms | DRAM read GB | DRAM write GB | DRAM % peak | warps active % | issue active % | regs | L2 hit % | warp instr (M) | stall long-sb | stall barrier |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, d in cfg.items():
        if k.startswith("_"):
            continue
        md.append(f"| {k} | {d.get('duration_ms', 0):.3f} | {d.get('dram_read_bytes', 0) / 1e9:.3f} | "
                  f"{d.get('dram_write_bytes', 0) / 1e9:.3f} | {d.get('dram_pct_peak', 0):.1f} | "
                  f"{d.get('warps_active_pct', 0):.1f} | {d.get('issue_active_pct', 0):.1f} | {d.get('registers', 0):.0f} | "
                  f"{d.get('l2_hit_pct', 0):.1f} | {d.get('warp_instructions', 0) / 1e6:.1f} | "
                  f"{d.get('stall_long_scoreboard', 0):.2f} | {d.get('stall_barrier', 0):.2f} |")
    json.dump(summary, open(js_path, "w"), indent=1, sort_keys=True)
    open(os.path.join(PROF, f"{args.round}_{args.config}.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
