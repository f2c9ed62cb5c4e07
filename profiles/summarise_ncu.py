"""Summarise ncu reports / launch lists into profiles/<round>_*.json|md.

    python profiles/summarise_ncu.py <round> gpurun_out/prof_*.ncu-rep [--launches gpurun_out/launches.csv]

Reads reports with `ncu -i <rep> --page raw --csv` (no GPU needed).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("time_us", "gpu__time_duration.sum", 1.0),
    ("dram_read_MB", "dram__bytes_read.sum", None),
    ("dram_write_MB", "dram__bytes_write.sum", None),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    ("registers", "launch__registers_per_thread", 1.0),
    ("grid", "launch__grid_size", 1.0),
    ("block", "launch__block_size", 1.0),
    ("stall_long_scoreboard", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", 1.0),
    ("stall_short_scoreboard", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", 1.0),
    ("stall_barrier", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", 1.0),
    ("stall_wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", 1.0),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
    ("lsu_pipe_pct", "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", 1.0),
    ("lsu_shared_pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
    ("inst_executed", "smsp__inst_executed.sum", 1.0),
]

UNIT_SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "usecond": 1.0, "msecond": 1e3,
              "nsecond": 1e-3, "us": 1.0, "ms": 1e3, "ns": 1e-3}


def read_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for name, metric, _ in METRICS:
            if metric not in hdr:
                continue
            i = hdr.index(metric)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if name.endswith("_MB") or name == "time_us":
                v *= UNIT_SCALE.get(u, 1.0)
            rec[name] = round(v, 3)
        if "dram_read_MB" in rec and "time_us" in rec:
            rec["dram_GBps"] = round((rec["dram_read_MB"] + rec.get("dram_write_MB", 0)) / rec["time_us"] * 1e3, 1)
        out.append(rec)
    return out


SETUP = ("k_generate",)  # input generation: untimed setup
QUERY = ("k_prepare", "k_seed", "k_groups", "k_bound", "k_lbscan", "k_refine", "k_refine_tma", "k_finalize",
         "k_pack_bsf", "k_import_bsf", "k_merge_results")


def read_launches(path):
    per = defaultdict(lambda: {"launches": 0, "total_us": 0.0, "dram_MB": 0.0})
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    for r in rows[1:]:
        name = r[ki].replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = name.split("(")[0].split("<")[0].strip().split("::")[-1]
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        if r[mi] == "gpu__time_duration.sum":
            per[name]["launches"] += 1
            per[name]["total_us"] += v * UNIT_SCALE.get(r[ui], 1.0)
        elif r[mi].startswith("dram__bytes"):
            per[name]["dram_MB"] += v * UNIT_SCALE.get(r[ui], 1e-6)
    tot = sum(p["total_us"] for k, p in per.items() if k not in SETUP) or 1.0
    qtot = sum(p["total_us"] for k, p in per.items() if k in QUERY) or 1.0
    out = {}
    for k, v in sorted(per.items(), key=lambda kv: -kv[1]["total_us"]):
        rec = {"launches": v["launches"], "total_us": round(v["total_us"], 1), "dram_MB": round(v["dram_MB"], 1)}
        if k not in SETUP:
            rec["share_excl_setup"] = round(v["total_us"] / tot, 4)
        if k in QUERY:
            rec["share_of_query"] = round(v["total_us"] / qtot, 4)
        out[k] = rec
    return out


def main():
    rnd = sys.argv[1]
    reps = [a for a in sys.argv[2:] if a.endswith(".ncu-rep")]
    launches = None
    if "--launches" in sys.argv:
        launches = sys.argv[sys.argv.index("--launches") + 1]
    here = os.path.dirname(os.path.abspath(__file__))
    summary = {"round": rnd, "reports": {}}
    for rep in reps:
        summary["reports"][os.path.basename(rep)] = read_report(rep)
    if launches:
        summary["launch_list"] = read_launches(launches)
    with open(os.path.join(here, f"{rnd}_ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    lines = [f"# ncu summary — {rnd}", ""]
    for rep, recs in summary["reports"].items():
        lines.append(f"## {rep}")
        for r in recs:
            lines.append("- " + ", ".join(f"{k}={v}" for k, v in r.items()))
        lines.append("")
    if launches:
        lines.append("## launch list (gpu__time_duration.sum + DRAM bytes, cold-cache, serialised)")
        for k, v in summary["launch_list"].items():
            lines.append(f"- {k}: " + ", ".join(f"{a}={b}" for a, b in v.items()))
    with open(os.path.join(here, f"{rnd}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
