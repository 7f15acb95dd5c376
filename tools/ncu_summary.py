#!/usr/bin/env python
"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked).

    python tools/ncu_summary.py --round r01 [--tag v1]

* launches.csv (the `--metrics gpu__time_duration.sum` launch list of a bench
  command) -> per-kernel count / total / share / average.
* *.ncu-rep (`--set full` captures) -> key metrics, stall reasons, hottest
  SASS lines; every capture also refreshes profiles/ncu_traffic.json
  (DRAM bytes of that launch, read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import argparse
import collections
import csv
import glob
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.avg.per_cycle_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(r[ui], 1.0)
        a = agg[r[ki].split("(")[0]]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'share':>6s} {'avg_us':>10s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:40s} {c:8d} {t:12.1f} {t / tot:6.3f} {t / c:10.1f}")
    return "\n".join(lines)


def raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    return rows[0], rows[1], rows[2:]


def source_top(rep, n=20):
    r = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))[2:]
    rows = [x for x in rows if len(x) > 5 and x[2].isdigit()]
    tot = sum(int(x[2]) for x in rows) or 1
    top = sorted(rows, key=lambda x: -int(x[2]))[:n]
    return "\n".join(f"{int(x[2]) / tot:6.3f}  {x[1].strip()[:80]}" for x in top)


def summarize_rep(rep):
    h, u, vals = raw(rep)
    out = []
    for v in vals[:1]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.append(f"kernel: {name}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"  {k:64s} {v[i]:>18s} {u[i]}")
        st = [(h[i], float(v[i].replace(",", ""))) for i in range(len(h))
              if h[i].startswith("smsp__average_warps_issue_stalled") and h[i].endswith("_per_issue_active.ratio")]
        out.append("  stall reasons (warps per issue-active cycle):")
        for k, x in sorted(st, key=lambda t: -t[1])[:8]:
            out.append(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {x:.3f}")
        d = {k: v[h.index(k)] for k in KEYS if k in h}
        d["_units"] = {k: u[h.index(k)] for k in KEYS if k in h}
    out.append("  hottest SASS (share of stall samples):")
    out.append("    " + source_top(rep).replace("\n", "\n    "))
    return "\n".join(out), d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    tag = f"_{a.tag}" if a.tag else ""
    lc = os.path.join(OUT, "launches.csv")
    if os.path.exists(lc):
        s = launches(lc)
        open(os.path.join(PROF, f"{a.round}{tag}_launches.txt"), "w").write(
            "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised; compare shares)\n" + s + "\n")
        print(s)
    for rep in sorted(glob.glob(os.path.join(OUT, "*.ncu-rep"))):
        base = os.path.basename(rep)[:-8]
        s, d = summarize_rep(rep)
        open(os.path.join(PROF, f"{a.round}{tag}_ncu_{base}.txt"), "w").write(s + "\n")
        print(s)
        names = {"prof_onesweep": "onesweep_kernel", "prof_detect": "detect_kernel", "prof_interp": "interp_kernel",
                 "prof_bucket_scatter": "bucket_scatter_kernel", "prof_bucket_detect": "bucket_detect_kernel",
                 "prof_filter": "filter_kernel", "prof_k1c": "rc_k1c"}
        if base in names:
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            byts = sum(float(d[k].replace(",", "")) * mult[d["_units"][k]]
                       for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            path = os.path.join(PROF, "ncu_traffic.json")
            tr = json.load(open(path)) if os.path.exists(path) else {}
            name = names[base]
            tr[name] = {"dram_bytes_per_launch": byts,
                        "warp_instructions_per_launch": float(d["smsp__inst_executed.sum"].replace(",", "")),
                        "ipc_per_sm": float(d["sm__inst_executed.avg.per_cycle_active"].replace(",", "")),
                        "source": f"profiles/{a.round}{tag}_ncu_{base}.txt (ncu --set full --cache-control all, "
                                  "one launch of the bench workload)"}
            json.dump(tr, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
