#!/usr/bin/env python3
"""Summarize an ncu report (.ncu-rep) or a launch-list CSV into profiles/.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep  -o profiles/r01_ncu.json [--blocks]
  python tools/ncu_summary.py --launches gpurun_out/launches.csv -o profiles/r01_launches.json

For each profiled kernel: duration, issued instructions, IPC, issue-slot
utilization, occupancy, registers, DRAM bytes read/written (the `traffic`
term of the roofline), pipe utilizations and warp-stall breakdown; with
--blocks also the hottest basic blocks (instruction-count groups) and the
top stalled SASS instructions.  Requires the `ncu` CLI (present in the build
container; no GPU needed to read a report).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys
from collections import Counter, defaultdict

DETAILS = {
    "Duration": "duration_us", "Executed Ipc Active": "ipc_active", "Issue Slots Busy": "issue_slots_busy_pct",
    "Issued Instructions": "issued_instructions", "Registers Per Thread": "registers",
    "Achieved Active Warps Per SM": "achieved_warps_per_sm", "Theoretical Active Warps per SM": "theoretical_warps_per_sm",
    "Eligible Warps Per Scheduler": "eligible_warps_per_scheduler", "No Eligible": "no_eligible_pct",
    "L1/TEX Hit Rate": "l1_hit_pct", "L2 Hit Rate": "l2_hit_pct", "DRAM Throughput": "dram_throughput_pct",
    "Compute (SM) Throughput": "sm_throughput_pct", "SM Frequency": "sm_ghz", "Grid Size": "grid", "Block Size": "block",
}
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
STALLS = ["long_sb", "wait", "not_selected", "selected", "short_sb", "math", "branch_resolving", "no_inst", "dispatch",
          "lg", "mio", "sleep", "barrier", "membar", "drain"]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return x


def summarize_report(path, blocks):
    kernels = []
    rows = ncu_csv(["-i", path, "--page", "details", "--csv"])
    h = rows[0]
    by_id = defaultdict(dict)
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (d.get("ID"), d.get("Kernel Name"))
        if d.get("Metric Name") in DETAILS:
            by_id[key][DETAILS[d["Metric Name"]]] = num(d["Metric Value"])
    raw = ncu_csv(["-i", path, "--page", "raw", "--csv"])
    rh = raw[0]
    units = dict(zip(rh, raw[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1 << 20, "GB": 1 << 30}
    raw_rows = [dict(zip(rh, r)) for r in raw[2:]]
    for (kid, name), vals in by_id.items():
        k = {"id": kid, "kernel": name, **vals}
        for rr in raw_rows:
            if rr.get("ID") == kid:
                for m in RAW:
                    if m in rr:
                        v = num(rr[m])
                        if m.startswith("dram__bytes") and isinstance(v, float):
                            v *= scale.get(units.get(m, "byte"), 1)
                        k[m] = v
        k["dram_bytes"] = (k.get("dram__bytes_read.sum") or 0) + (k.get("dram__bytes_write.sum") or 0)
        kernels.append(k)
    if blocks:
        src = ncu_csv(["-i", path, "--page", "source", "--csv", "--print-source", "sass"])
        cur = None
        per = []
        for r in src:
            if r and r[0] == "Kernel Name":
                cur = {"name": r[1], "rows": []}
                per.append(cur)
            elif r and r[0] == "Address":
                cur["h"] = r
            elif cur and "h" in cur and len(r) == len(cur["h"]):
                cur["rows"].append(dict(zip(cur["h"], r)))
        # the source page lists kernels in ID order (names are formatted
        # differently from the details page); keep the first listing of each
        seen, uniq = set(), []
        for b in per:
            if b["name"] not in seen and b["rows"]:
                seen.add(b["name"])
                uniq.append(b)
        for kk, b in zip(sorted(kernels, key=lambda k: int(k["id"])), uniq):
            data = b["rows"]
            tot = sum(int(d["Instructions Executed"]) for d in data) or 1
            stalls = {s: sum(int(d.get("stall_" + s, 0) or 0) for d in data) for s in STALLS}
            groups = defaultdict(lambda: [0, 0, Counter(), ""])
            for d in data:
                n = int(d["Instructions Executed"])
                src_ = d["Source"].strip()
                op = (src_.split()[1] if src_.startswith("@") else src_.split()[0]).split(".")[0]
                g = groups[n]
                g[0] += 1
                g[1] += n
                g[2][op] += 1
                g[3] = g[3] or d["Address"][-6:]
            kk["stall_samples"] = stalls
            kk["blocks"] = [{"exec": n, "instrs": c, "share": round(s / tot, 4), "first": f,
                             "ops": dict(ops.most_common(10))}
                            for n, (c, s, ops, f) in sorted(groups.items(), key=lambda x: -x[1][1])[:10]]
            top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"]))[:12]
            kk["top_stalled"] = [{"addr": d["Address"][-6:], "exec": int(d["Instructions Executed"]),
                                  "sass": d["Source"].strip()[:60],
                                  "stalls": {s: int(d["stall_" + s]) for s in STALLS
                                             if d.get("stall_" + s) not in (None, "", "0")}} for d in top]
    return {"report": path, "kernels": kernels}


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    h = None
    per = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            per[d["Kernel Name"]].append(float(d["Metric Value"]))
    out = []
    for n, v in per.items():
        v = sorted(v)
        out.append({"kernel": n, "launches": len(v), "median_ns": v[len(v) // 2], "min_ns": v[0], "max_ns": v[-1]})
    return {"launch_list": path, "metric": "gpu__time_duration.sum", "kernels": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("-o", "--out")
    ap.add_argument("--blocks", action="store_true")
    a = ap.parse_args()
    res = summarize_launches(a.launches) if a.launches else summarize_report(a.report, a.blocks)
    txt = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(txt + "\n")
    else:
        sys.stdout.write(txt + "\n")


if __name__ == "__main__":
    main()
