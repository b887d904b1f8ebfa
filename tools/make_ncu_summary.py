#!/usr/bin/env python3
"""Builds profiles/ncu_summary.json (read by bench.py for roofline.traffic and
roofline.issue) from the per-config full captures profiles/<tag>_ncu_full_cfg*.json
written by tools/r02_refresh.sh.  Usage: python tools/make_ncu_summary.py r02"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_22901_b200 import workloads as W  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
out = {"source": f"ncu --set full --clock-control none --import-source on, one launch of each config's kernels "
                  f"(tools/r02_refresh.sh; per-kernel summaries in profiles/{tag}_ncu_full_cfg{{1,2,3,4}}.json, "
                  f"launch list of the cfg4 headline bench in profiles/{tag}_ncu_launches_cfg4.json)",
       "phase1_dram_bytes_per_launch": {}, "phase1_instr_per_candidate": {}, "kernels": {}}
for c in ("cfg4", "cfg1", "cfg3", "cfg2"):
    p = os.path.join(ROOT, "profiles", f"{tag}_ncu_full_{c}.json")
    if not os.path.exists(p):
        continue
    d = json.load(open(p))
    wl = W.ALL[c]()
    cand = wl.n_searches * len(wl.radii) * len(wl.angles)
    ks = {}
    for k in d["kernels"]:
        name = k["kernel"].split("(")[0].split("::")[-1].split("<")[0]
        if name in ks:
            continue
        ks[name] = {"duration": k["duration_us"], "issued_instructions": k["issued_instructions"],
                    "issue_slots_busy_pct": k["issue_slots_busy_pct"], "dram_bytes": k["dram_bytes"]}
        if name == "phase1_kernel":
            out["phase1_dram_bytes_per_launch"][c] = int(k["dram_bytes"])
            out["phase1_instr_per_candidate"][c] = round(k["issued_instructions"] * 32 / cand, 2)
    out["kernels"][c] = ks
out["note"] = ("dram = dram__bytes_read.sum + dram__bytes_write.sum of the kernel; instr per candidate = issued warp "
               "instructions x 32 / candidates. PAIRS phase 1 writes the pass masks (1 bit per candidate); "
               "lists_kernel turns them into the tile lists. cfg4 phase 1 updates per-search counts and first "
               "indices (atomics) and reads sc_index. Durations as ncu prints them (ms for kernels over 1 ms, else us).")
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
print(json.dumps(out["phase1_instr_per_candidate"]), json.dumps(out["phase1_dram_bytes_per_launch"]))
