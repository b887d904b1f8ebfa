#!/usr/bin/env python3
"""Feasibility sweep timing: the reference's default sweep
(756 cells, feasibility.cpp:16-36) through our feasibility_matrix (every cell
in one batched launch, select_best on the device: CVG_OUT_BEST) against the
reference's own feasibility_matrix + export (oracle/_ref, host cores), and the
cfg1 batch through ctx.search with output 'best' / 'pairs'.  Wall clock, host
arrays in, results out.  Usage: python tools/bench_sweep.py [-o out.json]"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_22901_b200 as cv  # noqa: E402
from paper_2507_22901_b200 import workloads as W  # noqa: E402


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e3, 4)


ap = argparse.ArgumentParser()
ap.add_argument("-o", default=None)
a = ap.parse_args()
text = '{"version": 1}'
cfg = cv.config_from_json(text)
out = {"sweep": "SearchConfig::defaults() (feasibility.cpp:16-36): %d cells" % cfg.combo_count()}
out["ours_matrix_ms"] = timed(lambda: cv.feasibility_matrix(cfg), 20)
out["ours_matrix_export_ms"] = timed(lambda: cv.export_matrix(cv.feasibility_matrix(cfg), "csv", True), 20)
ctx = cv.Context(0)
wl = W.cfg1()
for o in ("best", "pairs"):
    out[f"cfg1_{o}_e2e_ms"] = timed(lambda: ctx.search(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii,
                                                        wl.angles, output=o), 20)
try:
    from oracle.oracle import RefCodec

    ref = RefCodec()
    out["reference_matrix_export_ms"] = timed(lambda: ref.export(text, "csv", True), 3)
    out["reference_note"] = "the reference's own feasibility_matrix + export_matrix (oracle/_ref, all host threads)"
    out["exports_identical"] = cv.export_matrix(cv.feasibility_matrix(cfg), "csv", True) == ref.export(text, "csv", True)
except Exception as e:  # noqa: BLE001
    out["reference"] = f"unavailable: {e}"
print(json.dumps(out))
if a.o:
    json.dump(out, open(a.o, "w"), indent=1)
