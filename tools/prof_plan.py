#!/usr/bin/env python3
"""Runs one config's device plan a few times (for ncu: skip the warm-up
launches with -s).  Usage: python tools/prof_plan.py cfg4 [--runs 3] [--path fast] [--output first]"""
import argparse
import os
import sys

# CVG_PKG_ROOT: import the package from another build tree (A/B of two builds in one run)
sys.path.insert(0, os.environ.get("CVG_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2507_22901_b200 as cv  # noqa: E402
from paper_2507_22901_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--path", default="fast")
ap.add_argument("--output", default=None)
a = ap.parse_args()
wl = W.ALL[a.config]()
ctx = cv.Context(0)
plan = ctx.plan(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles, output=a.output or wl.output,
                path=a.path)
plan.run(0)
n = plan.sync()
if (a.output or wl.output) == "pairs":
    plan.reserve(max(n, 1))
for _ in range(a.runs):
    plan.run(0)
    plan.sync()
print(a.config, "pairs", n, "kernel_ms", plan.last_kernel_ms())
if (a.output or wl.output) == "pairs":
    plan.set_phase_marks(True)
    plan.run(0)
    plan.sync()
    print(a.config, "phases_ms (phase1[+lists], scan, emit)", [round(x, 4) for x in plan.last_phase_ms()])
