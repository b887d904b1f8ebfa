import sys, time, os
import numpy as np
import paper_2507_22901_b200 as cv
from paper_2507_22901_b200 import workloads as W
w = W.cfg4()
ctx = cv.Context(0)
for i in range(4):
    print(f"--- call {i}", file=sys.stderr, flush=True)
    t = time.perf_counter()
    r = ctx.search(w.targets, w.patterns, w.v_th, w.r_novib, w.radii, w.angles, output=w.output)
    print(f"call {i}: {(time.perf_counter()-t)*1e3:.2f} ms", r["stats"], file=sys.stderr, flush=True)
    del r
