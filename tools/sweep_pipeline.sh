#!/bin/bash
# e2e time of cfg1/cfg3 vs the number of pipelined ranges (CVG_PIPELINE_K).
for cfg in cfg1 cfg3; do
  for k in 1 2 3 4 6 8; do
    for even in "" 1; do
      if [ -n "$even" ]; then export CVG_PIPELINE_EVEN=1; else unset CVG_PIPELINE_EVEN; fi
      CVG_PIPELINE_K=$k CVG_TRACE= python - "$cfg" "$k" "$even" <<'PY'
import sys, time, os
os.environ.pop("CVG_TRACE", None)
import numpy as np
import paper_2507_22901_b200 as cv
from paper_2507_22901_b200 import workloads as W
w = getattr(W, sys.argv[1])()
ctx = cv.Context(0)
ts = []
for i in range(25):
    t = time.perf_counter()
    r = ctx.search(w.targets, w.patterns, w.v_th, w.r_novib, w.radii, w.angles)
    ts.append(time.perf_counter() - t)
    del r
ts = np.array(ts[5:]) * 1e3
print(f"{sys.argv[1]} K={sys.argv[2]} even={sys.argv[3] or 0}: median {np.median(ts):.3f} ms  min {ts.min():.3f}", flush=True)
PY
    done
  done
done
