#!/bin/bash
# cfg4 end-to-end call time (cvg_search, host arrays in, results out) vs the
# number of pipelined search ranges (CVG_PIPELINE_K) and ramp / even / shaped
# bounds (cvg_search.cpp: ramp_bounds, shaped_bounds).
# Usage (under gpurun, repo root): tools/sweep_ranges_cfg4.sh [K...]
KS=${@:-4 6 8 10 12 16 24}
for k in $KS; do
  for even in 0 1 shaped; do
    unset CVG_PIPELINE_EVEN; export CVG_RANGE_SHAPE=0
    if [ "$even" = 1 ]; then export CVG_PIPELINE_EVEN=1; fi
    if [ "$even" = shaped ]; then export CVG_RANGE_SHAPE=1; fi
    CVG_PIPELINE_K=$k python - "$k" "$even" <<'PY'
import sys, time
import numpy as np
import paper_2507_22901_b200 as cv
from paper_2507_22901_b200 import workloads as W
w = W.cfg4()
ctx = cv.Context(0)
ts, ph = [], []
for i in range(14):
    t = time.perf_counter()
    r = ctx.search(w.targets, w.patterns, w.v_th, w.r_novib, w.radii, w.angles, output=w.output)
    _ = int(r["n_pairs"])
    ts.append(time.perf_counter() - t)
    ph.append((r["stats"]["prep_ms"], r["stats"]["device_ms"], r["stats"]["total_ms"], r["stats"]["kernel_ms"]))
    del r
ts = np.array(ts[4:]) * 1e3
ph = np.median(np.array(ph[4:]), axis=0)
print(f"cfg4 K={sys.argv[1]} bounds={sys.argv[2]}: median {np.median(ts):.2f} ms  min {ts.min():.2f}  "
      f"prep {ph[0]:.1f} device {ph[1]:.1f} total {ph[2]:.1f} kernels {ph[3]:.1f}", flush=True)
PY
  done
done
