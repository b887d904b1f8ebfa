#!/bin/bash
# cfg4 end-to-end call time vs the range weights (CVG_RANGE_WEIGHTS, cvg_search.cpp: shaped_bounds).
# Usage (under gpurun, repo root): tools/sweep_range_weights_cfg4.sh "1,2,4,4,4,4,2,1" ...
for w in "$@"; do
  K=$(echo "$w" | tr ',' '\n' | wc -l)
  CVG_RANGE_SHAPE=1 CVG_RANGE_WEIGHTS=$w CVG_PIPELINE_K=$K python - "$w" <<'PY'
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
print(f"cfg4 weights={sys.argv[1]}: median {np.median(ts):.2f} ms  min {ts.min():.2f}  "
      f"prep {ph[0]:.1f} device {ph[1]:.1f} total {ph[2]:.1f} kernels {ph[3]:.1f}", flush=True)
PY
done
