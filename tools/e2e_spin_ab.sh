nproc; lscpu | grep -i "thread\|core\|socket\|model name" | head -5
for rep in 1 2; do for sp in 0 200; do
  CVG_POOL_SPIN_US=$sp python - <<'PY'
import os, time, numpy as np, statistics
import paper_2507_22901_b200 as cv
from paper_2507_22901_b200 import workloads as W
ctx = cv.Context(0)
for name in ("cfg1", "cfg3"):
    w = getattr(W, name)()
    r = ctx.search(w.targets, w.patterns, w.v_th, w.r_novib, w.radii, w.angles); del r
    ts, lib = [], []
    for i in range(30):
        t = time.perf_counter()
        r = ctx.search(w.targets, w.patterns, w.v_th, w.r_novib, w.radii, w.angles)
        _ = int(r["n_pairs"])
        ts.append(time.perf_counter() - t); lib.append(r["stats"]["total_ms"])
        del r
    print(f"spin={os.environ['CVG_POOL_SPIN_US']} {name}: wall mean {1e3*statistics.mean(ts):.3f} med {1e3*statistics.median(ts):.3f} max {1e3*max(ts):.3f} | lib mean {statistics.mean(lib):.3f}", flush=True)
PY
done; done
