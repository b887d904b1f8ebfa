"""Per-call e2e breakdown of repeated cfg1 searches; prints the slow calls."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_22901_b200 as cv  # noqa: E402
from paper_2507_22901_b200 import workloads as W  # noqa: E402

ctx = cv.Context(0)
w = W.cfg1()
r = ctx.search(w.targets, w.patterns, w.v_th, w.r_novib, w.radii, w.angles)
del r
rows = []
for i in range(60):
    t = time.perf_counter()
    r = ctx.search(w.targets, w.patterns, w.v_th, w.r_novib, w.radii, w.angles)
    t1 = time.perf_counter()
    st = r["stats"]
    del r
    t2 = time.perf_counter()
    rows.append(((t1 - t) * 1e3, (t2 - t1) * 1e3, st["total_ms"], st["prep_ms"], st["h2d_ms"], st["device_ms"], st["d2h_ms"]))
med = statistics.median(x[0] for x in rows)
print(f"median call {med:.3f} ms")
for i, x in enumerate(rows):
    if x[0] > 1.3 * med or x[1] > 0.1:
        print(i, " ".join(f"{v:.3f}" for v in x))
