"""Host/device timeline of repeated end-to-end searches (CVG_TRACE=1)."""
import os
import sys
import time

import numpy as np

os.environ.setdefault("CVG_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_22901_b200 as cv  # noqa: E402
from paper_2507_22901_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
w = getattr(W, name)()
ctx = cv.Context(0)
res = None
for i in range(8):
    t = time.perf_counter()
    res = ctx.search(w.targets, w.patterns, w.v_th, w.r_novib, w.radii, w.angles, output=w.output)
    dt = time.perf_counter() - t
    print(f"call {i}: {dt * 1e3:.3f} ms  stats total {res['stats']['total_ms']:.3f}", file=sys.stderr, flush=True)
