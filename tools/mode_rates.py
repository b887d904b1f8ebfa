import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2507_22901_b200 as cv
from paper_2507_22901_b200 import workloads as W
ctx = cv.Context(0)
wl = W.cfg1()
for mode, basis in ((0, 0), (0, 1), (1, 0), (1, 1)):
    args = (wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles)
    ctx.search(*args, output="counts", delta_mode=mode, delta_basis=basis)
    best = 1e9; ks = None
    for _ in range(3):
        t0 = time.perf_counter(); res = ctx.search(*args, output="counts", delta_mode=mode, delta_basis=basis)
        best = min(best, time.perf_counter() - t0); ks = res["stats"]
    print(f"mode={mode} basis={basis} pairs={int(res['counts'].sum())} wall={best*1e3:.2f}ms "
          f"Gcand/s(wall)={wl.candidates/best/1e9:.1f} stats={ks}")
