#!/bin/bash
# Per-kernel durations (ncu launch list) of one config's plan runs, summarized
# per kernel name.  Usage (under gpurun): tools/launch_times.sh cfg2 [runs]
c=$1; runs=${2:-2}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lt_$c.csv \
  python tools/prof_plan.py $c --runs $runs ${LT_ARGS} > /dev/null 2>&1
python - "$c" <<'PY'
import csv, sys, collections
c = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/lt_{c}.csv")) if len(r) > 10]
h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value"); iu = h.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[iv].replace(",", "")); v *= {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1.0)
    d[r[ik].split("(")[0].split("::")[-1]].append(v)
for k, v in d.items():
    print(c, k, "n", len(v), "median_us", round(sorted(v)[len(v) // 2], 1))
PY
