#!/bin/bash
# Round-2 measurement cycle on the GPU box (run under gpurun from the repo
# root): GPU tests, the default bench line (cfg4 + the other configs), the
# reference arm.  Usage: tools/r02_cycle.sh [pytest-args...]
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?
tail -c 600 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_exit=$?
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], d["roofline"]["step_kernels_ms"])
print("memo", d.get("memoized", {}).get("nominal_value"), d.get("memoized", {}).get("wall_s"))
print("cpu", d["cpu_baseline"]["value"], d["cpu_baseline"].get("memoized", {}).get("nominal_value"))
for k, v in d.get("configs", {}).items():
    print(k, v["value"], v["e2e"]["value"], v["phase_ms"], v.get("roofline_frac_phase1"), v.get("cpu_baseline", {}).get("value"))
r = json.load(open("gpurun_out/bench_ref.json"))
print("ref", r["value"], r.get("memoized", {}).get("nominal_value"))
PY
