#!/bin/bash
# Quick GPU check (run under gpurun from the repo root): GPU tests, then the
# bench lines of the given configs without the CPU baseline.
# Usage: tools/quick_cycle.sh [cfg...]   (default: cfg1 cfg2 cfg3)
CFGS=${@:-cfg1 cfg2 cfg3}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
for c in $CFGS; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "import json;d=json.load(open(\"gpurun_out/bench_$c.json\"));print(\"$c\",d[\"value\"],d[\"roofline\"][\"step_kernels_ms\"],d[\"e2e\"][\"value\"])"; done
