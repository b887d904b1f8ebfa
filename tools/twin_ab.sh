#!/bin/bash
# Twin tiles A/B (run under gpurun from the repo root): the twin / PAIRS
# parity tests, then cfg2 (and cfg1 / cfg3) bench lines with twins on / off.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "twin or cfg2_fine or huge_single or plan_overflow or strip_tiles or cfg1_full or cfg3" > gpurun_out/twin_tests.log 2>&1; echo tests_exit=$?; tail -3 gpurun_out/twin_tests.log
for tw in 1 0; do
  for c in cfg2 cfg1; do
    CVG_TWIN=$tw timeout 600 python bench.py --config $c --no-cpu-baseline --no-others --e2e-steps 1 > gpurun_out/twin${tw}_$c.json 2> gpurun_out/twin${tw}_$c.err
    python -c "import json;d=json.load(open('gpurun_out/twin${tw}_$c.json'));print('twin=$tw $c',d['value'],d['roofline']['step_kernels_ms'])"
  done
done
