#!/bin/bash
# A/B of the strip tiles on cfg4 (kernel time), then the parity tests that cover them.
for v in 0 1 1; do CVG_STRIPS=$v timeout 300 python tools/prof_plan.py cfg4 --runs 5 2>&1 | sed "s/^/strips=$v /"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "column or strip or cfg4 or memo or pair_view or cfg1 or cfg0 or audit or edge" 2>&1 | tail -3
