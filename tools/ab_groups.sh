#!/bin/bash
# A/B of the PAIRS strip tiles (kernel time per config, phase split).
for c in cfg0 cfg1 cfg3 cfg2 cfg4; do for v in 0 1; do CVG_STRIPS=$v timeout 300 python tools/prof_plan.py $c --runs 5 2>&1 | tail -2 | sed "s/^/strips=$v /"; done; done
[ "$1" = "tests" ] && timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
