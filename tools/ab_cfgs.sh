#!/bin/bash
# Kernel time per config (phase split) of the current build; "tests" also runs the GPU suite.
for c in cfg0 cfg1 cfg3 cfg2 cfg4; do timeout 300 python tools/prof_plan.py $c --runs 5 2>&1 | tail -2; done
if [ "$1" = "tests" ]; then timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3; fi
true
