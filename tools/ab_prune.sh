#!/bin/bash
# fast vs pruned per config (kernel time), then the GPU tests
for c in cfg1 cfg3 cfg2 cfg4; do for p in fast pruned; do timeout 300 python tools/prof_plan.py $c --runs 3 --path $p 2>&1 | tail -2 | sed "s/^/$p /"; done; done
[ "$1" = "tests" ] && timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
true
