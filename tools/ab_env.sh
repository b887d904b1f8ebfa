#!/bin/bash
# Quick A/B of env settings on plan timings (run under gpurun from the repo
# root).  Usage: tools/ab_env.sh "cfg2 cfg1" "CVG_EMIT_SHIFT=9" "CVG_EMIT_SHIFT=10" ...
CFGS=$1; shift
for c in $CFGS; do
  for e in "$@"; do
    echo "== $c $e"; env $e timeout 300 python tools/prof_plan.py $c --runs 5 2>&1 | tail -2
  done
done
