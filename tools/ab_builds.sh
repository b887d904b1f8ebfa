#!/bin/bash
# A/B of package builds in one GPU run (run under gpurun from the repo root):
# each _exp/<name>/ holds a copy of paper_2507_22901_b200/ (with its .so
# files); "cur" is the working tree.  Usage: tools/ab_builds.sh "cfg1 cfg4" base cur
CFGS=$1; shift
for rep in 1 2; do
for c in $CFGS; do
  for b in "$@"; do
    root=$PWD; [ "$b" != cur ] && root=$PWD/_exp/$b
    echo "== $c $b"; CVG_PKG_ROOT=$root timeout 300 python tools/prof_plan.py $c --runs 5 2>&1 | tail -2
  done
done
done
