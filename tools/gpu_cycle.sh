#!/bin/bash
# One measurement cycle on the GPU box (run under gpurun from the repo root):
# GPU tests, bench (cfg1), launch list and one full ncu capture of the search
# kernels.  Usage: tools/gpu_cycle.sh <tag> [pytest-args...]
TAG=${1:-cycle}; shift
timeout 1200 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1|emit|scan" -s 9 -c 3 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu2.log 2>&1
echo ncu_exit=$? >> gpurun_out/ncu2.log
