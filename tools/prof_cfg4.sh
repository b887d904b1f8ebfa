#!/bin/bash
# ncu --set full of cfg4's phase-1 kernel (run under gpurun); summary with the
# hottest basic blocks into gpurun_out/prof4/.
O=gpurun_out/prof4; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1" -s 2 -c 1 -o $O/cfg4 python tools/prof_plan.py cfg4 --runs 2 > $O/ncu.log 2>&1; echo ncu=$?
python tools/ncu_summary.py $O/cfg4.ncu-rep --blocks -o $O/ncu_cfg4.json
find $O -name "*.ncu-rep" -size +60M -delete
