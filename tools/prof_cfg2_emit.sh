#!/bin/bash
# ncu --set full of cfg2's lists + emit kernels (run under gpurun).
O=gpurun_out/prof2; mkdir -p $O
timeout 300 python tools/prof_plan.py cfg2 --runs 3 > $O/plain.log 2>&1; echo plain=$?; cat $O/plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lists|emit" -s 4 -c 2 -o $O/cfg2_le python tools/prof_plan.py cfg2 --runs 3 > $O/ncu.log 2>&1; echo ncu=$?
python tools/ncu_summary.py $O/cfg2_le.ncu-rep --blocks -o $O/ncu_cfg2_le.json
ls -la $O
find $O -name "*.ncu-rep" -size +60M -delete
