#!/bin/bash
# ncu evidence for round 2 (run under gpurun): launch list of the headline
# bench, full captures of phase 1 (cfg4, cfg1) and of phase 1 + emit (cfg2).
O=gpurun_out/prof; mkdir -p $O
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-others --e2e-steps 1"
timeout 600 $CMD > $O/plain.json 2> $O/plain.err; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg4.csv $CMD > $O/ncu_l.log 2>&1; echo launches=$?
for c in cfg4 cfg1; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1" -s 2 -c 1 -o $O/p1_$c python tools/prof_plan.py $c > $O/ncu_$c.log 2>&1; echo $c=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1|emit" -s 4 -c 2 -o $O/p1emit_cfg2 python tools/prof_plan.py cfg2 > $O/ncu_cfg2.log 2>&1; echo cfg2=$?
ls -la $O
