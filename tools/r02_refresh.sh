#!/bin/bash
# Round-2 ncu evidence (run under gpurun from the repo root): the headline
# bench's launch list, and one full capture of each config's kernels.
O=gpurun_out/refresh; mkdir -p $O
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-others --e2e-steps 1"
timeout 600 $CMD > $O/plain.json 2> $O/plain.err; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg4.csv $CMD > $O/ncu_l.log 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"phase1" -s 2 -c 1 -o $O/full_cfg4 python tools/prof_plan.py cfg4 > $O/ncu_cfg4.log 2>&1; echo cfg4=$?
for c in cfg1 cfg3 cfg2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1|lists|scan|emit" -s 8 -c 4 -o $O/full_$c python tools/prof_plan.py $c --runs 3 > $O/ncu_$c.log 2>&1; echo $c=$?
done
ls -la $O
# summaries on the box (the .ncu-rep files exceed gpurun's copy-back limit)
for c in cfg4 cfg1 cfg3 cfg2; do python tools/ncu_summary.py $O/full_$c.ncu-rep --blocks -o $O/ncu_full_$c.json; done
python tools/ncu_summary.py --launches $O/launches_cfg4.csv -o $O/ncu_launches_cfg4.json
rm -f $O/*.ncu-rep
