#!/bin/bash
# Round-end evidence on the GPU box (run under gpurun from the repo root):
# every config's bench line (with the CPU baseline), the reference arm, the
# cfg1 launch list and one full ncu capture of the cfg1 search kernels.
mkdir -p gpurun_out/refresh
O=gpurun_out/refresh
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests_exit=$? >> $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for c in cfg1 cfg0 cfg2 cfg3 cfg4; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_cfg1.csv $CMD > $O/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1|emit|scan" -s 9 -c 3 -o $O/prof_cfg1 $CMD > $O/ncu2.log 2>&1
echo ncu_exit=$? >> $O/ncu2.log
