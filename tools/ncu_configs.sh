O=gpurun_out/ncucfg; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "edge_grids or continuous or frame_diff" > $O/edge_tests.log 2>&1; echo tests_exit=$? >> $O/edge_tests.log; tail -3 $O/edge_tests.log
for c in cfg2 cfg3 cfg4; do
  timeout 900 ncu --set full --clock-control none -k regex:"phase1" -s 3 -c 1 -o $O/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_$c.log 2>&1; echo $c ncu=$?
done
