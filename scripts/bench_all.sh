#!/bin/bash
# Bench lines for every config (bench.py defaults per config), plus the ncu
# launch list of the default bench command (C3).  Outputs in gpurun_out/.
mkdir -p gpurun_out
for c in C1 C2 C4 C4b C5; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 > gpurun_out/bench_all_$c.json 2> gpurun_out/bench_all_$c.err
done
timeout 900 python bench.py > gpurun_out/bench_all_C3.json 2> gpurun_out/bench_all_C3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/launches_C3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
