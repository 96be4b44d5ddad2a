#!/bin/bash
# Round-2 GPU pass: parity suite, smoke, a bench line per config (timed
# regions >= ~1 s), the launch list of the default bench command and one
# ncu --set full capture per chain kernel.  Outputs under gpurun_out/r2/.
O=gpurun_out/r2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
  for cs in C1:300 C2:50 C4:250 C4b:200 C5:2; do
    c=${cs%%:*}; k=${cs##*:}
    timeout 900 python bench.py --config $c --steps $k --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
  done
fi
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file $O/launches_C3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
  for spec in "C3 4096 k_chain6_step" "C1 1024 k_chain5_step" "C2 1024 k_chain5_step"; do
    set -- $spec
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o $O/ncu_$1 -f python scripts/prof_run.py $1 $2 2 > $O/ncu_$1.log 2>&1
  done
fi
ls -la $O
