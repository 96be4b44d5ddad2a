#!/bin/bash
# v7 quick: C3 bench (v7 vs v6), parity spot check, optional ncu.  gpurun_out/c7q/
O=gpurun_out/c7q; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain4 or rollout_c3" > $O/parity.log 2>&1; echo "rc $?" >> $O/parity.log
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_v7.json 2> $O/bench_v7.err
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain7_step -s 1 -c 1 \
    -o $O/ncu_C3_v7 -f python scripts/prof_run.py C3 4096 2 > $O/ncu_C3.log 2>&1
fi
tail -n 3 $O/parity.log; tail -n 1 $O/bench_v7.json | cut -c 1-400
