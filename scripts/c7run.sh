#!/bin/bash
# v7 chain kernel: parity spot checks + C3 A/B against v6.  Outputs in gpurun_out/c7/.
O=gpurun_out/c7; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain4 or rollout_c" > $O/parity.log 2>&1; echo "rc $?" >> $O/parity.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k C3 > $O/fullsize.log 2>&1; echo "rc $?" >> $O/fullsize.log
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_v7.json 2> $O/bench_v7.err
PBAD_GPU_CHAIN_V6=1 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_v6.json 2> $O/bench_v6.err
for c in C1 C2; do PBAD_GPU_CHAIN_V7=1 timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_v7_$c.json 2> $O/bench_v7_$c.err; done
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain7_step -s 1 -c 1 \
    -o $O/ncu_C3_v7 -f python scripts/prof_run.py C3 4096 2 > $O/ncu_C3.log 2>&1
fi
tail -3 $O/parity.log $O/fullsize.log
