#!/bin/bash
# v6 iteration: chain parity spot checks + C3 bench (+ optional ncu).  gpurun_out/c6q/
O=gpurun_out/c6q; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "chain4 or rollout_c or C3" > $O/parity.log 2>&1; echo "rc $?" >> $O/parity.log
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain6_step -s 1 -c 1 \
    -o $O/ncu_C3 -f python scripts/prof_run.py C3 4096 2 > $O/ncu_C3.log 2>&1
fi
tail -n 3 $O/parity.log; python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print('C3', d['ms_per_step'], d['value'])"
