#!/bin/bash
# energy-form LM on the CTA kernel: parity tests + C3LM bench.  gpurun_out/elm/
O=gpurun_out/elm; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_energy_lm.py -q -x > $O/parity.log 2>&1; echo "rc $?" >> $O/parity.log
timeout 1200 python -m pytest tests/test_gpu_resid.py tests/test_gpu_tree.py -q -x > $O/regress.log 2>&1; echo "rc $?" >> $O/regress.log
timeout 900 python bench.py --config C3LM --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_C3LM.json 2> $O/bench_C3LM.err
tail -n 3 $O/parity.log $O/regress.log; tail -c 600 $O/bench_C3LM.json; tail -3 $O/bench_C3LM.err
