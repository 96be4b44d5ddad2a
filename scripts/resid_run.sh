#!/bin/bash
# residual/energy CTA kernel iteration: parity + C5/C3LM bench + phase clocks.  gpurun_out/rs/
O=gpurun_out/rs; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_resid.py tests/test_gpu_energy_lm.py tests/test_gpu_fullsize.py -q -x -k "resid or energy or C5 or lm" > $O/parity.log 2>&1; echo "rc $?" >> $O/parity.log
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_C5.json 2>/dev/null
timeout 900 python bench.py --config C3LM --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C3LM.json 2>/dev/null
PBAD_GPU_LIB=build/var_phase.so timeout 300 python scripts/prof_run.py C3LM 148 2 2>&1 | tail -2 > $O/phase.log
PBAD_GPU_LIB=build/var_phase.so timeout 300 python scripts/prof_run.py C5 148 1 2>&1 | tail -2 >> $O/phase.log
tail -n 2 $O/parity.log; cat $O/phase.log
for f in $O/bench_*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['mean_iterations_per_step'])"); done
