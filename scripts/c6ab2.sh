#!/bin/bash
# chain6 A/B on C3: default library vs build/var_<name>.so variants, then the
# chain parity tests on each variant.  Output: gpurun_out/c6ab2/
O=gpurun_out/c6ab2; mkdir -p $O
for v in default ${VARS:-}; do
  if [ $v = default ]; then L=""; else L="PBAD_GPU_LIB=build/var_$v.so"; fi
  env $L timeout 400 python bench.py --config C3 --steps 4 --warmup 3 --no-cpu-baseline > $O/bench_$v.json 2> $O/bench_$v.err
  python -c "import json; d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'], d['clocks'])" >> $O/summary.txt 2>&1
done
for v in ${PVARS:-}; do
  PBAD_GPU_LIB=build/var_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "chain4 or rollout_c or C3 or v6" > $O/parity_$v.log 2>&1; echo "$v parity rc $?" >> $O/summary.txt
  tail -2 $O/parity_$v.log >> $O/summary.txt
done
cat $O/summary.txt
