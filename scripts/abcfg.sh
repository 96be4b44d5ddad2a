#!/bin/bash
# A/B of library variants on one bench config:
#   CFG=C5 STEPS=2 VARS="rh1 ..." bash scripts/abcfg.sh   -> gpurun_out/abcfg/
O=gpurun_out/abcfg; mkdir -p $O
for v in default ${VARS:-}; do
  if [ $v = default ]; then L=""; else L="PBAD_GPU_LIB=build/var_$v.so"; fi
  env $L timeout 900 python bench.py --config ${CFG:-C5} --steps ${STEPS:-2} --warmup 3 --no-cpu-baseline > $O/bench_${CFG}_$v.json 2> $O/bench_${CFG}_$v.err
  python -c "import json; d=json.loads(open('$O/bench_${CFG}_$v.json').read().strip().splitlines()[-1]); print('${CFG}', '$v', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O/summary.txt 2>&1
done
cat $O/summary.txt
