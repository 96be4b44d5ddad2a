# chain6 A/B: default build vs variants (C3, 4 steps), plus a parity spot check
for v in default kb16; do
  if [ $v = default ]; then L=""; else L="PBAD_GPU_LIB=build/var_$v.so"; fi
  env $L timeout 300 python bench.py --config C3 --steps 4 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/r2_c6ab.log
done
PBAD_GPU_CHAIN_V6=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "v6 or rollout or matches" 2>&1 | tail -3 >> gpurun_out/r2_c6ab.log
