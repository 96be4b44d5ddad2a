#!/bin/bash
# A/B runs: default lib and variants on C5/C4 (bench legs, short)
mkdir -p gpurun_out
run() { # tag lib config steps warmup
  if [ -n "$2" ]; then export PBAD_GPU_LIB=$2; else unset PBAD_GPU_LIB; fi
  timeout 300 python bench.py --config $3 --steps $4 --warmup $5 --no-cpu-baseline > gpurun_out/ab_$1.out 2> gpurun_out/ab_$1.err
}
run c5_default "" C5 2 1
run c5_cholreg build/var_cholreg.so C5 1 1
run c5_cholsm build/var_cholsm.so C5 1 1
run c4_default "" C4 3 2
run c4_noinline build/var_cholreg.so C4 3 2
