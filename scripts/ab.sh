#!/bin/bash
# A/B runs of library variants (bench legs, short); outputs gpurun_out/ab_<tag>.out
mkdir -p gpurun_out
run() { # tag lib config steps warmup
  if [ -n "$2" ]; then export PBAD_GPU_LIB=$2; else unset PBAD_GPU_LIB; fi
  timeout 300 python bench.py --config $3 --steps $4 --warmup $5 --no-cpu-baseline > gpurun_out/ab_$1.out 2> gpurun_out/ab_$1.err
}
for spec in "$@"; do
  IFS=: read tag lib cfg steps warm <<< "$spec"
  run $tag "$lib" $cfg $steps $warm
done
