#!/bin/bash
# usage: ncu_one.sh TAG KERNEL_REGEX CONFIG B STEPS [SKIP] [MAXIT] -> gpurun_out/TAG.ncu-rep
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${6:-1} -c 1 \
  -o gpurun_out/$1 -f python scripts/prof_run.py $3 $4 $5 $7 > gpurun_out/$1.log 2>&1
