#!/bin/bash
# ncu --set full captures of the top kernels (one launch each), reports to gpurun_out/
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain4_step -s 0 -c 1 \
  -o gpurun_out/${TAG}_C3_chain4 -f python scripts/prof_run.py C3 4096 1 > gpurun_out/${TAG}_ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_step|k_tree" -s 1 -c 1 \
  -o gpurun_out/${TAG}_C4 -f python scripts/prof_run.py C4 4096 2 > gpurun_out/${TAG}_ncu_c4.log 2>&1
ls -la gpurun_out
