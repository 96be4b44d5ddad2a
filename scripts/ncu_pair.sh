#!/bin/bash
# two ncu --set full captures per call (reports stay under gpurun's 64 MiB copy-back):
#   scripts/ncu_pair.sh TAG1 REGEX1 SKIP1 "ARGS1" TAG2 REGEX2 SKIP2 "ARGS2"
O=gpurun_out/ncu; mkdir -p $O
while [ $# -ge 4 ]; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $O/$1 -f python scripts/prof_run.py $4 > $O/$1.log 2>&1
  shift 4
done
ls -la $O
