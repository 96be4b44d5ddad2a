#!/bin/bash
# Build a variant of libpbad_gpu.so that differs only in one translation
# unit's -D flags (the other objects come from build/, made by
# paper_1709_04145_b200.build):
#   scripts/obj_variant.sh NAME pbad_resid -DFOO=1 ...  ->  build/var_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
mkdir -p build/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  -Xptxas -v -Iinclude -Ipaper_1709_04145_b200/csrc "$@" -c paper_1709_04145_b200/csrc/$src.cu \
  -o build/var_$name/$src.cu.o > build/var_$name/ptxas.log 2>&1
objs=$(ls build/*.o | grep -v "/$src.cu.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name.so $objs build/var_$name/$src.cu.o
echo build/var_$name.so
