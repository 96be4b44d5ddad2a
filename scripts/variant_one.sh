#!/bin/bash
# Variant library with ONE translation unit rebuilt with extra flags, the rest
# taken from build/*.o:  scripts/variant_one.sh NAME SRC.cu -DFOO=1 ... -> build/var_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
ARCH="-gencode arch=compute_100a,code=sm_100a"
F="-O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -Iinclude -Ipaper_1709_04145_b200/csrc"
mkdir -p build/var_$name
nvcc $ARCH $F "$@" -c paper_1709_04145_b200/csrc/$src -o build/var_$name/$src.o
objs=""
for o in build/*.o; do b=$(basename $o); [ "$b" = "$src.o" ] || objs="$objs $o"; done
nvcc $ARCH -shared -o build/var_$name.so $objs build/var_$name/$src.o
echo build/var_$name.so
