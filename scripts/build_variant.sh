#!/bin/bash
# Build an alternative libpbad_gpu.so with extra -D flags for kernel A/B runs:
#   scripts/build_variant.sh NAME -DFOO=0 ...   ->  build/var_NAME.so
# select it at run time with PBAD_GPU_LIB=build/var_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/var_$name
ARCH="-gencode arch=compute_100a,code=sm_100a"
F="-O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -Iinclude -Ipaper_1709_04145_b200/csrc"
for s in pbad_kernels pbad_chain pbad_chain4 pbad_chain5 pbad_chain6 pbad_tree pbad_tree_lbfgs pbad_resid; do
  nvcc $ARCH $F "$@" -c paper_1709_04145_b200/csrc/$s.cu -o build/var_$name/$s.o &
done
wait
nvcc $ARCH -O2 -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-mfma -Iinclude -Ipaper_1709_04145_b200/csrc "$@" \
  -x cu -c paper_1709_04145_b200/csrc/pbad_host.cpp -o build/var_$name/pbad_host.o
nvcc $ARCH -shared -o build/var_$name.so build/var_$name/*.o
echo build/var_$name.so
