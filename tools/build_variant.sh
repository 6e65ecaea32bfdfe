#!/bin/bash
# Build an experimental variant of libhydro.so with extra -D defines into
# paper_2104_11404_b200/_build/var/NAME.so (for tools/ab_lib.py); the in-tree library is
# untouched.   usage: bash tools/build_variant.sh NAME [-DFOO=1 ...]
set -e
NAME=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_2104_11404_b200
D=$P/_build/var; mkdir -p $D
[ -n "$NOBUILD" ] || python -c "import sys; sys.path.insert(0, '$P'); import build; build.build()" > /dev/null
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
  -Xcompiler -fPIC -Xptxas -v "$@" -c $P/csrc/hydro_api.cu -o $D/$NAME.o > $D/$NAME.ptxas.log 2>&1
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/$NAME.so $D/$NAME.o \
  $P/_build/tables.cpp.o -Xlinker --no-undefined
grep -A2 "Compiling entry function '_ZN2hk14force2d_kernelILb0ELi0ELb0ELb0E" $D/$NAME.ptxas.log | grep spill
