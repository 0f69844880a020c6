#!/bin/bash
# usage: tools/build_variant.sh NAME -DFLAG=.. ...  -> variants/libpssgp_NAME.so (thread path only)
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
     -DPSSGP_NO_WIDE "$@" -o variants/libpssgp_$name.so paper_2102_09964_b200/csrc/pssgp_api.cu paper_2102_09964_b200/csrc/pssgp_f32.cu
cuobjdump --dump-resource-usage variants/libpssgp_$name.so 2>/dev/null | grep -A1 "ILi3ELi0EEEvNS_7KParams" | \
  grep -o "Function _ZN5pssgp[0-9]*[a-z_]*\|REG:[0-9]*\|STACK:[0-9]*\|LOCAL:[0-9]*" | paste - - - - | sed "s/^/$name /"
