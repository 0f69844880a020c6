#!/bin/bash
# usage: tools/build_variant_full.sh NAME -DFLAG=.. ...  -> variants/libpssgp_NAME.so (all paths incl. wide)
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
     "$@" -o variants/libpssgp_$name.so paper_2102_09964_b200/csrc/pssgp_api.cu paper_2102_09964_b200/csrc/pssgp_f32.cu
cuobjdump --dump-resource-usage variants/libpssgp_$name.so 2>/dev/null | grep -A1 "kw_.*ILi16E" | \
  grep -o "Function _ZN5pssgp4wide[0-9]*[a-z_]*\|REG:[0-9]*\|STACK:[0-9]*\|LOCAL:[0-9]*" | paste - - - - | sed "s/^/$name /"
