#!/bin/bash
# A/B build: libgpuim_<name>.so = the in-tree objects with one source (SRC,
# default refine_fused) recompiled under extra defines; select it with
# GIM_LIB_NAME=libgpuim_<name>.so
# usage: [SRC=initial] scripts/build_variant.sh mb2 -DGIM_FUSED_MIN_BLOCKS=2
set -e
NAME=$1; shift
cd "$(dirname "$0")/.."
python -c "from paper_2510_12196_b200.build import build; build()"
mkdir -p build/obj_$NAME
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I include -I paper_2510_12196_b200/csrc "$@" \
  -c paper_2510_12196_b200/csrc/${SRC:-refine_fused}.cu -o build/obj_$NAME/${SRC:-refine_fused}.o
objs=$(ls build/obj/*.o | grep -v ${SRC:-refine_fused}.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2510_12196_b200/libgpuim_$NAME.so \
  $objs build/obj_$NAME/${SRC:-refine_fused}.o -lcudart
ls -la paper_2510_12196_b200/libgpuim_$NAME.so
