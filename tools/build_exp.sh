#!/bin/bash
# build an experimental libstkb200 variant: tools/build_exp.sh <name> [-DFOO ...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
od=exp/obj_$name; mkdir -p $od
srcs="star_f32_r1 star_f32_r2 star_f32_r3 star_f32_r4 star_f64_r1 star_f64_r2 star_f64_r3 star_f64_r4 star_dispatch star_tb star_exact box_exact star2d expr_kernels stkb200"
for s in $srcs; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include -DSTKB_VARIANTS=${STKB_BUILD_VARIANTS:-1} "$@" -c paper_2309_04671_b200/csrc/$s.cu -o $od/$s.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $od/*.o -o exp/$name.so
echo exp/$name.so
