#!/bin/bash
# build_variant.sh NAME "-DFLAG ..." : libzeco_gla.so compiled with extra flags into var/NAME/ (git-ignored, travels to the GPU box)
set -e
NAME=$1; shift
OUT=var/$NAME; mkdir -p $OUT
for f in paper_2507_01004_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DZGLA_BUILD "$@" -c $f -o $OUT/$b.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libzeco_gla.so $OUT/*.o -lcuda
echo built $OUT/libzeco_gla.so
