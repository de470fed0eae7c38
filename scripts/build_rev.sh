#!/bin/bash
# build_rev.sh REV NAME : libzeco_gla.so of git revision REV into var/NAME/ (same-box A/B against HEAD)
set -e
REV=$1; NAME=$2; T=$(mktemp -d)
mkdir -p $T/paper_2507_01004_b200/csrc $T/include
for f in $(git ls-tree --name-only $REV paper_2507_01004_b200/csrc/) include/zeco_gla.h; do git show $REV:$f > $T/$f; done
OUT=var/$NAME; mkdir -p $OUT
for f in $T/paper_2507_01004_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DZGLA_BUILD -c $f -o $T/$b.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libzeco_gla.so $T/*.o -lcuda
rm -rf $T; echo built $OUT/libzeco_gla.so
