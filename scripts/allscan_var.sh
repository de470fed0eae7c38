#!/bin/bash
# All-Scan compile variants built ON the box (var/ does not travel): name -> flags, virtual P=8 latency
build() { # name flags...
  local n=$1; shift; mkdir -p /tmp/v_$n
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DZGLA_BUILD "$@" -c paper_2507_01004_b200/csrc/allscan.cu -o /tmp/v_$n/allscan.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/v_$n/libzeco_gla.so /tmp/v_$n/allscan.o $(ls build/*.o | grep -v allscan) -lcuda
}
build base & build w4c2 -DZGLA_AS_WPT=4 -DZGLA_AS_LIST_CAP=2048 & build w2c2 -DZGLA_AS_WPT=2 -DZGLA_AS_LIST_CAP=2048 & build w4 -DZGLA_AS_WPT=4 & build b2 -DZGLA_AS_BATCH=2 -DZGLA_AS_WPT=4 -DZGLA_AS_LIST_CAP=2048 &
wait
for v in base w4c2 w2c2 w4 b2; do
  ZGLA_LIB=/tmp/v_$v/libzeco_gla.so python scripts/allscan_bench.py --virtual 8 --iters 10 2>&1 | python -c "
import json,sys
r=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print('$v', ' '.join(f\"{d['H']}x{d['d']}:{d['allscan_us_mean']:.1f}\" for d in r if d['K']==4))"

done
