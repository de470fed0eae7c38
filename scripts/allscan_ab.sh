#!/bin/bash
# All-Scan virtual-rank latency: in-tree build vs var/prev
python -m pytest tests/test_gpu_allscan_spmd.py tests/test_gpu_generic.py tests/test_gpu_spmd_ipc.py -q -x 2>&1 | tail -1
for L in "" "ZGLA_LIB=var/prev/libzeco_gla.so"; do
  echo "== ${L:-base}"
  env $L python scripts/allscan_bench.py --virtual 8 --iters 30 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if (d['H'],d['d']) in ((16,128),(4,64)) and d['K'] in (1,4,8,16): print(d['H'],d['d'],'K',d['K'],round(d['allscan_us_mean'],1))"
done
