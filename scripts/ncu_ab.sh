#!/bin/bash
# isolated (ncu, cold cache) kernel times of the in-tree build vs var/<name>
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="ZGLA_LIB=var/$v/libzeco_gla.so"; fi
  env $L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bwd_out|fwd_out|seg_state" -s 6 -c 8 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import sys,csv
r=[x for x in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h=r[0]; i=h.index('Kernel Name'); j=h.index('Metric Value')
from collections import defaultdict
t=defaultdict(list)
for x in r[1:]: t[x[i].split('(')[0][-22:]].append(float(x[j]))
print('$v', {k: round(sum(v)/len(v)/1000,1) for k,v in t.items()})"
done
