#!/bin/bash
# segments vs pieces work split across head geometries (graph-timed step)
for cfg in "--heads 16 --dim 128" "--heads 32 --dim 128" "--heads 32 --dim 64" "--heads 48 --dim 128" "--heads 12 --dim 128"; do
  for P in segments pieces; do
    ZGLA_PLAN=$P python bench.py $cfg --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$P', round(d['ms_per_step'],4), round(d['value']/1e6,2), 'Mtok/s')"
  done
done
