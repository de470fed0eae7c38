#!/bin/bash
# graph step + all eager phases, in-tree vs var/<name>, interleaved twice
for r in 1 2; do for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="ZGLA_LIB=var/$v/libzeco_gla.so"; fi
  env $L python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms']; print('$v', round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in p.items()})"
done; done
