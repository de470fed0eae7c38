#!/bin/bash
# graph-bench step time of compile variants var/<name> vs the in-tree build, interleaved twice
for r in 1 2; do
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="ZGLA_LIB=var/$v/libzeco_gla.so"; fi
  env $L python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms']; print('$v', 'ms/step', round(d['ms_per_step'],4), 'fo', p['fwd_output'], 'bo', p['bwd_output'])"
done; done
