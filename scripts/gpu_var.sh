#!/bin/bash
# compare compile variants var/<name>/libzeco_gla.so against the in-tree build (graph bench + trace)
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="ZGLA_LIB=var/$v/libzeco_gla.so"; fi
  env $L python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'ms/step', round(d['ms_per_step'],4), d['phase_ms'])"
  env $L python scripts/trace_pipeline.py 77 2>&1 | grep -A0 "STEADY bwd\|CTAS bwd"
done
