#!/bin/bash
# like gpu_var2.sh, printing every phase (fwd_local / bwd_local include the segment scans)
for r in 1 2; do
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="ZGLA_LIB=var/$v/libzeco_gla.so"; fi
  env $L python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms']; print('$v', 'ms/step', round(d['ms_per_step'],4), ' '.join(f'{k}={v:.4f}' for k,v in p.items()))"
done; done
