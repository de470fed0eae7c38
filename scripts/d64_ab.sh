#!/bin/bash
# d = 64 step time (H=32 x 64, 16K tokens, and H=4 x 64) for the in-tree build vs variants, interleaved twice
for r in 1 2; do for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="ZGLA_LIB=var/$v/libzeco_gla.so"; fi
  for hd in "32 64" "16 128"; do set -- $hd
    env $L python bench.py --heads $1 --dim $2 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms']; print('$v', 'H=$1 d=$2', 'ms/step', round(d['ms_per_step'],4), 'fo', p['fwd_output'], 'bo', p['bwd_output'])"
  done
done; done
