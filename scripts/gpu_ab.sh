#!/bin/bash
# A/B: gpu tests, then bench with and without an env toggle (default ZGLA_PDL)
VAR=${1:-ZGLA_PDL}
python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3
for v in 0 1 0 1; do
  env $VAR=$v python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$VAR=$v', 'ms/step', round(d['ms_per_step'],4), d['phase_ms'])" || tail -3 gpurun_out/ab_$v.err
done
