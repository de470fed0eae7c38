#!/bin/bash
# host-buffer pipeline: gpu tests + e2e group sweep
python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -4
for G in 1 4 8 16; do
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 5 --e2e-groups $G > gpurun_out/bench_e2e_$G.json 2> gpurun_out/bench_e2e_$G.err
  python -c "import json; d=json.load(open('gpurun_out/bench_e2e_$G.json')); print('G=$G', 'ms/step', round(d['ms_per_step'],4), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'e2e tok/s', round(d['e2e']['value']))" || tail -5 gpurun_out/bench_e2e_$G.err
done
