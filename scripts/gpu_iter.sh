#!/bin/bash
# quick iteration: gpu tests + bench (no ncu)
python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -4
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
python -c "import json; d=json.load(open('gpurun_out/bench_iter.json')); print('ms/step', d['ms_per_step'], 'tok/s', d['value'], d['phase_ms'], 'step frac', d['roofline_step']['frac'])" || tail gpurun_out/bench_iter.err
python scripts/trace_pipeline.py 77 2>&1 | tail -26
