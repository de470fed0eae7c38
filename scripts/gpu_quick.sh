#!/bin/bash
# quick check after a kernel change: parity tests of the fast path, one-CTA trace, graph bench
python -m pytest tests/test_gpu_fast.py tests/test_gpu_engine.py tests/test_gpu_host.py -q -x 2>&1 | tail -2
python scripts/trace_pipeline.py 77 2>&1 | tail -6
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'],4), d['phase_ms'])"
