#!/bin/bash
# A/B of compile variants: fast-path GPU tests with the in-tree build, then interleaved graph-timed
# bench runs of the in-tree build ("new") and var/<name>/libzeco_gla.so for each name given
# usage: gpu_libab.sh [--tests "pytest args"] name...
TESTS="tests/test_gpu_fast.py tests/test_gpu_pdl.py"
if [ "$1" = "--tests" ]; then TESTS=$2; shift 2; fi
[ -n "$TESTS" ] && python -m pytest $TESTS -q -x --timeout 600 2>&1 | tail -2
for rep in 1 2 3; do
  for v in new "$@"; do
    if [ $v = new ]; then L=""; else L="ZGLA_LIB=var/$v/libzeco_gla.so"; fi
    env $L python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-variants --e2e-steps ${E2E_STEPS:-2} > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
    python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', 'ms/step', round(d['ms_per_step'],4), d['phase_ms'], 'e2e', round(d['e2e']['ms_per_step'],3))" || tail -3 gpurun_out/ab_$v.err
  done
done
