#!/bin/bash
# e2e (host-buffer call) ms/step for several head-group counts, interleaved twice on one box
for r in 1 2; do for G in "$@"; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variants --e2e-steps 10 --e2e-groups $G 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('G=$G e2e ms', round(d['e2e']['ms_per_step'],3))"
done; done
