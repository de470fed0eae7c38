#!/bin/bash
python -m pytest tests/test_gpu_host.py -q -x 2>&1 | tail -2
for X in dma sm hyb; do for G in 4 8 16; do
  ZGLA_XFER=$X python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 --e2e-groups $G 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$X G=$G e2e ms', round(d['e2e']['ms_per_step'],3))"
done; done
ZGLA_XFER=hyb python scripts/host_trace.py 8 2>&1 | tail -9
