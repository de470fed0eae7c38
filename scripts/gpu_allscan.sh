#!/bin/bash
# All-Scan protocol tests + virtual-rank latency sweep (config 4 shape)
python -m pytest tests/test_gpu_allscan_spmd.py tests/test_gpu_spmd_ipc.py tests/test_gpu_generic.py tests/test_gpu_engine.py -q -x --timeout 600 2>&1 | tail -2
python scripts/allscan_bench.py --virtual 8 --iters 30 > gpurun_out/allscan_virtual8.jsonl 2>&1
python scripts/allscan_bench.py --virtual 4 --iters 30 > gpurun_out/allscan_virtual4.jsonl 2>&1
python scripts/allscan_bench.py --virtual 2 --iters 30 > gpurun_out/allscan_virtual2.jsonl 2>&1
python scripts/allscan_bench.py --virtual 1 --iters 30 > gpurun_out/allscan_virtual1.jsonl 2>&1
python - <<'PY'
import json
for P in (1, 8):
    for l in open(f"gpurun_out/allscan_virtual{P}.jsonl"):
        if not l.startswith("{"): print(l.strip()); continue
        d = json.loads(l)
        if d["K"] in (1, 4, 16, 128): print(P, d["H"], d["d"], d["K"], round(d["allscan_us_mean"], 2), round(d["allscan_us_best"], 2))
PY
