#!/bin/bash
# session-3 closing evidence: GPU tests, smoke, bench, reference arm, launch list, full ncu captures of
# the three fused kernels, All-Scan virtual-rank bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -4 > gpurun_out/gputests.txt; cat gpurun_out/gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; head -c 400 gpurun_out/bench_full.json; echo
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; head -c 300 gpurun_out/bench_ref.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 24 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-variants --e2e-steps 1 > /dev/null 2>&1
for k in bwd_out_kernel fwd_out_kernel seg_state_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants --e2e-steps 1 > /dev/null 2>&1
done
python scripts/allscan_bench.py --virtual 8 --iters 20 > gpurun_out/allscan_virtual.jsonl 2>&1; tail -3 gpurun_out/allscan_virtual.jsonl
ls gpurun_out
