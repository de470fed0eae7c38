#!/bin/bash
# full round evidence: tests, smoke, bench, launch list, ncu captures, all-scan virtual bench
python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; cat gpurun_out/bench_full.json | head -c 600; echo
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; head -c 400 gpurun_out/bench_ref.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 24 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
for k in bwd_out_kernel fwd_out_kernel seg_state_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
python scripts/allscan_bench.py --virtual 8 --iters 20 > gpurun_out/allscan_virtual.jsonl 2>&1; tail -3 gpurun_out/allscan_virtual.jsonl
ls gpurun_out
