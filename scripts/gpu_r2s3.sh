#!/bin/bash
# session-3 baseline: full GPU suite, smoke, bench, reference arm, launch list, bwd_out ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -8 > gpurun_out/s3_gputests.txt; cat gpurun_out/s3_gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; head -c 3000 gpurun_out/s3_bench.json; echo
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s3_bench_ref.json 2>&1; head -c 1500 gpurun_out/s3_bench_ref.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 24 --csv --log-file gpurun_out/s3_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_out_kernel -s 2 -c 1 -o gpurun_out/s3_prof_bwd_out_kernel python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls gpurun_out
