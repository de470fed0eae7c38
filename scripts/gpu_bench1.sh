#!/bin/bash
# bench + ncu launch list + full ncu capture of the dominant kernel
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -8
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
tail -45 gpurun_out/launches.csv | cut -c1-220
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_out_kernel -s 3 -c 1 -o gpurun_out/prof_bwd python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_out_kernel -s 3 -c 1 -o gpurun_out/prof_fwd python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls -la gpurun_out
