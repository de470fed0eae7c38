#!/bin/bash
# full ncu captures of the fused kernels (one launch each)
for k in bwd_out_kernel fwd_out_kernel seg_state_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep
