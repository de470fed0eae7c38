#!/bin/bash
# compute-sanitizer passes over the GPU paths (run on the GPU box): memcheck (smoke + fast-path parity +
# host pipeline / peer All-Scan / SIMT), synccheck and racecheck on the fused kernels.  Summaries go to
# gpurun_out/sanitize_*.txt; profiles/r01s6_sanitizers.txt is the committed record.
mkdir -p gpurun_out
compute-sanitizer --tool memcheck --leak-check full python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_smoke.txt 2>&1
compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_fast.py -q -x -k "matches_oracle or d64 or strided or long_segments" > gpurun_out/sanitize_fast.txt 2>&1
compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_host.py tests/test_gpu_allscan_spmd.py tests/test_gpu_generic.py -q -x > gpurun_out/sanitize_host.txt 2>&1
compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_fast.py -q -x -k "matches_oracle or long_segments" > gpurun_out/sanitize_sync.txt 2>&1
compute-sanitizer --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_fast.py -q -x -k segmentation > gpurun_out/sanitize_race.txt 2>&1
for f in gpurun_out/sanitize_*.txt; do echo "$f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $f | tail -1)"; done
