nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q --timeout 600 -x 2>&1 | tail -3
python bench.py --no-cpu-baseline > gpurun_out/r2_base_bench.json 2> gpurun_out/r2_base_bench.err; head -c 1500 gpurun_out/r2_base_bench.json; echo
python scripts/allscan_bench.py --virtual 8 --iters 20 > gpurun_out/r2_allscan_virtual.jsonl 2>&1; tail -5 gpurun_out/r2_allscan_virtual.jsonl
