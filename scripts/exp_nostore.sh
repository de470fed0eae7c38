#!/bin/bash
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.load(sys.stdin); print('BASE', d['phase_ms'])"
make NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DZGLA_EXP_NOSTORE" -B -j8 > /dev/null 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.load(sys.stdin); print('NOSTORE', d['phase_ms'])"
