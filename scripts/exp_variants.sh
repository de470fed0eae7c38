#!/bin/bash
# timing-only experiment builds of the fused kernels: pass -D flags (e.g. "-DZGLA_EXP_NOSTORE");
# results of the EXP variants are wrong by construction.  The default build is restored at the end.
BASE="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DZGLA_BUILD"
for v in "" "$@"; do
  make NVFLAGS="$BASE $v" -B -j8 > /dev/null 2>&1
  echo "== variant [$v]"
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.load(sys.stdin); print('phases', d['phase_ms'])"
  python scripts/trace_pipeline.py 5 2>&1 | grep STEADY
done
make -B -j8 > /dev/null 2>&1
