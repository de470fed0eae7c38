#!/bin/bash
# bench sweep over tokens per GPU and head geometry (one GLA layer fwd+bwd, CUDA graph timing)
for cfg in "--heads 16 --dim 128 --seq 4096" "--heads 16 --dim 128 --seq 16384" "--heads 16 --dim 128 --seq 65536" \
           "--heads 16 --dim 128 --seq 131072" "--heads 8 --dim 128 --seq 16384" "--heads 32 --dim 128 --seq 16384" \
           "--heads 32 --dim 64 --seq 16384" "--heads 32 --dim 64 --seq 131072" "--heads 4 --dim 64 --seq 4096"; do
  python bench.py $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-variants --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; r=d['roofline_step']
print(json.dumps({'heads': c['heads'], 'head_dim': c['head_dim'], 'tokens': c['tokens_per_gpu'], 'ms_per_step': round(d['ms_per_step'],4),
 'Mtok_s': round(d['value']/1e6,2), 'step_hbm_frac': round(r['frac'],3), 'dominant': d['roofline']['kernel'], 'dominant_frac': round(d['roofline']['frac'],3)}))"
done
