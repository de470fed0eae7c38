#!/usr/bin/env python
"""Randomised parity sweep of the fused bf16 path (per-rank entry points + the list-form All-Scan) against
the f64 oracle: heads, head dim (64 pairs / zero-filled, 128), tiles per rank, ranks, gate distribution,
segment count (the `sms` plan parameter).  One JSON line per case plus a summary; evidence for the parity
claim beyond the fixed test cases (python scripts/parity_sweep.py [N] [seed])."""
import json
import math
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import gla_oracle as orc  # noqa: E402
from tests.test_gpu_fast import bf16_round, oracle, run_fast  # noqa: E402
from tests.helpers import rel  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
GATES = {"default": (orc.DECAY_LOW, orc.DECAY_HIGH), "long": (orc.LONG_DECAY_LOW, orc.LONG_DECAY_HIGH),
         "strong": (math.log(0.3), math.log(0.9))}
worst = {}
t_start = time.time()
for i in range(N):
    D = rng.choice([64, 128])
    H = rng.choice([1, 2, 3, 4, 5, 8, 12, 16, 24]) if D == 128 else rng.choice([1, 2, 3, 4, 6, 8, 16, 32])
    P = rng.choice([1, 1, 2, 3, 4, 8])
    tiles = rng.choice([1, 2, 3, 5, 8, 13, 21, 32, 48, 64])
    while H * P * tiles * 64 > 16384 and tiles > 1:
        tiles //= 2
    L = tiles * 64
    gname = rng.choice(list(GATES))
    sms = rng.choice([None, None, 1, 2, 7, 37, 148])
    seed = rng.randrange(1 << 30)
    lo, hi = GATES[gname]
    q, k, v, g = orc.make_inputs(P, L, H, D, D, seed, lo, hi)
    do = orc.make_cotangent(seed, H, P * L, D)
    q, k, v, do = (bf16_round(x) for x in (q, k, v, do))
    g = g.astype(np.float32).astype(np.float64)
    got = run_fast(q, k, v, g, do, P, sms=sms)
    want = oracle(q, k, v, g, do, P)
    errs = {kk: rel(got[kk], want[kk]) for kk in ("o", "dq", "dk", "dv", "dg")}
    line = {"case": i, "H": H, "D": D, "P": P, "L_per_rank": L, "gates": gname, "sms": sms,
            "errs": {kk: float(f"{e:.3e}") for kk, e in errs.items()}}
    print(json.dumps(line), flush=True)
    for kk, e in errs.items():
        if e > worst.get(kk, (0, None))[0]:
            worst[kk] = (e, i)
print(json.dumps({"summary": True, "cases": N, "tolerance": 1e-2, "seconds": round(time.time() - t_start, 1),
                  "worst": {kk: {"rel": float(f"{e:.3e}"), "case": c} for kk, (e, c) in worst.items()},
                  "all_within_tolerance": all(e <= 1e-2 for e, _ in worst.values())}), flush=True)
