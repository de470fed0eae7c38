"""dg / output accuracy against the f64 oracle as the shard grows (one head, d = 128, default gates):
the fused bf16 path and the fp32 SIMT path on the same bf16-rounded inputs (runs the NumPy oracle on the
host: ~1 min per 128K tokens)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import gla_oracle as orc
from paper_2507_01004_b200 import ops


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def step(q, k, v, g, do, dtype, sms=None):
    h, L, D = q.shape
    sh = ops.ZecoShard(h, L, D, D, 64, dtype, sms=sms)
    Q, K_, V, DO = (torch.from_numpy(x).to("cuda", dtype) for x in (q, k, v, do))
    G = torch.from_numpy(g).to("cuda", torch.float32)
    sh.fwd_local(K_, V, G)
    o = sh.fwd_output(Q, K_, V, G, None)
    sh.bwd_local(Q, G, DO)
    gr = sh.bwd_output(Q, K_, V, G, DO, None, None)
    torch.cuda.synchronize()
    return [o.double().cpu().numpy()] + [x.double().cpu().numpy() for x in gr]


sizes = [int(x) for x in sys.argv[1:]] or [16384, 65536, 131072]
for L in sizes:
    for lo, hi, gname in ((orc.DECAY_LOW, orc.DECAY_HIGH, "default"), (orc.LONG_DECAY_LOW, orc.LONG_DECAY_HIGH, "long")):
        q, k, v, g = orc.make_inputs(1, L, 1, 128, 128, 5, lo, hi)
        do = orc.make_cotangent(5, 1, L, 128)
        bf = lambda x: torch.from_numpy(x).to(torch.bfloat16).double().numpy()  # noqa: E731
        q, k, v, do = bf(q), bf(k), bf(v), bf(do)
        g = g.astype(np.float32).astype(np.float64)
        t0 = time.time()
        o, saved, _ = orc.zeco_forward(q, k, v, g, 1, 64)
        (dq, dk, dv, dg), _ = orc.zeco_backward(q, k, v, g, do, 1, 64, saved)
        t_or = time.time() - t0
        want = [o, dq, dk, dv, dg]
        row = {"L": L, "gates": gname, "oracle_s": round(t_or, 1)}
        for name, dt in (("bf16", torch.bfloat16), ("fp32", torch.float32)):
            got = step(q, k, v, g, do, dt)
            row[name] = {n: round(rel(a, b), 6) for n, a, b in zip(("o", "dq", "dk", "dv", "dg"), got, want)}
        print(json.dumps(row), flush=True)
