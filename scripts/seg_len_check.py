"""dg accuracy of the fused bf16 path against the f64 oracle vs the segment length (one head, 16K tokens,
default gates): the number of segments is set through the `sms` plan parameter."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import gla_oracle as orc
from paper_2507_01004_b200 import ops


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
for lo, hi, gname in ((orc.DECAY_LOW, orc.DECAY_HIGH, "default"), (orc.LONG_DECAY_LOW, orc.LONG_DECAY_HIGH, "long")):
    q, k, v, g = orc.make_inputs(1, L, 1, 128, 128, 5, lo, hi)
    do = orc.make_cotangent(5, 1, L, 128)
    bf = lambda x: torch.from_numpy(x).to(torch.bfloat16).double().numpy()  # noqa: E731
    q, k, v, do = bf(q), bf(k), bf(v), bf(do)
    g = g.astype(np.float32).astype(np.float64)
    o, saved, _ = orc.zeco_forward(q, k, v, g, 1, 64)
    (dq, dk, dv, dg), _ = orc.zeco_backward(q, k, v, g, do, 1, 64, saved)
    for sms in (1, 4, 9, 37, 148):
        sh = ops.ZecoShard(1, L, 128, 128, 64, torch.bfloat16, sms=sms)
        Q, K_, V, DO = (torch.from_numpy(x).to("cuda", torch.bfloat16) for x in (q, k, v, do))
        G = torch.from_numpy(g).to("cuda", torch.float32)
        sh.fwd_local(K_, V, G)
        oo = sh.fwd_output(Q, K_, V, G, None)
        sh.bwd_local(Q, G, DO)
        gr = sh.bwd_output(Q, K_, V, G, DO, None, None)
        torch.cuda.synchronize()
        got = [oo] + list(gr)
        errs = {n: round(rel(x.double().cpu().numpy(), y), 6) for n, x, y in zip(("o", "dq", "dk", "dv", "dg"), got,
                                                                                  (o, dq, dk, dv, dg))}
        # where does the dg error sit: per-token error norm at the segment ends vs elsewhere
        e = np.linalg.norm(gr[3].double().cpu().numpy()[0] - dg[0], axis=1)
        print(json.dumps({"L": L, "gates": gname, "sms": sms, "tiles_per_segment": round(L / 64 / min(sms, L // 64), 1),
                          **errs, "dg_err_first_token": float(e[0]), "dg_err_last_token": float(e[-1]),
                          "dg_norm_per_token": float(np.linalg.norm(dg[0]) / np.sqrt(L))}), flush=True)
