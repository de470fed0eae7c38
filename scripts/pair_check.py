"""d = 64 head-pair path vs the oracle (diagnostics while the PAIR kernels are built): forward (and, with
--bwd, backward) of P ranks through the per-rank entry points + list-form All-Scan."""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import gla_oracle as orc
from paper_2507_01004_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--heads", type=int, default=4)
ap.add_argument("--P", type=int, default=2)
ap.add_argument("--L", type=int, default=512)
ap.add_argument("--bwd", action="store_true")
ap.add_argument("--sms", type=int, default=None)
a = ap.parse_args()
H, P, L, D, C = a.heads, a.P, a.L, 64, 64
q, k, v, g = orc.make_inputs(P, L, H, D, D, 3, orc.LONG_DECAY_LOW, orc.LONG_DECAY_HIGH)
do = orc.make_cotangent(3, H, P * L, D)
bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)  # noqa: E731
Q, K, V, DO = bf(q), bf(k), bf(v), bf(do)
G = torch.from_numpy(g).to("cuda", torch.float32)
q, k, v, do = (x.double().cpu().numpy() for x in (Q, K, V, DO))
g = G.double().cpu().numpy()
part = lambda X, p: X[:, p * L:(p + 1) * L].contiguous()  # noqa: E731
shards = [ops.ZecoShard(H, L, D, D, C, torch.bfloat16, sms=a.sms) for _ in range(P)]
loc = [shards[p].fwd_local(part(K, p), part(V, p), part(G, p)) for p in range(P)]
S = torch.stack([x[0] for x in loc])
gt = torch.stack([x[1] for x in loc])
recv, scanned = ops.allscan_local(S, gt, 4, 0)
o = torch.cat([shards[p].fwd_output(part(Q, p), part(K, p), part(V, p), part(G, p), recv[p] if p else None)
               for p in range(P)], 1)
torch.cuda.synchronize()
want_o, saved, _ = orc.zeco_forward(q, k, v, g, P, C)
print("o", orc.rel_err(o.double().cpu().numpy(), want_o))
print("prev", orc.rel_err(recv.double().cpu().numpy(), np.stack(saved["prev"])))
print("scanned", orc.rel_err(scanned.double().cpu().numpy(), np.stack(saved["scanned"])))
for hh in range(H):
    e = orc.rel_err(o[hh].double().cpu().numpy(), want_o[hh])
    if e > 1e-2:
        print("  head", hh, "o err", e)
if a.bwd:
    d0 = torch.stack([shards[p].bwd_local(part(Q, p), part(G, p), part(DO, p)) for p in range(P)])
    dsn, _ = ops.allscan_local(d0, gt, 4, 1)
    gr = [shards[p].bwd_output(part(Q, p), part(K, p), part(V, p), part(G, p), part(DO, p), recv[p] if p else None,
                               dsn[p] if p < P - 1 else None) for p in range(P)]
    torch.cuda.synchronize()
    want_g, _ = orc.zeco_backward(q, k, v, g, do, P, C, saved)
    for i, n in enumerate(("dq", "dk", "dv", "dg")):
        got = torch.cat([x[i] for x in gr], 1).double().cpu().numpy()
        print(n, orc.rel_err(got, want_g[i]))
        for hh in range(H):
            e = orc.rel_err(got[hh], want_g[i][hh])
            if e > 1e-2:
                print("  head", hh, n, "err", e)
