"""Does bwd_out (K6) reuse L2 lines left by bwd_local (K4)?  And fwd_out (K3) those of fwd_local (K1)?
Times the consumer kernel after its producer, with and without an L2 flush in between."""
import math, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_01004_b200 import ops
H, L, D = 16, 16384, 128
dev = torch.device("cuda")
q, k, v, do = ((torch.rand(H, L, D, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(4))
g = torch.rand(H, L, D, device=dev) * (math.log(0.999) - math.log(0.9)) + math.log(0.9)
sh = ops.ZecoShard(H, L, D, D, 64, torch.bfloat16)
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
def t_consumer(flush_between, which):
    ts = []
    for i in range(13):
        if which == "fwd":
            sh.fwd_local(k, v, g)
        else:
            sh.fwd_local(k, v, g); sh.fwd_output(q, k, v, g); sh.bwd_local(q, g, do)
        if flush_between:
            flush.fill_(i)
        e[0].record()
        if which == "fwd":
            sh.fwd_output(q, k, v, g)
        else:
            sh.bwd_output(q, k, v, g, do)
        e[1].record(); torch.cuda.synchronize()
        if i >= 3:
            ts.append(e[0].elapsed_time(e[1]) * 1e3)
    return round(statistics.median(ts), 1)
for which in ("fwd", "bwd"):
    print(which, "consumer us: after producer", t_consumer(False, which), "| after producer + L2 flush", t_consumer(True, which))
