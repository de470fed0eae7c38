"""Dense vs token-major (strided zgla_tensor) fused kernels at cfg2: per-phase CUDA-event times."""
import math, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_01004_b200 import ops
H, L, D = 16, 16384, 128
dev = torch.device("cuda")
def mk(dt, tm):
    if tm:
        return torch.empty(L, H, D, dtype=dt, device=dev).transpose(0, 1)
    return torch.empty(H, L, D, dtype=dt, device=dev)
def run(tm_in, tm_out, reps=20, g_tm=None):
    q, k, v, do = (mk(torch.bfloat16, tm_in) for _ in range(4))
    g = mk(torch.float32, tm_in if g_tm is None else g_tm)
    for x in (q, k, v, do):
        x.uniform_(-1, 1)
    g.uniform_(math.log(0.9), math.log(0.999))
    o = mk(torch.bfloat16, tm_out)
    grads = tuple(mk(torch.bfloat16, tm_out) for _ in range(3)) + (mk(torch.float32, tm_out),)
    sh = ops.ZecoShard(H, L, D, D, 64, torch.bfloat16)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ts = []
    for i in range(reps + 3):
        ev[0].record(); sh.fwd_local(k, v, g); ev[1].record(); sh.fwd_output(q, k, v, g, out=o); ev[2].record()
        sh.bwd_local(q, g, do); ev[3].record(); sh.bwd_output(q, k, v, g, do, grads=grads); ev[4].record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append([ev[j].elapsed_time(ev[j + 1]) * 1e3 for j in range(4)])
    return [round(statistics.median(t[j] for t in ts), 1) for j in range(4)]
for tin, tout in ((False, False), (True, False), (False, True), (True, True)):
    print(f"inputs {'token-major' if tin else 'dense'}, outputs {'token-major' if tout else 'dense'}: "
          f"fwd_local/fwd_output/bwd_local/bwd_output us = {run(tin, tout)}")
print(f"q/k/v/dO token-major, g and outputs dense: {run(True, False, g_tm=False)}")
