"""GLA core at the model's per-GPU shape (H heads x 128K tokens): device entry points (dense [h, L, d]) vs the
autograd layer function (token-major strided views, as GLAModel calls it), CUDA-event timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_01004_b200 import distributed as zd
from paper_2507_01004_b200.layer import zeco_gla

H, L, D = int(sys.argv[1]) if len(sys.argv) > 1 else 16, 131072, 128
if len(sys.argv) > 2:
    D = int(sys.argv[2])
dev = torch.device("cuda")


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


q, k, v, do = (torch.rand(H, L, D, device=dev).to(torch.bfloat16) for _ in range(4))
g = torch.rand(H, L, D, device=dev) * -0.1 - 1e-3
rank = zd.ZecoRank(H, L, D, 64, torch.bfloat16)
sh = rank.shard
fwd = lambda: (sh.fwd_local(k, v, g), sh.fwd_output(q, k, v, g, None))  # noqa: E731
bwd = lambda: (sh.bwd_local(q, g, do), sh.bwd_output(q, k, v, g, do, None, None))  # noqa: E731
print(f"device entry points, dense: fwd {timed(fwd):.3f} ms, bwd {timed(bwd):.3f} ms")

# token-major: [L, H*D] buffers viewed as [H, L, D]
tm = lambda x: x.permute(1, 0, 2).contiguous().view(L, H * D).view(L, H, D).permute(1, 0, 2)  # noqa: E731
qt, kt, vt = (tm(x).detach().requires_grad_(True) for x in (q, k, v))
gt = tm(g).detach().requires_grad_(True)
dot = tm(do)
o = None


def lf():
    global o
    o = zeco_gla(qt, kt, vt, gt, 64, None, 4)


def lb():
    o2 = zeco_gla(qt, kt, vt, gt, 64, None, 4)
    o2.backward(dot)


print(f"layer function, token-major: fwd {timed(lf):.3f} ms, fwd+bwd {timed(lb):.3f} ms")

# the same entry points on the token-major views (strided inputs; outputs into token-major buffers)
qd, kd, vd, gd = (x.detach() for x in (qt, kt, vt, gt))
tmo = lambda dt: torch.empty(L, H * D, device=dev, dtype=dt).view(L, H, D).permute(1, 0, 2)  # noqa: E731
o_tm = tmo(torch.bfloat16)
grads_tm = (tmo(torch.bfloat16), tmo(torch.bfloat16), tmo(torch.bfloat16), tmo(torch.float32))
fwd_s = lambda: (sh.fwd_local(kd, vd, gd), sh.fwd_output(qd, kd, vd, gd, None, out=o_tm))  # noqa: E731
bwd_s = lambda: (sh.bwd_local(qd, gd, dot), sh.bwd_output(qd, kd, vd, gd, dot, None, None, grads=grads_tm))  # noqa: E731
print(f"device entry points, token-major views: fwd {timed(fwd_s):.3f} ms, bwd {timed(bwd_s):.3f} ms")
bwd_s2 = lambda: (sh.bwd_local(q, g, do), sh.bwd_output(q, k, v, g, do, None, None, grads=grads_tm))  # noqa: E731
print(f"device entry points, dense inputs, token-major grads: bwd {timed(bwd_s2):.3f} ms")
bwd_s3 = lambda: (sh.bwd_local(qd, gd, dot), sh.bwd_output(qd, kd, vd, gd, dot, None, None))  # noqa: E731
print(f"device entry points, token-major inputs, dense grads: bwd {timed(bwd_s3):.3f} ms")
