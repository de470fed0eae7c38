"""Head-group blocking probe (diagnostics): a cfg2 step run as G groups of H/G heads, each group's
producer -> consumer kernels back to back so the consumer re-reads k/v/g (q/dO/g) from L2.

    python scripts/group_probe.py [G ...]
Prints graph-timed ms/step per G (and per order variant)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_01004_b200 import ops

H, L, D, C = 16, 16384, 128, 64
dev = torch.device("cuda")
gen = torch.Generator(device=dev).manual_seed(0)
u = lambda lo, hi, dt: (torch.rand((H, L, D), device=dev, generator=gen) * (hi - lo) + lo).to(dt)  # noqa: E731
q, k, v, do = (u(-1, 1, torch.bfloat16) for _ in range(4))
g = u(math.log(0.9), math.log(0.999), torch.float32)
o = torch.empty_like(q)
grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty_like(g))


def make(G, sms=None):
    hg = H // G
    shards = [ops.ZecoShard(hg, L, D, D, C, torch.bfloat16, sms=sms) for _ in range(G)]
    sl = [slice(i * hg, (i + 1) * hg) for i in range(G)]

    def step_seq():
        for sh, s in zip(shards, sl):
            sh.fwd_local(k[s], v[s], g[s])
            sh.fwd_output(q[s], k[s], v[s], g[s], None, out=o[s])
        for sh, s in zip(shards, sl):
            sh.bwd_local(q[s], g[s], do[s])
            sh.bwd_output(q[s], k[s], v[s], g[s], do[s], None, None, grads=tuple(x[s] for x in grads))

    def step_interleave():
        # fwd: K1(0) K1(1) K3(0) K1(2) K3(1) ... (comm-overlap order)
        for i in range(G + 1):
            if i < G:
                shards[i].fwd_local(k[sl[i]], v[sl[i]], g[sl[i]])
            if i >= 1:
                j = i - 1
                shards[j].fwd_output(q[sl[j]], k[sl[j]], v[sl[j]], g[sl[j]], None, out=o[sl[j]])
        for i in range(G + 1):
            if i < G:
                shards[i].bwd_local(q[sl[i]], g[sl[i]], do[sl[i]])
            if i >= 1:
                j = i - 1
                shards[j].bwd_output(q[sl[j]], k[sl[j]], v[sl[j]], g[sl[j]], do[sl[j]], None, None,
                                     grads=tuple(x[sl[j]] for x in grads))
    return step_seq, step_interleave


def time_graph(fn, iters=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    res = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            gr.replay()
        b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / iters)
    return min(res)


Gs = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
for G in Gs:
    seq, inter = make(G)
    print(f"G={G} seq {time_graph(seq):.4f} ms  interleave {time_graph(inter):.4f} ms", flush=True)
