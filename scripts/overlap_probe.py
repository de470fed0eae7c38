"""How much All-Scan latency does ZecoRank's head-group overlap schedule hide?  (single GPU)

A peer chain is replaced by distributed.LatencyChain: one spinning CTA that holds its stream for d us
(rank 1 of 2: the layer applies a received prev state, as a middle rank does).  For each injected chain
latency d the cfg2 layer step (fwd + bwd, CUDA graph) is timed serially (G = 1: the chain on the compute
stream, fully exposed) and with the overlap schedule (G groups, chains on a high-priority stream).

    python scripts/overlap_probe.py [--lat 0 10 20 40 80] [--groups 1 2 4]
Prints one JSON line per (G, d): ms per step, and exposed = step(G, d) - step(G, 0)."""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_01004_b200 import distributed as zd

ap = argparse.ArgumentParser()
ap.add_argument("--lat", type=float, nargs="+", default=[0, 10, 20, 40, 80])
ap.add_argument("--groups", type=int, nargs="+", default=[1, 2, 4])
ap.add_argument("--heads", type=int, default=16)
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--seq", type=int, default=16384)
ap.add_argument("--iters", type=int, default=30)
a = ap.parse_args()
H, L, D = a.heads, a.seq, a.dim
dev = torch.device("cuda")
gen = torch.Generator(device=dev).manual_seed(0)
u = lambda lo, hi, dt: (torch.rand((H, L, D), device=dev, generator=gen) * (hi - lo) + lo).to(dt)  # noqa: E731
q, k, v, do = (u(-1, 1, torch.bfloat16) for _ in range(4))
g = u(math.log(0.9), math.log(0.999), torch.float32)
o = torch.empty_like(q)
grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty_like(g))


def time_step(G, lat_us):
    layer = zd.ZecoRank(H, L, D, 64, torch.bfloat16, comm=zd.LatencyChain(lat_us * 1000), overlap_groups=G)

    def step():
        layer.forward(q, k, v, g, out=o)
        layer.backward(q, k, v, g, do, grads=grads)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(a.iters):
            gr.replay()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / a.iters
        best = ms if best is None else min(best, ms)
    return best


for G in a.groups:
    base = None
    for d in a.lat:
        ms = time_step(G, d)
        base = ms if base is None else base
        print(json.dumps({"groups": G, "chain_us_per_direction": d, "ms_per_step": round(ms, 5),
                          "exposed_us": round((ms - base) * 1e3, 2), "heads": H, "dim": D, "seq": L}), flush=True)
