#!/usr/bin/env python
"""BASELINE config 5: GLA-1.3B (24 layers, hidden 2048, 16 heads of 128) training step
(fwd + bwd + AdamW) on a token shard per GPU, ZeCO sequence parallel across ranks.

    python scripts/model_bench.py [--tokens 131072] [--layers 24] [--steps 5]
    torchrun --nproc-per-node N scripts/model_bench.py ...   (N ranks: one 1M-token sequence at 8 x 128K)

Synthetic tokens, random-init weights; per-block activation recompute.  Prints one JSON line
(rank 0) with tokens/s (whole job), MFU against the measured dense bf16 peak and the share of
the step spent in the ZeCO GLA kernels (timed separately on the same shapes).
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_01004_b200 import distributed as zd  # noqa: E402
from paper_2507_01004_b200.layer import GLAConfig, GLAModel, model_flops_per_token, num_params, zeco_gla  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=131072, help="tokens per GPU")
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-recompute", action="store_true")
    ap.add_argument("--heads", type=int, default=16, help="16 x 128 (default) or 32 x 64 (the paper's GLA-1B heads)")
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = GLAConfig(layers=args.layers, recompute=not args.no_recompute, heads=args.heads)
    comm = zd.AllScanP2P(cfg.heads, cfg.hidden // cfg.heads, cfg.hidden // cfg.heads) if world > 1 else None
    torch.manual_seed(0)
    model = GLAModel(cfg, comm=comm, device=dev)
    model.train()
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, fused=True)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    tok = torch.randint(0, cfg.vocab, (args.tokens,), device=dev, generator=gen)
    lab = torch.randint(0, cfg.vocab, (args.tokens,), device=dev, generator=gen)

    def step():
        opt.zero_grad(set_to_none=True)
        loss = model(tok, lab)
        loss.backward()
        opt.step()
        return loss

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # the GLA core alone on one layer's shapes (fwd + bwd), x layers (+1 fwd for the recompute)
    d = cfg.hidden // cfg.heads
    q, k, v = (torch.randn(cfg.heads, args.tokens, d, device=dev).to(torch.bfloat16).requires_grad_(True)
               for _ in range(3))
    g = (torch.rand(cfg.heads, args.tokens, d, device=dev) * -0.1 - 1e-3).requires_grad_(True)
    for _ in range(3):
        zeco_gla(q, k, v, g, cfg.chunk_len, comm, cfg.num_blocks).sum().backward()
    c0, c1, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    c0.record()
    o = zeco_gla(q, k, v, g, cfg.chunk_len, comm, cfg.num_blocks)
    c1.record()
    o.backward(torch.ones_like(o))
    c2.record()
    torch.cuda.synchronize()
    core_ms = cfg.layers * ((2 if cfg.recompute else 1) * c0.elapsed_time(c1) + c1.elapsed_time(c2))

    peak = 1422.5
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f).get("bf16_tflops_sustained", peak))
    except Exception:
        pass
    fpt = model_flops_per_token(cfg)
    tps = world * args.tokens / (ms / 1e3)
    line = {"metric": "GLA-1.3B training step tokens/s (config 5)", "value": tps, "unit": "tokens/s",
            "n_gpus": world, "ms_per_step": ms, "loss": float(loss.item()),
            "config": {"layers": cfg.layers, "hidden": cfg.hidden, "heads": cfg.heads, "head_dim": d,
                       "tokens_per_gpu": args.tokens, "global_tokens": world * args.tokens,
                       "params": num_params(model), "recompute": cfg.recompute, "optimizer": "AdamW (fused)",
                       "dtype": "bf16", "data": "synthetic tokens, random init"},
            "mfu": fpt * tps / world / 1e12 / peak, "tflops_per_gpu": fpt * tps / world / 1e12,
            "gla_core_ms": core_ms, "gla_core_share": core_ms / ms,
            "peak_mem_gb": torch.cuda.max_memory_allocated() / 2 ** 30}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
