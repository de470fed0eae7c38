#!/usr/bin/env python
"""The autograd GLA layer function (layer.zeco_gla, the path GLAModel takes) sequence-parallel over P
processes with the product All-Scan (AllScanP2P, CUDA-IPC peer memory), runnable with every rank on ONE
GPU:  torchrun --nproc-per-node P scripts/spmd_layer_check.py --same-device

Every rank builds the same full sequence, runs its contiguous shard forward + backward through zeco_gla
(head-slice views of token-major buffers, as the model passes them), and rank 0 gathers outputs and
gradients and compares them with the float64 torch GLA on the whole sequence (bf16 rtol 1e-2)."""

import argparse
import math
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    a, b = a.double(), b.double()
    return (a - b).norm().item() / max(b.norm().item(), 1e-300)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--same-device", action="store_true")
    ap.add_argument("--heads", type=int, default=2)
    ap.add_argument("--seq", type=int, default=512, help="tokens per rank")
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--rounds", type=int, default=2)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", 0 if args.same_device else int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo" if args.same_device else "nccl")
    from paper_2507_01004_b200 import distributed as zd
    from paper_2507_01004_b200.layer import gla_reference, zeco_gla

    H, L, D = args.heads, args.seq, args.dim
    T = world * L
    gen = torch.Generator(device=dev).manual_seed(4321)
    u = lambda lo, hi: torch.rand(H, T, D, device=dev, generator=gen) * (hi - lo) + lo  # noqa: E731
    q_f, k_f, v_f = (u(-1, 1).to(torch.bfloat16) for _ in range(3))
    g_f = u(math.log(0.9), math.log(0.999))
    w_f = u(-1, 1).to(torch.bfloat16)  # output cotangent
    comm = zd.AllScanP2P(H, D, D)

    def shard_tm(x):  # this rank's tokens as [H, L, D] head slices of a token-major [L, H*D] buffer
        x = x[:, rank * L:(rank + 1) * L]
        buf = x.permute(1, 0, 2).contiguous().view(L, H * D)
        return buf.view(L, H, D).permute(1, 0, 2)

    for _ in range(args.rounds):  # repeated calls advance the chain's epochs in both directions
        leaves = [shard_tm(x).detach().requires_grad_(True) for x in (q_f, k_f, v_f, g_f)]
        o = zeco_gla(*leaves, 64, comm, 4)
        o.backward(shard_tm(w_f))
    torch.cuda.synchronize()
    mine = [o.detach()] + [x.grad for x in leaves]
    got = []
    for t in mine:  # gather along tokens (gloo: host tensors)
        parts = [torch.empty_like(t.contiguous().cpu()) for _ in range(world)]
        dist.all_gather(parts, t.contiguous().cpu())
        got.append(torch.cat(parts, 1))
    if rank == 0:
        ref = [x.detach().double().requires_grad_(True) for x in (q_f, k_f, v_f, g_f)]
        o_ref = gla_reference(*ref)
        o_ref.backward(w_f.double())
        want = [o_ref.detach().cpu()] + [x.grad.cpu() for x in ref]
        ok = True
        for name, a, b in zip(("o", "dq", "dk", "dv", "dg"), got, want):
            e = rel(a, b)
            print(f"layer {name} rel err {e:.3e}", flush=True)
            ok &= e <= 1e-2
        print("SPMD layer check OK" if ok else "SPMD layer check FAILED", flush=True)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
