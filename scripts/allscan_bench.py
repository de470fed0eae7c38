#!/usr/bin/env python
"""All-Scan microbenchmark (BASELINE config 4).

Multi-GPU (real NVLink peer memory, one process per GPU):
    torchrun --nproc-per-node P scripts/allscan_bench.py
  times, per state size (H, d) and block depth K: the in-kernel P2P chain
  (product), the NCCL send/recv chain and the NCCL all-gather-of-states
  (LASP-2) baselines; max over ranks of CUDA-event time.

Single GPU (no peers available):
    python scripts/allscan_bench.py --virtual P
  runs the same per-rank device code (rank_body) for P virtual ranks inside
  one launch of the list-form kernel, so the number is the flag protocol
  latency through device memory / L2, not NVLink; reported as such.
"""

import argparse
import ctypes
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIZES = [(4, 64), (16, 64), (16, 128), (32, 128), (64, 128)]
BLOCKS = [1, 2, 4, 8, 16, 32, 64, 128]


def timeit(fn, iters=50, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.mean(ts), statistics.median(ts)


def graph_time(fn, reps=20, iters=10):
    """per-call device time: `reps` calls captured in one CUDA graph, replayed `iters` times (no host
    launch overhead inside the timed region); returns (mean, best) in us"""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / reps)
    return statistics.mean(ts), min(ts)


def virtual(P, iters):
    """All P ranks in ONE launch of the list-form kernel (same chain_slice device code as the SPMD
    kernel, LL words through device memory + L2): the kernel time is the chain latency."""
    from paper_2507_01004_b200 import _native, ops
    lib = _native.load()
    out = []
    for h, d in SIZES:
        local = torch.rand(P, h, d, d, device="cuda")
        logs = -torch.rand(P, h, d, device="cuda")
        recv, scanned = torch.empty_like(local), torch.empty_like(local)
        for K in [k for k in BLOCKS if k <= d]:
            def fn():
                _native.check(lib.zgla_allscan_local(P, h, d, d, _native.ZGLA_F32, K, 0, ops._p(local), ops._p(logs),
                                                     ops._p(recv), ops._p(scanned), ops._stream()), "allscan")
            mean, best = graph_time(fn, iters=iters)
            out.append({"mode": "virtual-ranks-one-gpu (list-form kernel, graph-timed)", "P": P, "H": h, "d": d,
                        "K": K, "state_bytes": h * d * d * 4, "allscan_us_mean": mean, "allscan_us_best": best,
                        "tau_min_nvlink_us": h * d * d * 4 / 900e3})
    return out


def spmd(iters):
    from paper_2507_01004_b200.distributed import AllScanNCCL, AllScanP2P, lasp2_states
    rank, world = dist.get_rank(), dist.get_world_size()
    out = []
    for h, d in SIZES:
        p2p = AllScanP2P(h, d, d, max_blocks=128)
        nccl = AllScanNCCL()
        local = torch.rand(h, d, d, device="cuda")
        logs = -torch.rand(h, d, device="cuda")
        rows = {}

        def maxr(x):
            t = torch.tensor([x], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        for K in [k for k in BLOCKS if k <= d]:
            dist.barrier()
            m, p = timeit(lambda: p2p(local, logs, K, 0), iters)
            rows[f"p2p_K{K}"] = (maxr(m), maxr(p))
        dist.barrier()
        rows["nccl_sendrecv"] = tuple(maxr(x) for x in timeit(lambda: nccl(local, logs, 1, 0), iters))
        dist.barrier()
        rows["nccl_allgather_lasp2"] = tuple(maxr(x) for x in timeit(lambda: lasp2_states(local, logs, 0), iters))
        if rank == 0:
            for k, (m, p) in rows.items():
                out.append({"mode": "nvlink", "P": world, "H": h, "d": d, "impl": k, "state_bytes": h * d * d * 4,
                            "us_mean": m, "us_p50": p})
        p2p.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--virtual", type=int, default=0, help="P virtual ranks on one GPU")
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    if args.virtual:
        for row in virtual(args.virtual, args.iters):
            print(json.dumps(row))
        return
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    rows = spmd(args.iters)
    if dist.get_rank() == 0:
        for row in rows:
            print(json.dumps(row))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
