#!/usr/bin/env python
"""Benchmark: ZeCO GLA layer forward + backward (BASELINE.json config 2 per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload per rank: one GLA layer, H=16 heads, d_k=d_v=128, 16,384 tokens,
chunk 64, bf16 q/k/v/dO, fp32 log-gates ~ U(log .9, log .999) (synthetic,
seeded per rank).  A step = fwd (local scan, All-Scan FWD, outputs with fused
correction) + bwd (local reverse scan, All-Scan BWD, gradients with fused
correction).  N>1 is weak scaling (16K tokens per GPU), launched by torchrun.

Prints ONE JSON line on rank 0 (see README "bench contract").
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s/GPU, ZeCO GLA layer fwd+bwd, 1/2/4/8 B200 weak scaling; All-Scan µs"
UNIT = "tokens/s"
PEAK_FALLBACK_HBM = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--heads", type=int, default=16)
    p.add_argument("--seq", type=int, default=16384, help="tokens per GPU")
    p.add_argument("--dim", type=int, default=128)
    p.add_argument("--chunk", type=int, default=64)
    p.add_argument("--blocks", type=int, default=4, help="All-Scan pipeline blocks K")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-variants", action="store_true", help="skip the extra H=32 x d=64 line item")
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--e2e-groups", type=int, default=2, help="head groups of the host-buffer pipeline")
    p.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph")
    p.add_argument("--same-device", action="store_true",
                   help="validation only: all ranks on cuda:0 with a gloo bootstrap (timings meaningless)")
    return p.parse_args()


# ------------------------------------------------------------------ helpers

def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    except Exception:
        return PEAK_FALLBACK_HBM, 1400.0, "fallback"


def bytes_per_token_head(dk, dv):
    """Algorithmic (compulsory) HBM bytes: bf16 q,k,v,o,dO,dq,dk,dv; fp32 g, dg."""
    fwd = 8 * dk + 4 * dv
    bwd = 16 * dk + 6 * dv
    return fwd, bwd


def flops_per_token_head(C, dk, dv):
    fwd = 2 * C * (dk + dv) + 4 * dk * dv
    bwd = 2 * C * (3 * dk + 2 * dv) + 12 * dk * dv
    return fwd, bwd


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the timed region runs."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz, self.ok = [], set(), None, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _names(self, mask):
        nv = self.nv
        table = {
            "gpu_idle": getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1),
            "applications_clocks_setting": getattr(nv, "nvmlClocksEventReasonApplicationsClocksSetting", 0x2),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sync_boost": getattr(nv, "nvmlClocksEventReasonSyncBoost", 0x10),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        return {k for k, bit in table.items() if mask & bit}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
                self.reasons |= self._names(fn(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def load_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu summary (profiles/)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("bwd_out_kernel", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------ CPU legs (the reference's own CPU path)

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_kind():
    """'reference' when the unmodified glasp is installed in baseline/_ref (build() does it), else 'port'."""
    return "reference" if os.path.isfile(os.path.join(REF_DIR, "glasp", "engine.py")) else "port"


def _cpu_heads(job):
    """Worker: one fwd+bwd of the reference CPU path on a subset of heads; returns seconds of compute.

    kind 'reference' runs the unmodified glasp (baseline/_ref) through its public API --
    run_forward/run_backward(SINGLE_DEVICE) (glasp/engine.py:176-210, 301-345) on
    generate_sequence inputs (glasp/instances.py:25-51); kind 'port' runs oracle/gla_oracle.py."""
    heads, L, D, C, seed, kind, P, K = job
    rng = np.random.default_rng(seed + 1)
    do = rng.uniform(-1, 1, (heads, P * L, D))
    if kind == "reference":
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from glasp.cluster import NetConfig, create_cluster
        from glasp.collectives import PipelineConfig
        from glasp.engine import StrategyKind, run_backward, run_forward
        from glasp.gla import ModelDims
        from glasp.instances import generate_sequence
        seq = generate_sequence(P, L, C, ModelDims(heads, D, D), seed)
        strat = StrategyKind.ZECO if P > 1 else StrategyKind.SINGLE_DEVICE
        pipe = PipelineConfig(K) if P > 1 else PipelineConfig()
        t0 = time.perf_counter()
        art = run_forward(seq, strat, create_cluster(P, NetConfig()), pipe)
        run_backward(seq, do, strat, create_cluster(P, NetConfig()), pipe, art)
        return time.perf_counter() - t0
    from oracle import gla_oracle as orc
    q, k, v, g = orc.make_inputs(P, L, heads, D, D, seed=seed)
    t0 = time.perf_counter()
    o, saved, _ = orc.zeco_forward(q, k, v, g, P, C)
    orc.zeco_backward(q, k, v, g, do, P, C, saved)
    return time.perf_counter() - t0


class CpuPool:
    """A warm process pool over heads (heads are independent).  Workers are spawned, import the
    reference and run one untimed map BEFORE any timed region, so timings cover compute only."""

    def __init__(self, H, D, C, kind, workers):
        import multiprocessing as mp
        self.H, self.D, self.C, self.kind = H, D, C, kind
        self.workers = max(1, min(workers, H))
        saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in saved:  # one BLAS thread per worker: the pool supplies the parallelism
            os.environ[k] = "1"
        try:
            self.pool = mp.get_context("spawn").Pool(self.workers) if self.workers > 1 else None
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        self.run(64)  # warm: imports + first-touch, untimed

    def jobs(self, L, seed=0):
        per = [self.H // self.workers + (1 if i < self.H % self.workers else 0) for i in range(self.workers)]
        return [(n, L, self.D, self.C, seed + i, self.kind, 1, 1) for i, n in enumerate(per) if n > 0]

    def run(self, L, seed=0):
        """Wall seconds for one fwd+bwd of all H heads over an L-token shard."""
        jobs = self.jobs(L, seed)
        t0 = time.perf_counter()
        if self.pool is None:
            for j in jobs:
                _cpu_heads(j)
        else:
            self.pool.map(_cpu_heads, jobs)
        return time.perf_counter() - t0

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def cpu_legs(H, D, C, L_sample, repeats, steps_note):
    """The CPU baseline: the reference path, pool-parallel over heads (headline) + single-process variants."""
    kind = _reference_kind()
    cores = os.cpu_count() or 1
    pool = CpuPool(H, D, C, kind, cores)
    times = [pool.run(L_sample, seed=s) for s in range(repeats)]
    pool.close()
    t = statistics.mean(times)
    src = ("unmodified glasp 0.1.0 (baseline/_ref) run_forward/run_backward(SINGLE_DEVICE), f64"
           if kind == "reference" else "oracle/gla_oracle.py (NumPy restatement of glasp), f64")
    out = {"value": L_sample / t, "unit": UNIT, "cores": pool.workers, "kind": kind,
           "sample": f"all {H} heads x {L_sample} tokens, d={D}, C={C}, one fwd+bwd per {steps_note}; {src}; "
                     f"heads spread over {pool.workers} warm spawned processes (1 BLAS thread each), "
                     f"pool start-up outside the timed region; {cores} host cores",
           "ms_per_step": t * 1e3}
    return out


def cpu_single_process(H, D, C, L, P, K, seed=0):
    """Variant: the reference path in THIS process (numpy's own threading), as BASELINE.md section 4 times it."""
    kind = _reference_kind()
    dt = _cpu_heads((H, L, D, C, seed, kind, P, K))
    return {"value": P * L / dt, "unit": UNIT, "seconds": dt, "kind": kind, "processes": 1,
            "sample": f"H={H}, d={D}, C={C}, {P} rank(s) x {L} tokens, "
                      f"{'ZECO K=' + str(K) if P > 1 else 'SINGLE_DEVICE'}, f64, one process"}


def cpu_collectives(P=8, H=16, D=128, K=4, reps=3):
    """Variant: the reference's All-Scan (glasp/collectives.py:70-140) and its all-gather-of-states baseline
    (all_gather_grouped, glasp/collectives.py:149-174) at BASELINE config 4's 1 MiB-per-rank state, wall
    clock of the CPU implementation (virtual cluster, one process; best of `reps`)."""
    if _reference_kind() != "reference":
        return {"unavailable": "baseline/_ref (the unmodified glasp) is not installed"}
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from glasp.cluster import NetConfig, create_cluster
    from glasp.collectives import PipelineConfig, ScanDirection, all_gather_grouped, all_scan
    from glasp.gla import CumDecay, State
    rng = np.random.default_rng(0)
    states = [State(rng.uniform(-1, 1, (H, D, D))) for _ in range(P)]
    decays = [CumDecay(rng.uniform(-2, 0, (H, D))) for _ in range(P)]
    best_scan = best_ag = float("inf")
    for _ in range(reps):
        cl = create_cluster(P, NetConfig())
        t0 = time.perf_counter()
        all_scan(cl, states, decays, PipelineConfig(num_blocks=K), ScanDirection.FWD)
        best_scan = min(best_scan, time.perf_counter() - t0)
        cl = create_cluster(P, NetConfig())
        t0 = time.perf_counter()
        all_gather_grouped(cl, {"s": [x.values for x in states], "g": [x.log_values for x in decays]})
        best_ag = min(best_ag, time.perf_counter() - t0)
    return {"all_scan_us": best_scan * 1e6, "all_gather_states_us": best_ag * 1e6, "P": P, "K": K,
            "state_bytes_per_rank_fp32": H * D * D * 4, "kind": "reference", "processes": 1,
            "sample": f"unmodified glasp all_scan(FWD, K={K}) / all_gather_grouped over a virtual cluster of {P} "
                      f"ranks, H={H}, d={D} (f64 arrays), wall clock, best of {reps}"}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path on this box's host cores."""
    if rank != 0:
        return
    H, D, C = args.heads, args.dim, args.chunk
    L_sample = 1024
    kind = _reference_kind()
    cores = os.cpu_count() or 1
    pool = CpuPool(H, D, C, kind, cores)
    for i in range(max(args.warmup, 0)):
        pool.run(L_sample, seed=1000 + i)
    times = [pool.run(L_sample, seed=s) for s in range(args.steps)]
    pool.close()
    t = statistics.mean(times)
    rate = L_sample / t
    src = ("unmodified glasp 0.1.0 (baseline/_ref) run_forward/run_backward(SINGLE_DEVICE), f64"
           if kind == "reference" else "oracle/gla_oracle.py (NumPy restatement of glasp), f64")
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (glasp generate_sequence, seeded)", "impl": "reference",
        "config": {"workload": "cfg2: GLA layer fwd+bwd, H=16, d_k=d_v=128, 16384 tokens/GPU, chunk 64 "
                               f"(CPU: bounded sample of {L_sample} tokens x all heads per step)",
                   "heads": H, "head_dim": D, "chunk": C, "tokens_per_gpu": args.seq},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": pool.workers, "kind": kind,
                         "sample": f"all {H} heads x {L_sample} tokens per step; {src}; heads over "
                                   f"{pool.workers} warm processes (pool start-up untimed); {cores} host cores"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "variants": {
            "single_process_cfg2_sample": cpu_single_process(H, D, C, 256, 1, 1),
            "single_process_cfg1": cpu_single_process(4, 64, 64, 2048, 2, 4),
            "collectives_cfg4": cpu_collectives(),
        },
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ N>1: All-Scan vs the baselines (same run)

def _time_calls(fn, reps, use_graph, barrier, max_over_ranks):
    """Mean device microseconds per fn() call: `reps` back-to-back calls captured in a CUDA graph (else
    eager), after a warm-up; barrier + synchronize on both sides; max over ranks."""
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    graph, timed_as = None, "eager"
    if use_graph:
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                fn()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            barrier()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for _ in range(reps):
                    fn()
            graph.replay()
            timed_as = "cuda_graph"
        except Exception as e:  # a baseline that cannot be captured is timed eagerly
            graph, timed_as = None, f"eager ({type(e).__name__} under capture)"
            torch.cuda.synchronize()
    samples = []
    for _ in range(5):
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if graph is not None:
            graph.replay()
        else:
            for _ in range(reps):
                fn()
        b.record()
        torch.cuda.synchronize()
        samples.append(a.elapsed_time(b) * 1e3 / reps)
    return max_over_ranks(statistics.median(samples)), timed_as


def collective_bench(comm, H, D, K, dev, rank, world, same_device, barrier, max_over_ranks):
    """BASELINE config 3's comparison in the bench run itself: the product All-Scan (in-kernel NVLink chain,
    AllScanP2P) vs the NCCL send/recv chain (AllScanNCCL) vs the LASP-2 all-gather of states + reduction
    (lasp2_states), on the layer's fp32 state [H, D, D]; plus a peer-copy bandwidth probe and tau_min."""
    import torch
    from paper_2507_01004_b200 import distributed as zd
    gen = torch.Generator(device=dev).manual_seed(77 + rank)
    s_loc = torch.rand((H, D, D), device=dev, generator=gen) * 2 - 1
    g_tot = -2 * torch.rand((H, D), device=dev, generator=gen)
    nccl = zd.AllScanNCCL()
    use_graph = not same_device
    res = {"state_bytes": H * D * D * 4, "K": K, "P": world}
    res["p2p_us"], res["p2p_timed_as"] = _time_calls(lambda: comm(s_loc, g_tot, K, 0), 20, use_graph, barrier,
                                                     max_over_ranks)
    res["p2p_bwd_us"], _ = _time_calls(lambda: comm(s_loc, g_tot, K, 1), 20, use_graph, barrier, max_over_ranks)
    res["nccl_chain_us"], res["nccl_chain_timed_as"] = _time_calls(lambda: nccl(s_loc, g_tot), 10, use_graph,
                                                                   barrier, max_over_ranks)
    res["allgather_states_us"], res["allgather_timed_as"] = _time_calls(lambda: zd.lasp2_states(s_loc, g_tot), 10,
                                                                        use_graph, barrier, max_over_ranks)
    res["allgather_over_allscan"] = res["allgather_states_us"] / res["p2p_us"]
    res["tau_min_us"] = res["state_bytes"] / 900e9 * 1e6  # S / B_link, B_link = 900 GB/s per direction (spec)
    res["nvlink_frac"] = res["tau_min_us"] / res["p2p_us"]
    if not same_device and torch.cuda.device_count() > 1:  # measured peer copy rate rank -> rank + 1
        peer = torch.device("cuda", (dev.index + 1) % torch.cuda.device_count())
        src = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        dst = torch.empty(256 << 20, dtype=torch.uint8, device=peer)
        for _ in range(2):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        gbs = 5 * src.numel() / (a.elapsed_time(b) / 1e3) / 1e9
        res["p2p_copy_gbs"] = gbs
        res["tau_measured_copy_us"] = res["state_bytes"] / (gbs * 1e9) * 1e6
        del src, dst
    return res


def allscan_virtual(H, D, K, dev, iters=20):
    import torch
    from paper_2507_01004_b200 import _native, ops
    lib = _native.load()
    out = {"note": "P ranks on one GPU (list-form kernel, LL words through L2), not NVLink; us per call",
           "state_bytes_per_rank": H * D * D * 4, "K": K}
    for P in (2, 4, 8):
        local = torch.rand(P, H, D, D, device=dev)
        logs = -torch.rand(P, H, D, device=dev)
        recv, scanned = torch.empty_like(local), torch.empty_like(local)

        def call():
            _native.check(lib.zgla_allscan_local(P, H, D, D, _native.ZGLA_F32, K, 0, ops._p(local), ops._p(logs),
                                                 ops._p(recv), ops._p(scanned), ops._stream()), "allscan")
        for _ in range(3):
            call()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            call()
        torch.cuda.current_stream().wait_stream(side)
        with torch.cuda.graph(graph):
            for _ in range(iters):
                call()
        graph.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        torch.cuda.synchronize()
        out[f"P{P}_us"] = round(a.elapsed_time(b) * 1e3 / iters, 2)
    return out


def dropin_cfg1(reps=5):
    """BASELINE config 1 through the drop-in's reference API exactly as a glasp user calls it (NumPy f64 in and
    out, run_forward / run_backward(ZECO) with the virtual-cluster bookkeeping): the same call the reference
    arm's single_process_cfg1 times on the CPU, here on the fp64 CUDA kernels (host copies included)."""
    import time
    import torch
    from paper_2507_01004_b200 import (ModelDims, NetConfig, PipelineConfig, StrategyKind, create_cluster,
                                       generate_sequence, run_backward, run_forward)
    P, L, H, D, C, K = 2, 2048, 4, 64, 64, 4
    seq = generate_sequence(P, L, C, ModelDims(H, D, D), 0)
    do = np.random.default_rng(1).uniform(-1, 1, (H, P * L, D))

    def call():
        art = run_forward(seq, StrategyKind.ZECO, create_cluster(P, NetConfig()), PipelineConfig(K))
        run_backward(seq, do, StrategyKind.ZECO, create_cluster(P, NetConfig()), PipelineConfig(K), art)
    call()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        call()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return {"value": P * L / best, "unit": UNIT, "seconds": best, "dtype": "f64",
            "call": "paper_2507_01004_b200.run_forward / run_backward(ZECO), NumPy f64 arrays, P=2 x 2048 tokens, "
                    "H=4, d=64, K=4 (the reference arm's single_process_cfg1 on the drop-in), best of 5"}


def variant_step(H, L, D, C, seed, dev, steps):
    """ms per fwd+bwd step (CUDA graph; inputs larger than L2) of another head geometry."""
    import torch
    from paper_2507_01004_b200 import distributed as zd
    gen = torch.Generator(device=dev).manual_seed(seed * 1000 + 7)

    def uni(lo, hi, dt):
        return (torch.rand((H, L, D), device=dev, generator=gen) * (hi - lo) + lo).to(dt)
    q, k, v, do = (uni(-1, 1, torch.bfloat16) for _ in range(4))
    g = uni(math.log(0.9), math.log(0.999), torch.float32)
    layer = zd.ZecoRank(H, L, D, C, torch.bfloat16)
    o = torch.empty_like(q)
    grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty_like(g))

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
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        graph.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    fwd_b, bwd_b = bytes_per_token_head(D, D)
    hbm, _, _ = peaks()
    return {"heads": H, "head_dim": D, "tokens": L, "ms_per_step": ms, "tokens_per_s": L / (ms / 1e3),
            "fast_path": "head pairs" if D == 64 and H % 2 == 0 else "d=128",
            "hbm_frac_step": (fwd_b + bwd_b) * H * L / (ms / 1e3) / 1e9 / hbm}


# ------------------------------------------------------------------ GPU arm

def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":  # CPU only; under torchrun rank 0 alone runs it, the others exit 0
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    if args.same_device:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if args.same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(x):
        t = torch.tensor([x], device="cpu" if args.same_device else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    from paper_2507_01004_b200 import distributed as zd

    H, L, D, C = args.heads, args.seq, args.dim, args.chunk
    gen = torch.Generator(device=dev).manual_seed(args.seed * 1000 + rank)

    def uni(shape, lo, hi, dt):
        return (torch.rand(shape, device=dev, generator=gen) * (hi - lo) + lo).to(dt)

    q = uni((H, L, D), -1, 1, torch.bfloat16)
    k = uni((H, L, D), -1, 1, torch.bfloat16)
    v = uni((H, L, D), -1, 1, torch.bfloat16)
    g = uni((H, L, D), math.log(0.9), math.log(0.999), torch.float32)
    do = uni((H, L, D), -1, 1, torch.bfloat16)
    comm = zd.AllScanP2P(H, D, D) if world > 1 else None
    layer = zd.ZecoRank(H, L, D, C, torch.bfloat16, comm=comm, num_blocks=args.blocks)
    assert layer.shard.fast, "fused tcgen05 path not selected"
    o = torch.empty_like(q)
    grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty_like(g))
    stream = torch.cuda.current_stream()

    phases = ["fwd_local", "fwd_allscan", "fwd_output", "bwd_local", "bwd_allscan", "bwd_output"]

    def step(evs=None):
        def mark(i):
            if evs is not None:
                evs[i].record()  # current stream: the capture stream while a graph is being captured
        mark(0)
        s_loc, g_tot = layer.shard.fwd_local(k, v, g)
        mark(1)
        prev = None
        if comm is not None:
            recv, _ = comm(s_loc, g_tot, args.blocks, 0)
            prev = recv if rank > 0 else None
        mark(2)
        layer.shard.fwd_output(q, k, v, g, prev, out=o)
        mark(3)
        ds0 = layer.shard.bwd_local(q, g, do)
        mark(4)
        ds_next = None
        if comm is not None:
            recv_b, _ = comm(ds0, g_tot, args.blocks, 1)
            ds_next = recv_b if rank < world - 1 else None
        mark(5)
        layer.shard.bwd_output(q, k, v, g, do, prev, ds_next, grads=grads)
        mark(6)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # per-phase breakdown: eager launches with events between phases (diagnostic only)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(7)] for _ in range(min(args.steps, 20))]
    for e in evs:
        step(e)
    torch.cuda.synchronize()
    per_phase = {p: statistics.mean(e[j].elapsed_time(e[j + 1]) for e in evs) for j, p in enumerate(phases)}
    # the timed region: the step captured once as a CUDA graph and replayed K times (with peers too:
    # the All-Scan chain keeps its epochs in device memory, so replays advance the protocol)
    use_graph = not args.no_graph
    graph = None
    if use_graph:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        # a second capture of the same step with timing-event nodes between the phases: per-kernel times
        # of graph-launched kernels (event nodes cost ~4 us each, so this graph is not the timed one)
        graph_ev = torch.cuda.CUDAGraph()
        graph_evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(7)]
        with torch.cuda.graph(graph_ev):
            step(graph_evs)
        for _ in range(3):
            graph.replay()
    run_step = graph.replay if graph is not None else step
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        start.record()
        for i in range(args.steps):
            run_step()
        end.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(end)
    # per-phase kernel times from replays of the evented graph (mean of 10), else the eager pass
    phase_timed = per_phase
    if graph is not None:
        samples = []
        for _ in range(10):
            graph_ev.replay()
            torch.cuda.synchronize()
            samples.append([graph_evs[j].elapsed_time(graph_evs[j + 1]) for j in range(len(phases))])
        phase_timed = {p: statistics.mean(x[j] for x in samples) for j, p in enumerate(phases)}
    if world > 1:
        ms = max_over_ranks(ms)
    ms_step = ms / args.steps
    value = world * L / (ms_step / 1e3)

    # ---- end to end through the C-ABI with pinned HOST buffers (copies inside the timed region)
    # pinned host tensors carved from one staging arena each way (q k v dO g / o dq dk dv dg back to back,
    # as a loader filling a pinned staging area would lay them out): the host call then moves each head
    # group's equal-sized tensors with one 2-D copy
    def arena(tensors):
        sizes = [x.numel() * x.element_size() for x in tensors]
        offs = [0]
        for b in sizes[:-1]:
            offs.append(offs[-1] + (b + 255) // 256 * 256)
        buf = torch.empty(offs[-1] + sizes[-1], dtype=torch.uint8, pin_memory=True)
        return [buf[o:o + b].view(x.dtype).view(x.shape) for o, b, x in zip(offs, sizes, tensors)]

    hq, hk, hv, hdo, hg = arena([q, k, v, do, g])
    for h_, d_ in ((hq, q), (hk, k), (hv, v), (hdo, do), (hg, g)):
        h_.copy_(d_)
    host_in = [hq, hk, hv, hg, hdo]
    host_out = arena([o, *grads])
    h2d = sum(x.numel() * x.element_size() for x in host_in)
    d2h = sum(x.numel() * x.element_size() for x in host_out)

    def e2e_step():
        # the public host-buffer call: heads pipelined H2D -> kernels -> D2H on three streams; consecutive
        # steps chain (step i+1's H2D runs under step i's D2H); host_wait() closes the timed region
        layer.forward_backward_host(host_in, host_out, head_groups=args.e2e_groups, overlap=True)

    e2e_step()
    layer.host_wait()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    layer.host_wait()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.e2e_steps
    if world > 1:
        e2e_ms = max_over_ranks(e2e_ms)

    # ---- roofline of the dominant kernel (bwd_out_kernel) and of the whole step
    hbm, tc_peak, peak_kind = peaks()
    fwd_b, bwd_b = bytes_per_token_head(D, D)
    fwd_f, bwd_f = flops_per_token_head(C, D, D)
    units = H * L
    dom = max(("fwd_output", "bwd_output", "fwd_local", "bwd_local"), key=lambda p: phase_timed[p])
    dom_bytes = {"fwd_output": fwd_b, "bwd_output": bwd_b, "fwd_local": 2 * D + 2 * D + 4 * D,
                 "bwd_local": 2 * D + 2 * D + 4 * D}[dom] * units
    dom_ms = phase_timed[dom]
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    step_bytes = (fwd_b + bwd_b) * units
    step_flops = (fwd_f + bwd_f) * units

    shown = [p for p in phases if world > 1 or not p.endswith("_allscan")]  # no All-Scan at N=1
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded U(-1,1) q/k/v/dO, g~U(log .9, log .999))",
        "config": {"workload": "cfg2: GLA layer fwd+bwd, H=16, d_k=d_v=128, 16384 tokens/GPU, chunk 64",
                   "heads": H, "head_dim": D, "chunk": C, "tokens_per_gpu": L, "global_tokens": world * L,
                   "allscan_blocks": args.blocks, "parallelism": f"zeco-sp{world}",
                   "l2": "inputs 384 MiB per GPU > 126 MiB L2 (no flush needed)"},
        "per_gpu_tokens_per_s": L / (ms_step / 1e3),
        "phase_ms": {p: round(phase_timed[p], 5) for p in shown},  # graph-launched (event nodes between)
        "phase_ms_eager": {p: round(per_phase[p], 5) for p in shown},
        "timed_as": "cuda_graph" if graph is not None else "eager",
        "roofline": {"kernel": {"fwd_output": "fwd_out_kernel", "bwd_output": "bwd_out_kernel",
                                "fwd_local": "seg_state_kernel<0>+seg_scan_kernel<0>", "bwd_local": "seg_state_kernel<1>+seg_scan_kernel<1>"}[dom],
                     "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": load_traffic(), "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": dom_bytes},
        "roofline_step": {"bound": "hbm", "algorithmic_bytes": step_bytes,
                          "achieved_gbs": step_bytes / (ms_step / 1e3) / 1e9,
                          "frac": step_bytes / (ms_step / 1e3) / 1e9 / hbm,
                          "tflops": step_flops / (ms_step / 1e3) / 1e12,
                          "tensor_frac": step_flops / (ms_step / 1e3) / 1e12 / tc_peak},
        "e2e": {"value": world * L / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "call": f"ZecoRank.forward_backward_host -> zgla_zeco_fwd_bwd_host, pinned host buffers, "
                        f"{args.e2e_groups} head groups pipelined H2D/kernels/D2H, consecutive steps chained"},
        "gpu_launches": args.steps * (6 + (2 if world > 1 else 0)),  # + the two All-Scan chain kernels
        "clocks": clk.summary(),
    }
    if world > 1:
        # in-step chain time (event nodes around the All-Scan inside the captured step; includes the wait
        # for the predecessors), then the isolated collective comparison of BASELINE config 3 / 4
        line["allscan_in_step_us"] = {"fwd": phase_timed["fwd_allscan"] * 1e3, "bwd": phase_timed["bwd_allscan"] * 1e3}
        line["allscan"] = collective_bench(comm, H, D, args.blocks, dev, rank, world, args.same_device,
                                           dist.barrier, max_over_ranks)

    if world == 1:
        # All-Scan microbench in the same run (BASELINE config 4 at this step's state size): P = 2 / 4 / 8 ranks
        # simulated on this GPU by the list-form kernel (the SPMD kernel's chain code, words through L2, one
        # launch), graph-timed; the NVLink numbers come from the N > 1 lines
        line["allscan_virtual"] = allscan_virtual(H, D, args.blocks, dev)
    if world == 1 and not args.no_variants and (H, D) == (16, 128):
        # the same token count as the paper's GLA-1B heads (32 x 64, BASELINE config 1's head size): the
        # d = 64 head-pair kernels, graph-timed the same way (an extra line item, not the headline)
        line["variants"] = {"h32_d64": variant_step(32, L, 64, C, args.seed, dev, args.steps),
                            "dropin_api_cfg1": dropin_cfg1()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_legs(H, D, C, 1024, 3, "repeat (3 repeats)")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
