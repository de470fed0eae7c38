"""Collectives of the list-form API (glasp/collectives.py), on the device.

``all_scan`` runs the paper's pipelined chain scan as ONE CUDA kernel in which
the P logical ranks exchange state blocks through device memory with the same
flag/ack protocol the multi-GPU kernel uses over NVLink peer memory
(csrc/allscan.cu).  ``all_gather``/``all_gather_grouped`` keep the
reference's modelled semantics (values are already resident; the ledger
records (P-1) * size per rank).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import torch

from . import _native, ops
from ._convert import acc_of, any_numpy, back, compute_dtype, to_dev
from .errors import ConfigError, DimsError


class ScanDirection(Enum):
    FWD = "fwd"
    BWD = "bwd"


@dataclass(frozen=True)
class PipelineConfig:
    """Number of d_k blocks the scanned state is split into (glasp/collectives.py:44-56)."""

    num_blocks: int = 1
    block_update_cost: float = 0.0

    def __post_init__(self):
        if self.num_blocks < 1:
            raise ConfigError(f"num_blocks must be >= 1, got {self.num_blocks}")
        if self.block_update_cost < 0.0:
            raise ConfigError("block_update_cost must be >= 0")


def _check_collective_shapes(cluster, values, what):
    if len(values) != cluster.num_ranks:
        raise DimsError(f"{what}: got {len(values)} entries for {cluster.num_ranks} ranks")
    shape = tuple(values[0].shape)
    for i, v in enumerate(values):
        if tuple(v.shape) != shape:
            raise DimsError(f"{what}: rank {i} has shape {tuple(v.shape)}, rank 0 has {shape}")


def charge_all_scan(cluster, P, h, ek, ev, pipe: PipelineConfig, direction: ScanDirection):
    """Virtual time + ledger of one All-Scan, operation for operation as glasp/collectives.py:103-138
    schedules it: the source stages each of the K blocks one tau_b apart, every later rank receives
    block b, (optionally) charges the per-block update, and forwards it.  Size-only payloads: the
    states themselves move on the device."""
    from .cluster import Payload

    if P == 1:
        return
    K = pipe.num_blocks
    block = h * (ek // K) * ev
    tau_b = cluster.net.tau(block)
    order = list(range(P)) if direction is ScanDirection.FWD else list(range(P - 1, -1, -1))
    head = order[0]
    t0 = cluster.clocks[head]
    for b in range(K):
        ready = cluster.side_event(head, t0 + b * tau_b, tau_b, f"all_scan:stage[{b}]", stream="net")
        cluster.p2p_send(head, order[1], Payload(block), primitive="all_scan", not_before=ready)
    for i in range(1, P):
        me, up = order[i], order[i - 1]
        for b in range(K):
            cluster.p2p_recv(me, up, primitive="all_scan", label=f"recv:all_scan[{b}]")
            if pipe.block_update_cost > 0.0:
                cluster.compute(me, pipe.block_update_cost, f"all_scan:update[{b}]")
            if i < P - 1:
                cluster.p2p_send(me, order[i + 1], Payload(block), primitive="all_scan")


def all_scan_device(cluster, local: torch.Tensor, logdecay: torch.Tensor, pipe: PipelineConfig,
                    direction: ScanDirection):
    """Device-tensor form: local [P,h,dk,dv], logdecay [P,h,dk] -> (recv, scanned) [P,h,dk,dv]."""
    P, h, dk, dv = local.shape
    if dk % pipe.num_blocks:
        raise ConfigError(f"num_blocks {pipe.num_blocks} does not divide key dim {dk}")
    if P == 1:
        return torch.zeros_like(local), local.clone()
    with cluster.phase(0, "all_scan", stream="net"):
        recv, scanned = ops.allscan_local(local, logdecay, pipe.num_blocks,
                                          _native.ZGLA_FWD if direction is ScanDirection.FWD else _native.ZGLA_BWD)
    charge_all_scan(cluster, P, h, dk, dv, pipe, direction)
    return recv, scanned


def all_scan(cluster, local_states, cumdecays, pipe: PipelineConfig, direction: ScanDirection):
    """Pipelined exclusive scan of states along the rank chain (glasp/collectives.py:70-140).

    Returns (recv, scanned) lists of State.  Bit-identical for every valid K.
    """
    from .gla import State

    vals = [s.values for s in local_states]
    _check_collective_shapes(cluster, vals, "all_scan states")
    h, ek, ev = vals[0].shape
    for i, cd in enumerate(cumdecays):
        if tuple(cd.log_values.shape) != (h, ek):
            raise DimsError(f"all_scan cumdecay {i} has shape {tuple(cd.log_values.shape)}")
    if ek % pipe.num_blocks != 0:
        raise ConfigError(f"num_blocks {pipe.num_blocks} does not divide key dim {ek}")
    npo = any_numpy(*vals)
    acc = acc_of(compute_dtype(vals[0]))
    local = torch.stack([to_dev(v, acc) for v in vals])
    logs = torch.stack([to_dev(c.log_values, acc) for c in cumdecays])
    recv, scanned = all_scan_device(cluster, local, logs, pipe, direction)
    return ([State(back(recv[p], npo)) for p in range(cluster.num_ranks)],
            [State(back(scanned[p], npo)) for p in range(cluster.num_ranks)])


def all_gather(cluster, values, primitive: str = "all_gather"):
    """Every rank ends up with all P tensors in rank order (glasp/collectives.py:143-146)."""
    return all_gather_grouped(cluster, {primitive: values})[primitive]


def all_gather_grouped(cluster, groups: dict):
    """Several tensor groups gathered in one round; ledger per group (glasp/collectives.py:149-174).

    The values are already resident (one device holds every logical rank); the cluster is charged
    the ring's (P-1) steps of tau(total elements) per rank, as the reference models it."""
    P = cluster.num_ranks
    for name, values in groups.items():
        _check_collective_shapes(cluster, values, name)
    if P == 1:
        return {name: [_copy(values[0])] for name, values in groups.items()}
    sizes = {name: _numel(values[0]) for name, values in groups.items()}
    step = cluster.net.tau(sum(sizes.values()))
    t0 = max(cluster.clocks)
    for r in range(P):
        for s in range(P - 1):
            cluster.side_event(r, t0 + s * step, step, f"all_gather:step[{s}]", stream="net")
        for name, el in sizes.items():
            cluster._count_sent(r, name, (P - 1) * el)
            cluster._count_received(r, name, (P - 1) * el)
        cluster.join(r, t0 + (P - 1) * step)
    return {name: [_copy(v) for v in values] for name, values in groups.items()}


def all_reduce(cluster, values):
    """Elementwise sum across ranks (summed on the device), charged as a ring reduce-scatter + all-gather
    (glasp/collectives.py:177-203)."""
    _check_collective_shapes(cluster, values, "all_reduce")
    npo = any_numpy(*values)
    dt = acc_of(compute_dtype(values[0]))
    stacked = torch.stack([to_dev(v, dt) for v in values])
    total = stacked[0].clone()
    for i in range(1, stacked.shape[0]):  # left fold, the reference's summation order
        total += stacked[i]
    P = cluster.num_ranks
    if P > 1:
        n = _numel(values[0])
        base, rem = divmod(n, P)
        sizes = [base + (1 if i < rem else 0) for i in range(P)]
        step = cluster.net.tau(max(sizes))
        t0 = max(cluster.clocks)
        for r in range(P):
            sent = sum(sizes[(r - s) % P] + sizes[(r - s + 1) % P] for s in range(P - 1))
            recv = sum(sizes[(r - s - 1) % P] + sizes[(r - s) % P] for s in range(P - 1))
            for s in range(2 * (P - 1)):
                cluster.side_event(r, t0 + s * step, step, f"all_reduce:step[{s}]", stream="net")
            cluster._count_sent(r, "all_reduce", sent)
            cluster._count_received(r, "all_reduce", recv)
            cluster.join(r, t0 + 2 * (P - 1) * step)
    return back(total, npo)


def _numel(x):
    return int(x.numel() if isinstance(x, torch.Tensor) else x.size)


def _copy(x):
    return x.clone() if isinstance(x, torch.Tensor) else x.copy()
