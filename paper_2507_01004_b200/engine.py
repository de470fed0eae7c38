"""Sequence-parallel forward/backward runs (drop-in for glasp/engine.py).

``run_forward`` / ``run_backward`` keep the reference signatures and return
``RunArtifacts``.  The P logical ranks of the list form are resident on the
current GPU; each rank's work goes through the per-rank ZeCO entry points of
the C ABI (ops.ZecoShard), and rank boundaries are crossed by the device
All-Scan kernel (ZeCO), a gather + reduction (LASP-2) or a serial chain
(LASP-1).  For bf16 inputs with d in {64, 128} the per-rank work runs on the
fused tcgen05 kernels; float64/float32 inputs run the exact / validation
kernels.  The one-process-per-GPU (SPMD) form lives in distributed.py.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import ops
from ._convert import acc_of, back, compute_dtype, to_dev
from .cluster import NetConfig, Payload, VirtualCluster, VirtualTimeline, VolumeLedger, create_cluster
from .collectives import PipelineConfig, ScanDirection, all_scan_device
from .errors import ConfigError, DimsError, DomainError, LayoutError, StateError
from .gla import CumDecay, GradShard, ModelDims, SeqShard, ShardLayout, State


class StrategyKind(Enum):
    ZECO = "zeco"
    LASP1 = "lasp1"
    LASP2 = "lasp2"
    SINGLE_DEVICE = "single"


@dataclass(frozen=True)
class ComputeCosts:
    """Accepted for signature compatibility (glasp/engine.py:61-72); real kernels are timed instead."""

    per_chunk: float = 1e-5
    per_state: float = 0.0

    def __post_init__(self):
        if self.per_chunk < 0.0 or self.per_state < 0.0:
            raise ConfigError("compute costs must be >= 0")


DEFAULT_COSTS = ComputeCosts()
FORWARD_PHASES = 3
BACKWARD_PHASES = 4


@dataclass
class GlobalSequence:
    """Full-length inputs plus the per-rank layout (glasp/engine.py:81-103)."""

    q: object
    k: object
    v: object
    g: object
    num_ranks: int
    layout: ShardLayout
    dims: ModelDims

    def __post_init__(self):
        if self.num_ranks < 1:
            raise LayoutError(f"num_ranks must be >= 1, got {self.num_ranks}")
        total = self.num_ranks * self.layout.seq_len
        if self.q.shape[1] != total:
            raise LayoutError(f"sequence length {self.q.shape[1]} != num_ranks * per-rank length {total}")

    @property
    def total_len(self) -> int:
        return self.num_ranks * self.layout.seq_len


def split(seq: GlobalSequence) -> list:
    """Contiguous per-rank shards (glasp/engine.py:106-116)."""
    L = seq.layout.seq_len
    return [SeqShard(q=seq.q[:, p * L:(p + 1) * L], k=seq.k[:, p * L:(p + 1) * L], v=seq.v[:, p * L:(p + 1) * L],
                     g=seq.g[:, p * L:(p + 1) * L], layout=seq.layout, dims=seq.dims)
            for p in range(seq.num_ranks)]


def merged_shard(seq: GlobalSequence) -> SeqShard:
    return SeqShard(q=seq.q, k=seq.k, v=seq.v, g=seq.g, layout=ShardLayout(seq.total_len, seq.layout.chunk_len),
                    dims=seq.dims)


@dataclass
class SavedForward:
    """What the backward needs from the forward (glasp/engine.py:119-127)."""

    strategy: StrategyKind
    prev_states: list
    final_states: list
    total_log_decays: list
    local_states: list | None = None


class RunArtifacts:
    """Outputs, ledger, (virtual) timeline, boundary states (lazy), grads (glasp/engine.py:130-137);
    ``measured_timeline`` adds the CUDA-event intervals of the device phases."""

    def __init__(self, outputs, ledger, timeline, boundary_states=None, grads=None, saved=None, _bounds_fn=None,
                 measured_timeline=None):
        self.outputs = outputs
        self.ledger = ledger
        self.timeline = timeline
        self.measured_timeline = measured_timeline
        self._boundary = boundary_states
        self._bounds_fn = _bounds_fn
        self.grads = grads
        self.saved = saved

    @property
    def boundary_states(self):
        if self._boundary is None and self._bounds_fn is not None:
            self._boundary = self._bounds_fn()
        return self._boundary


def _check_cluster(seq, strategy, cluster):
    if strategy is StrategyKind.SINGLE_DEVICE:
        if cluster is None:
            return create_cluster(1, NetConfig())
        if cluster.num_ranks != 1:
            raise ConfigError("single-device runs take a 1-rank cluster")
        return cluster
    if cluster is None:
        raise ConfigError(f"{strategy.value} requires a cluster")
    if cluster.num_ranks != seq.num_ranks:
        raise ConfigError(f"cluster has {cluster.num_ranks} ranks but sequence is split {seq.num_ranks} ways")
    return cluster


def _validate_sequence(seq):
    """What the reference checks when split() builds each rank's SeqShard (glasp/gla.py:95-107): tensor
    shapes, and log-decays finite and strictly negative (on the device, one pass)."""
    h, ek, ev = seq.dims.heads, seq.dims.key_dim, seq.dims.value_dim
    T = seq.total_len
    for name, arr, shape in (("q", seq.q, (h, T, ek)), ("k", seq.k, (h, T, ek)), ("v", seq.v, (h, T, ev)),
                             ("g", seq.g, (h, T, ek))):
        if tuple(arr.shape) != shape:
            raise DimsError(f"{name} has shape {tuple(arr.shape)}, expected {shape}")


def _device_inputs(seq, P):
    """Contiguous per-rank device copies (q, k, v, g) in the compute dtype, read from ``seq`` now."""
    _validate_sequence(seq)
    dt = compute_dtype(seq.q)
    acc = acc_of(dt)
    full = [to_dev(seq.q, dt), to_dev(seq.k, dt), to_dev(seq.v, dt), to_dev(seq.g, acc)]
    ops.check_log_decay(full[3])
    T = full[0].shape[1]
    L = T // P
    if P == 1:
        return [tuple(full)], dt
    return [tuple(x[:, p * L:(p + 1) * L].contiguous() for x in full) for p in range(P)], dt


def _is_numpy(seq):
    return isinstance(seq.q, np.ndarray)


def _np_dtype(seq):
    return seq.q.dtype if isinstance(seq.q, np.ndarray) else None


def _boundary_fn(ranks, C, prevs, npo):
    def build():
        out = []
        for (q, k, v, g), prev in zip(ranks, prevs):
            st, cm = ops.local_state_scan(k, v, g, C)
            lifted = ops.global_correct(st, cm, prev) if prev is not None else st
            out.append([State(back(lifted[n], npo)) for n in range(lifted.shape[0])])
        return out
    return build


def _local_scans(cluster, shards, ranks):
    """Each rank's local scan (K1 + K2), or None when a fused-path shard saw a 64-token tile whose summed
    log-decay leaves its exponent domain."""
    loc = []
    for r, (sh, (q, k, v, g)) in enumerate(zip(shards, ranks)):
        if cluster is not None:
            with cluster.phase(r, "local_scan"):
                loc.append(sh.fwd_local(k, v, g))
        else:
            loc.append(sh.fwd_local(k, v, g))
    for sh in shards:
        if sh.fast:
            try:
                sh.check_domain()
            except DomainError:
                return None
    return loc


def _widened(fn, seq, *args):
    """Run ``fn`` on an fp32 copy of a bf16 sequence (the SIMT kernels use the exact token recurrence and
    accept every gate the reference accepts) and hand back bf16 tensors like the fused path would."""
    wide = GlobalSequence(q=seq.q.float(), k=seq.k.float(), v=seq.v.float(), g=seq.g, num_ranks=seq.num_ranks,
                          layout=seq.layout, dims=seq.dims)
    args = [a.float() if isinstance(a, torch.Tensor) and a.dtype == torch.bfloat16 else a for a in args]
    art = fn(wide, *args)
    cast = (lambda t: t.to(torch.bfloat16) if isinstance(t, torch.Tensor) and t.dtype == torch.float32 else t)
    art.outputs = cast(art.outputs)
    if art.grads is not None:
        art.grads = GradShard(dq=cast(art.grads.dq), dk=cast(art.grads.dk), dv=cast(art.grads.dv), dg=art.grads.dg)
    return art


def run_forward(seq: GlobalSequence, strategy: StrategyKind, cluster: VirtualCluster | None,
                pipe: PipelineConfig = PipelineConfig(), costs: ComputeCosts = DEFAULT_COSTS,
                save_all: bool = False) -> RunArtifacts:
    """Distributed forward pass; outputs cover the full sequence (glasp/engine.py:176-298).

    Device work per rank goes through the ZeCO entry points; the cluster is charged the reference's
    virtual time for every phase (same labels, streams and durations), so ledger and timeline equal the
    reference's, while ``RunArtifacts.measured_timeline`` carries the CUDA-event times of the phases."""
    cluster = _check_cluster(seq, strategy, cluster)
    P = 1 if strategy is StrategyKind.SINGLE_DEVICE else seq.num_ranks
    C = seq.layout.chunk_len
    c = costs.per_chunk
    N = seq.layout.num_chunks * (seq.num_ranks if strategy is StrategyKind.SINGLE_DEVICE else 1)
    npo = _is_numpy(seq)
    ranks, dt = _device_inputs(seq, P)
    acc = acc_of(dt)
    h, dk, dv = seq.dims.heads, seq.dims.key_dim, seq.dims.value_dim
    L = ranks[0][0].shape[1]
    shards = [ops.ZecoShard(h, L, dk, dv, C, dt) for _ in range(P)]
    zero = torch.zeros((h, dk, dv), dtype=acc, device=ranks[0][0].device)
    outs = []
    pre = _local_scans(cluster, shards, ranks)
    if pre is None:  # a gate outside the fused bf16 path's exponent domain: the fp32 kernels take any gate
        return _widened(run_forward, seq, strategy, cluster, pipe, costs, save_all)

    if strategy in (StrategyKind.ZECO, StrategyKind.SINGLE_DEVICE, StrategyKind.LASP2):
        loc = pre
        for r in range(P):
            cluster.compute(r, N * c, "local_scan")
        finals = torch.stack([x[0] for x in loc])
        totals = torch.stack([x[1] for x in loc])
        entry = list(cluster.clocks)
        if strategy is StrategyKind.LASP2 and P > 1:
            from .collectives import all_gather_grouped
            all_gather_grouped(cluster, {"all_gather": list(finals), "all_gather_cumdecay": list(totals)})
            # every rank's decay-weighted reduction of the gathered states (glasp/engine.py:165-173)
            with cluster.phase(0, "state_reduce"):
                prevs_t, scanned_t = ops.allscan_local(finals, totals, 1, 0)
        elif strategy is StrategyKind.ZECO:
            prevs_t, scanned_t = all_scan_device(cluster, finals, totals, pipe, ScanDirection.FWD)
            for r in range(P):  # the intra-chunk precompute overlaps the collective (glasp/engine.py:226-228)
                cluster.join(r, cluster.side_event(r, entry[r], N * c, "intra_precompute", stream="compute2"))
        else:
            prevs_t, scanned_t = torch.zeros_like(finals), finals.clone()
        prevs = [None if (r == 0 and strategy is not StrategyKind.LASP2) else prevs_t[r] for r in range(P)]
        for r in range(P):
            if strategy is not StrategyKind.ZECO:  # per rank: reduction, precompute, outputs (engine.py:275-279)
                if strategy is StrategyKind.LASP2 and P > 1 and costs.per_state > 0.0:
                    cluster.compute(r, math.log2(P) * costs.per_state, "state_reduce")
                cluster.compute(r, N * c, "intra_precompute")
            with cluster.phase(r, "outputs"):
                q, k, v, g = ranks[r]
                outs.append(shards[r].fwd_output(q, k, v, g, prevs[r]))
            cluster.compute(r, N * c, "outputs")
        prev_list = [prevs_t[r] for r in range(P)]
        final_list = [scanned_t[r] for r in range(P)]
        total_list = [totals[r] for r in range(P)]
    elif strategy is StrategyKind.LASP1:
        prev_list, final_list, total_list = [], [], []
        prev = zero
        for r in range(P):
            q, k, v, g = ranks[r]
            if r > 0:
                cluster.p2p_recv(r, r - 1, primitive="p2p", label="recv:state")
            with cluster.phase(r, "rank_work"):
                s_loc, g_tot = shards[r].fwd_local(k, v, g)
                outs.append(shards[r].fwd_output(q, k, v, g, prev if r > 0 else None))
                final = ops.global_correct(s_loc[None], g_tot[None], prev)[0]
            for label in ("local_scan", "intra_precompute", "outputs"):
                cluster.compute(r, N * c, label)
            if r < P - 1:
                cluster.p2p_send(r, r + 1, Payload(h * dk * dv), primitive="p2p", label="send:state")
            prev_list.append(prev)
            final_list.append(final)
            total_list.append(g_tot)
            prev = final
    else:
        raise ConfigError(f"unsupported strategy {strategy}")

    o = outs[0] if P == 1 else torch.cat(outs, dim=1)
    local_states = None
    if save_all:
        local_states = []
        for (q, k, v, g) in ranks:
            st, _ = ops.local_state_scan(k, v, g, C)
            local_states.append([State(back(st[n], npo)) for n in range(st.shape[0])])
    saved = SavedForward(
        strategy=strategy,
        prev_states=[State(back(p, npo)) for p in prev_list],
        final_states=[State(back(f, npo)) for f in final_list],
        total_log_decays=[back(t, npo) for t in total_list],
        local_states=local_states,
    )
    return RunArtifacts(outputs=back(o, npo, _np_dtype(seq)), ledger=cluster.read_ledger(),
                        timeline=cluster.read_timeline(), saved=saved,
                        _bounds_fn=_boundary_fn(ranks, C, prev_list, npo),
                        measured_timeline=cluster.read_measured_timeline())


def run_backward(seq: GlobalSequence, d_out, strategy: StrategyKind, cluster: VirtualCluster | None,
                 pipe: PipelineConfig, saved_artifacts: RunArtifacts, costs: ComputeCosts = DEFAULT_COSTS
                 ) -> RunArtifacts:
    """Distributed backward pass using state saved by run_forward (glasp/engine.py:301-420).

    Like the reference it reads the inputs from ``seq`` and the boundary values from the PUBLIC saved
    fields (``prev_states``, ``total_log_decays``), so artifacts from any run_forward with the same
    sequence work.  The per-rank local forward is re-run on the device first: the backward kernels walk
    the forward's chunk states, which are recomputed from ``seq`` (the reference recomputes them from
    prev too, glasp/gla.py:405-412)."""
    cluster = _check_cluster(seq, strategy, cluster)
    saved = saved_artifacts.saved
    if saved is None:
        raise StateError("backward requires artifacts from a forward run")
    if saved.strategy is not strategy:
        raise StateError(f"saved forward used {saved.strategy.value}, backward asked for {strategy.value}")
    P = 1 if strategy is StrategyKind.SINGLE_DEVICE else seq.num_ranks
    if len(saved.prev_states) != P or len(saved.total_log_decays) != P:
        raise StateError(f"saved forward holds {len(saved.prev_states)} ranks, this run has {P}")
    C = seq.layout.chunk_len
    c = costs.per_chunk
    N = seq.layout.num_chunks * (seq.num_ranks if strategy is StrategyKind.SINGLE_DEVICE else 1)
    npo = _is_numpy(seq)
    h, dk, dv = seq.dims.heads, seq.dims.key_dim, seq.dims.value_dim
    ranks, dt = _device_inputs(seq, P)
    acc = acc_of(dt)
    L = ranks[0][0].shape[1]
    if tuple(d_out.shape) != (h, P * L, dv):
        raise DimsError(f"d_out has shape {tuple(d_out.shape)}, expected {(h, P * L, dv)}")
    dO = to_dev(d_out, dt)
    douts = [dO] if P == 1 else [dO[:, r * L:(r + 1) * L].contiguous() for r in range(P)]
    prevs = [to_dev(st.values, acc) for st in saved.prev_states]
    totals = torch.stack([to_dev(t, acc) for t in saved.total_log_decays])
    shards = [ops.ZecoShard(h, L, dk, dv, C, dt) for _ in range(P)]
    if _local_scans(None, shards, ranks) is None:  # same widening as the forward
        return _widened(run_backward, seq, d_out, strategy, cluster, pipe, saved_artifacts, costs)
    for r in range(P):  # the chunk states the backward kernels read (workspace of each rank's shard)
        q, k, v, g = ranks[r]
        if shards[r].fast:
            shards[r].fwd_output(q, k, v, g, prevs[r] if r > 0 or strategy is StrategyKind.LASP2 else None)
    parts = [None] * P

    if strategy in (StrategyKind.ZECO, StrategyKind.SINGLE_DEVICE, StrategyKind.LASP2):
        loc0 = []
        for r in range(P):
            with cluster.phase(r, "reverse_scan"):
                q, k, v, g = ranks[r]
                loc0.append(shards[r].bwd_local(q, g, douts[r]))
            cluster.compute(r, N * c, "reverse_scan")
        loc0 = torch.stack(loc0)
        entry = list(cluster.clocks)
        if strategy is StrategyKind.LASP2 and P > 1:
            from .collectives import all_gather_grouped
            all_gather_grouped(cluster, {"all_gather": list(loc0)})
            with cluster.phase(0, "state_reduce"):
                ds_nexts, _ = ops.allscan_local(loc0, totals, 1, 1)
        elif strategy is StrategyKind.ZECO:
            ds_nexts, _ = all_scan_device(cluster, loc0, totals, pipe, ScanDirection.BWD)
            for r in range(P):
                cluster.join(r, cluster.side_event(r, entry[r], 2 * N * c, "grad_precompute", stream="compute2"))
        else:
            ds_nexts = torch.zeros_like(loc0)
        for r in range(P):
            if strategy is not StrategyKind.ZECO:
                if strategy is StrategyKind.LASP2 and P > 1 and costs.per_state > 0.0:
                    cluster.compute(r, math.log2(P) * costs.per_state, "state_reduce")
                cluster.compute(r, 2 * N * c, "grad_precompute")
            with cluster.phase(r, "grad_outputs"):
                q, k, v, g = ranks[r]
                first = r == 0 and strategy is not StrategyKind.LASP2
                last = r == P - 1 and strategy is not StrategyKind.LASP2
                parts[r] = shards[r].bwd_output(q, k, v, g, douts[r], None if first else prevs[r],
                                                None if last else ds_nexts[r])
            cluster.compute(r, N * c, "grad_outputs")
    elif strategy is StrategyKind.LASP1:
        ds_next = torch.zeros((h, dk, dv), dtype=acc, device=dO.device)
        for r in range(P - 1, -1, -1):
            q, k, v, g = ranks[r]
            if r < P - 1:
                cluster.p2p_recv(r, r + 1, primitive="p2p", label="recv:dstate")
            cluster.compute(r, BACKWARD_PHASES * N * c, "rank_grad_work")
            with cluster.phase(r, "rank_grad_work"):
                loc = shards[r].bwd_local(q, g, douts[r])
                parts[r] = shards[r].bwd_output(q, k, v, g, douts[r], prevs[r] if r > 0 else None,
                                                ds_next if r < P - 1 else None)
                # ds_boundary = rev[0] + e^{G_tot} ds_next (glasp/gla.py:393-395)
                ds_bound = ops.global_correct(loc[None], totals[r][None], ds_next)[0]
            if r > 0:
                cluster.p2p_send(r, r - 1, Payload(h * dk * dv), primitive="p2p", label="send:dstate")
            ds_next = ds_bound
    else:
        raise ConfigError(f"unsupported strategy {strategy}")

    cat = (lambda i: parts[0][i]) if P == 1 else (lambda i: torch.cat([p[i] for p in parts], dim=1))
    nd = _np_dtype(seq)
    grads = GradShard(dq=back(cat(0), npo, nd), dk=back(cat(1), npo, nd), dv=back(cat(2), npo, nd),
                      dg=back(cat(3), npo, nd))
    return RunArtifacts(outputs=saved_artifacts.outputs, ledger=cluster.read_ledger(),
                        timeline=cluster.read_timeline(), boundary_states=None, grads=grads, saved=saved,
                        _bounds_fn=lambda: saved_artifacts.boundary_states,
                        measured_timeline=cluster.read_measured_timeline())


def ideal_makespan(strategy: StrategyKind, P: int, chunks_per_rank: int, costs: ComputeCosts = DEFAULT_COSTS,
                   backward_pass: bool = False) -> float:
    """Closed-form makespan without communication (glasp/engine.py:423-433)."""
    phases = BACKWARD_PHASES if backward_pass else FORWARD_PHASES
    work = phases * chunks_per_rank * costs.per_chunk
    if strategy in (StrategyKind.LASP1, StrategyKind.SINGLE_DEVICE):
        return P * work
    extra = math.log2(P) * costs.per_state if (strategy is StrategyKind.LASP2 and P > 1) else 0.0
    return work + extra


def overlap_schedule(t_local_scan: float, t_all_scan: float, t_intra_precompute: float, t_outputs: float):
    """Two-stream forward timeline of one rank (glasp/engine.py:436-460); feed it measured phase times."""
    from .cluster import Event

    for name, t in (("t_local_scan", t_local_scan), ("t_all_scan", t_all_scan),
                    ("t_intra_precompute", t_intra_precompute), ("t_outputs", t_outputs)):
        if t < 0.0:
            raise ConfigError(f"{name} must be >= 0, got {t}")
    events = []
    if t_local_scan > 0.0:
        events.append(Event(0, "local_scan", 0.0, t_local_scan, "compute"))
    if t_all_scan > 0.0:
        events.append(Event(0, "all_scan", t_local_scan, t_local_scan + t_all_scan, "net"))
    if t_intra_precompute > 0.0:
        events.append(Event(0, "intra_precompute", t_local_scan, t_local_scan + t_intra_precompute, "compute2"))
    barrier = t_local_scan + max(t_all_scan, t_intra_precompute)
    if t_outputs > 0.0:
        events.append(Event(0, "outputs", barrier, barrier + t_outputs, "compute"))
    return VirtualTimeline(events=tuple(events))
