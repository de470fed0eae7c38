"""One-process-per-GPU ZeCO (SPMD form of glasp/engine.py:218-237, 348-364).

``AllScanP2P`` is the product All-Scan: each rank's kernel stores its scanned
state blocks straight into the successor's inbox over NVLink (peer memory
mapped with CUDA IPC, handles exchanged once through torch.distributed) and
raises a per-block flag; no NCCL call on the data path (csrc/allscan.cu).

``AllScanNCCL`` (send/recv chain) and ``lasp2_states`` (all-gather of states +
decay-weighted reduction, glasp/engine.py:165-173) are the baselines the paper
compares against; they are kept only for measurement.

``ZecoRank`` strings the per-rank kernels and the collective together for one
GLA layer forward + backward; ``ledger`` counts elements per primitive like the
reference's VolumeLedger contract.
"""

from __future__ import annotations

import ctypes
import os
from collections import defaultdict

import torch
import torch.distributed as dist

from . import _native, ops
from .errors import ConfigError, DimsError, UnsupportedError


class AllScanP2P:
    """In-kernel NVLink chain All-Scan between the ranks of ``group`` (FWD: 0 -> P-1, BWD: P-1 -> 0)."""

    def __init__(self, heads, key_dim, value_dim, group=None, max_blocks=16, rank=None, world=None):
        self.group = group
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        self.shape = (heads, key_dim, value_dim)
        lib = _native.load()
        h = ctypes.c_void_p()
        _native.check(lib.zgla_allscan_create(self.rank, self.world, heads, key_dim, value_dim, max_blocks,
                                              ctypes.byref(h)), "zgla_allscan_create")
        self._h = h
        if self.world > 1:
            buf = (ctypes.c_char * 64)()
            _native.check(lib.zgla_allscan_export(self._h, buf), "zgla_allscan_export")
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(buf), group=group)
            nxt = handles[self.rank + 1] if self.rank + 1 < self.world else None
            prv = handles[self.rank - 1] if self.rank > 0 else None
            _native.check(lib.zgla_allscan_bind(self._h, nxt, prv), "zgla_allscan_bind")
            dist.barrier(group=group)

    def __call__(self, local: torch.Tensor, log_decay: torch.Tensor, num_blocks: int = 1, direction: int = 0):
        """-> (recv, scanned) for this rank; fp32 [h, dk, dv] / [h, dk] CUDA tensors."""
        h, dk, dv = self.shape
        for t, name, shp in ((local, "local", (h, dk, dv)), (log_decay, "log_decay", (h, dk))):
            if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
                raise UnsupportedError(f"AllScanP2P moves fp32 states: {name} must be a float32 CUDA tensor"
                                       f" (got {getattr(t, 'dtype', type(t))}); fp64 runs use the list form")
            if tuple(t.shape) != shp:
                raise DimsError(f"{name} has shape {tuple(t.shape)}, expected {shp}")
        # keep the dense copies alive until the (stream-ordered) launch has been enqueued
        loc = local.contiguous()
        dec = log_decay.contiguous()
        recv = torch.empty_like(loc)
        scanned = torch.empty_like(loc)
        _native.call("zgla_allscan_run", self._h, num_blocks, direction, ops._p(loc), ops._p(dec), ops._p(recv),
                     ops._p(scanned), ops._stream())
        return recv, scanned

    def split(self, heads):
        """A communicator over the same ranks for ``heads`` heads (one per head group of ZecoRank's
        overlap schedule; each group's chain has its own inboxes and epochs)."""
        return AllScanP2P(heads, self.shape[1], self.shape[2], group=self.group)

    def check(self, sync: bool = True) -> None:
        """DeadlockError if a chain wait of an earlier call timed out (a peer never arrived)."""
        _native.call("zgla_allscan_status", self._h, 1 if sync else 0)

    def bytes_sent(self) -> int:
        return int(_native.load().zgla_allscan_bytes_sent(self._h))

    def close(self):
        """Free the peer-mapped buffers.  Collective when world > 1: every rank drains its device and
        meets the others in a barrier first, so no peer still stores into (or acks to) this region."""
        if getattr(self, "_h", None):
            if self.world > 1 and dist.is_initialized():
                torch.cuda.synchronize()
                dist.barrier(group=self.group)
            _native.load().zgla_allscan_destroy(self._h)
            self._h = None

    def __del__(self):
        # no collective from a finalizer: only a communicator nobody can still be talking to is freed here
        try:
            if getattr(self, "_h", None) and (self.world == 1 or not dist.is_initialized()):
                _native.load().zgla_allscan_destroy(self._h)
                self._h = None
        except Exception:
            pass


def _scan_update(log_decay, recv, local):
    """scanned = e^{G} (.) recv + local; thin torch glue on the (small) state tensors of the baselines."""
    return torch.exp(log_decay)[..., None] * recv + local


class AllScanNCCL:
    """Baseline: All-Scan as a NCCL send/recv chain (whole state per hop, no block pipelining)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def split(self, heads):
        return self

    def __call__(self, local, log_decay, num_blocks=1, direction=0):
        order = list(range(self.world)) if direction == 0 else list(range(self.world - 1, -1, -1))
        pos = order.index(self.rank)
        # gloo moves host tensors only (validation runs with every rank on one device)
        host = local.is_cuda and dist.get_backend(self.group) == "gloo"
        recv = torch.zeros_like(local)
        if pos > 0:
            buf = recv.cpu() if host else recv
            dist.recv(buf, src=order[pos - 1], group=self.group)
            if host:
                recv.copy_(buf)
        scanned = _scan_update(log_decay, recv, local)
        if pos < self.world - 1:
            dist.send(scanned.cpu() if host else scanned, dst=order[pos + 1], group=self.group)
        return recv, scanned


class LatencyChain:
    """Single-GPU probe (diagnostics, not a collective): stands in for a peer chain by holding the stream
    for ``ns`` nanoseconds (one spinning CTA, ``zgla_selftest_spin``) and returning recv = 0.  It lets one
    GPU measure how much of a chain's latency ZecoRank's overlap schedule hides (scripts/overlap_probe.py).
    ``rank``/``world`` say which boundary states the layer applies (rank 1 of 2: prev and no ds_next)."""

    def __init__(self, ns, rank=1, world=2):
        self.ns, self.rank, self.world = int(ns), rank, world

    def split(self, heads):
        return self

    def __call__(self, local, log_decay, num_blocks=1, direction=0):
        _native.call("zgla_selftest_spin", self.ns, ops._stream())
        recv = torch.zeros_like(local)
        return recv, local


def lasp2_states(local, log_decay, direction=0, group=None):
    """Baseline (LASP-2): all-gather every rank's (state, decay), then the decay-weighted reduction."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    states = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    decays = torch.empty((world,) + tuple(log_decay.shape), dtype=log_decay.dtype, device=log_decay.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(states, local.contiguous(), group=group)
        dist.all_gather_into_tensor(decays, log_decay.contiguous(), group=group)
    else:  # gloo: no fused all-gather, host tensors
        st_h, dc_h = states.cpu(), decays.cpu()
        dist.all_gather(list(st_h.unbind(0)), local.contiguous().cpu(), group=group)
        dist.all_gather(list(dc_h.unbind(0)), log_decay.contiguous().cpu(), group=group)
        states.copy_(st_h)
        decays.copy_(dc_h)
    order = list(range(world)) if direction == 0 else list(range(world - 1, -1, -1))
    recv = torch.zeros_like(local)
    for r in order:
        if r == rank:
            break
        recv = _scan_update(decays[r], recv, states[r])
    return recv, _scan_update(log_decay, recv, local)


class ZecoRank:
    """One rank of ZeCO sequence-parallel GLA (one layer, fwd + bwd) over ``comm``."""

    def __init__(self, heads, seq_len, dim, chunk_len=64, dtype=torch.bfloat16, comm=None, num_blocks=4, sms=None,
                 early_inputs=True, overlap_groups=1):
        """``overlap_groups`` G > 1 (with peers): the All-Scan of each direction runs per head group on a
        high-priority communication stream while the compute stream works on the other groups -- the
        paper's "All-Scan || intra-chunk work" (glasp/engine.py:226-228, 356-358), done by pipelining
        independent heads instead of a deferred correction pass."""
        self.shard = ops.ZecoShard(heads, seq_len, dim, dim, chunk_len, dtype, sms=sms)
        # forward()/backward() take every input at once, so the early-input contract holds (ZGLA_EARLY_INPUTS=0
        # in the environment keeps it off, for A/B runs)
        if early_inputs and os.environ.get("ZGLA_EARLY_INPUTS", "1") != "0":
            _native.load().zgla_set_early_inputs(1)
        self.comm = comm
        self.K = num_blocks
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.ledger = defaultdict(int)
        if dim % num_blocks:
            raise ConfigError(f"num_blocks {num_blocks} does not divide key dim {dim}")
        self.G = int(overlap_groups)
        if self.G < 1 or heads % self.G:
            raise ConfigError(f"overlap_groups {overlap_groups} must divide the {heads} heads")
        if self.G > 1 and self.world > 1:
            self.hg = heads // self.G
            self.gshards = [ops.ZecoShard(self.hg, seq_len, dim, dim, chunk_len, dtype, sms=sms) for _ in range(self.G)]
            self.gcomms = [comm.split(self.hg) for _ in range(self.G)]
            self.comm_stream = torch.cuda.Stream(priority=-1)  # the chains jump the queue of compute kernels

    @property
    def grouped(self):
        return self.G > 1 and self.world > 1

    def _pipelined(self, local_fn, chain_fn, out_fn):
        """Compute stream: local(0) local(1) out(0) local(2) out(1) ... out(G-1); the chain of group j runs
        on the comm stream between local(j) and out(j), under local(j+1) / out(j-1)."""
        cs, ms = torch.cuda.current_stream(), self.comm_stream
        done = [None] * self.G
        res = [None] * self.G
        for j in range(self.G + 1):
            if j < self.G:
                x = local_fn(j)
                ev = torch.cuda.Event()
                ev.record(cs)
                ms.wait_event(ev)
                with torch.cuda.stream(ms):
                    res[j] = chain_fn(j, x)
                for t in x:
                    t.record_stream(ms)
                for t in res[j]:
                    t.record_stream(cs)
                done[j] = torch.cuda.Event()
                done[j].record(ms)
            if j >= 1:
                cs.wait_event(done[j - 1])
                out_fn(j - 1, res[j - 1])

    def forward(self, q, k, v, g, out=None, save_states=True):
        """``save_states=False``: forward only (inference / evaluation); skips the chunk-start states the
        backward reads, and a later backward raises StateError."""
        if self.grouped:
            return self._forward_grouped(q, k, v, g, out, save_states)
        self.shard.poll_domain()  # lazy: reports a bad gate seen by an earlier, completed call
        s_loc, g_tot = self.shard.fwd_local(k, v, g)
        prev = None
        if self.world > 1:
            recv, _ = self.comm(s_loc, g_tot, self.K, _native.ZGLA_FWD)
            self.ledger[("all_scan", "sent")] += s_loc.numel() if self.rank < self.world - 1 else 0
            prev = recv if self.rank > 0 else None
        self._prev, self._g_tot = prev, g_tot
        return self.shard.fwd_output(q, k, v, g, prev, out=out, save_states=save_states)

    def forward_backward_host(self, host_in, host_out, head_groups=2, overlap=False):
        """One layer forward + backward with inputs (q, k, v, g, dO) and outputs (o, dq, dk, dv, dg) in
        HOST memory (CPU torch tensors, pinned for full PCIe rate), through the C-ABI call
        ``zgla_zeco_fwd_bwd_host``: heads are pipelined in ``head_groups`` groups so host->device,
        kernels and device->host overlap.  Stream-ordered on the current stream; with ``overlap=True``
        consecutive calls chain (a call's H2D runs under the previous call's D2H) and completion is
        awaited with ``host_wait()``."""
        geo = self.shard.geo
        names = ("q", "k", "v", "g", "d_out", "o", "dq", "dk", "dv", "dg")
        acc = geo.acc
        dts = (geo.dtype, geo.dtype, geo.dtype, acc, geo.dtype, geo.dtype, geo.dtype, geo.dtype, geo.dtype, acc)
        widths = (geo.dk, geo.dk, geo.dv, geo.dk, geo.dv, geo.dv, geo.dk, geo.dk, geo.dv, geo.dk)
        ts = tuple(host_in) + tuple(host_out)
        if len(ts) != 10:
            raise ConfigError("forward_backward_host expects 5 inputs (q, k, v, g, dO) and 5 outputs")
        for t, n, dt, w in zip(ts, names, dts, widths):
            if not isinstance(t, torch.Tensor) or t.is_cuda or not t.is_contiguous():
                raise ConfigError(f"{n} must be a contiguous host (CPU) tensor")
            if t.dtype != dt or tuple(t.shape) != (geo.h, geo.L, w):
                raise ConfigError(f"{n}: expected {dt} {(geo.h, geo.L, w)}, got {t.dtype} {tuple(t.shape)}")
        if not 1 <= head_groups <= geo.h or (self.world > 1 and geo.h % head_groups):
            raise ConfigError(f"head_groups {head_groups} must be in [1, {geo.h}] (and divide the heads with peers)")
        lib = _native.load()
        nbytes = lib.zgla_zeco_fwd_bwd_host_bytes(ctypes.byref(self.shard.shape), self.shard.sms, head_groups)
        if nbytes < 0:
            raise ConfigError("invalid host-call geometry")
        buf = getattr(self, "_host_buf", None)
        if buf is None or buf.numel() < nbytes:
            buf = self._host_buf = torch.empty(nbytes, dtype=torch.uint8, device=self.shard.device)
        comm = None
        if self.world > 1:
            cache = self.__dict__.setdefault("_host_comm", {})
            if head_groups not in cache:
                cache[head_groups] = AllScanP2P(geo.h // head_groups, geo.dk, geo.dv, group=self.comm.group)
            comm = cache[head_groups]._h
        _native.call("zgla_zeco_fwd_bwd_host", ctypes.byref(self.shard.shape), self.shard.sms, head_groups, comm,
                     self.K, *(ctypes.c_void_p(t.data_ptr()) for t in ts), ops._p(buf), buf.numel(),
                     _native.ZGLA_HOST_OVERLAP if overlap else 0, ops._stream())
        if self.world > 1:
            self.ledger[("all_scan", "sent")] += geo.h * geo.dk * geo.dv * (
                (self.rank < self.world - 1) + (self.rank > 0))

    def host_wait(self):
        """Make the current stream wait for the last forward_backward_host(overlap=True) call's D2H."""
        _native.call("zgla_zeco_host_wait", ops._stream())

    def _forward_grouped(self, q, k, v, g, out, save_states=True):
        geo = self.shard.geo
        o = out if out is not None else torch.empty((geo.h, geo.L, geo.dv), dtype=geo.dtype, device=q.device)
        sl = [slice(j * self.hg, (j + 1) * self.hg) for j in range(self.G)]
        self._gprev, self._ggtot = [None] * self.G, [None] * self.G

        def local(j):
            self.gshards[j].poll_domain()
            return self.gshards[j].fwd_local(k[sl[j]], v[sl[j]], g[sl[j]])

        def chain(j, x):
            recv, _ = self.gcomms[j](x[0], x[1], self.K, _native.ZGLA_FWD)
            self._ggtot[j] = x[1]
            return (recv,)

        def output(j, r):
            prev = r[0] if self.rank > 0 else None
            self._gprev[j] = prev
            self.gshards[j].fwd_output(q[sl[j]], k[sl[j]], v[sl[j]], g[sl[j]], prev, out=o[sl[j]],
                                       save_states=save_states)

        self._pipelined(local, chain, output)
        self.ledger[("all_scan", "sent")] += o.shape[0] * geo.dk * geo.dv if self.rank < self.world - 1 else 0
        return o

    def _backward_grouped(self, q, k, v, g, d_out, grads):
        geo = self.shard.geo
        if grads is None:
            grads = tuple(torch.empty((geo.h, geo.L, w), dtype=dt, device=q.device)
                          for w, dt in ((geo.dk, geo.dtype), (geo.dk, geo.dtype), (geo.dv, geo.dtype), (geo.dk, geo.acc)))
        sl = [slice(j * self.hg, (j + 1) * self.hg) for j in range(self.G)]

        def local(j):
            return (self.gshards[j].bwd_local(q[sl[j]], g[sl[j]], d_out[sl[j]]),)

        def chain(j, x):
            recv, _ = self.gcomms[j](x[0], self._ggtot[j], self.K, _native.ZGLA_BWD)
            return (recv,)

        def output(j, r):
            dsn = r[0] if self.rank < self.world - 1 else None
            self.gshards[j].bwd_output(q[sl[j]], k[sl[j]], v[sl[j]], g[sl[j]], d_out[sl[j]], self._gprev[j], dsn,
                                       grads=tuple(x[sl[j]] for x in grads))

        self._pipelined(local, chain, output)
        self.ledger[("all_scan", "sent")] += geo.h * geo.dk * geo.dv if self.rank > 0 else 0
        return grads

    def backward(self, q, k, v, g, d_out, grads=None):
        if self.grouped:
            return self._backward_grouped(q, k, v, g, d_out, grads)
        self.shard.poll_domain()
        ds0 = self.shard.bwd_local(q, g, d_out)
        ds_next = None
        if self.world > 1:
            recv, _ = self.comm(ds0, self._g_tot, self.K, _native.ZGLA_BWD)
            self.ledger[("all_scan", "sent")] += ds0.numel() if self.rank > 0 else 0
            ds_next = recv if self.rank < self.world - 1 else None
        return self.shard.bwd_output(q, k, v, g, d_out, self._prev, ds_next, grads=grads)
