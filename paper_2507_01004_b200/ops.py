"""Device-level functional ops over torch CUDA tensors (thin layer over the C ABI).

Every function here launches kernels from libzeco_gla.so on the current torch
CUDA stream; torch only provides device memory and the stream.  Tensor layouts
follow the reference (glasp/gla.py:29-30): q, k, g ``[h, L, dk]``; v, o
``[h, L, dv]``; states ``[h, dk, dv]``; boundary-state lists stacked as
``[N+1, h, dk, dv]`` and cumulative log decays as ``[N+1, h, dk]``.

Precision is chosen by the dtype of q: bfloat16 (tcgen05 fast path for the
ZeCO entry points, fp32 g/states), float32 (fp32 validation mode) or float64
(exact reference semantics).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native
from .errors import ConfigError, DimsError, DomainError, StateError

_CODE = {torch.bfloat16: _native.ZGLA_BF16, torch.float32: _native.ZGLA_F32, torch.float64: _native.ZGLA_F64}


def acc_dtype(t_dtype: torch.dtype) -> torch.dtype:
    """dtype of g, dg and states for a given q/k/v dtype."""
    return torch.float64 if t_dtype == torch.float64 else torch.float32


def dtype_code(t_dtype: torch.dtype) -> int:
    try:
        return _CODE[t_dtype]
    except KeyError:
        raise ConfigError(f"unsupported tensor dtype {t_dtype}; use bfloat16, float32 or float64") from None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _req(t: torch.Tensor, name: str, dtype: torch.dtype, shape: tuple) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        raise DimsError(f"{name} must be a torch tensor")
    if not t.is_cuda:
        raise DimsError(f"{name} must live on a CUDA device")
    if tuple(t.shape) != tuple(shape):
        raise DimsError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != dtype:
        raise DimsError(f"{name} has dtype {t.dtype}, expected {dtype}")
    return t.contiguous()


def num_sms(device=None) -> int:
    return torch.cuda.get_device_properties(device or torch.cuda.current_device()).multi_processor_count


def make_shape(h, L, dk, dv, C, code) -> _native.Shape:
    if min(h, L, dk, dv, C) < 1:
        raise DimsError(f"dims must be positive: h={h} L={L} dk={dk} dv={dv} C={C}")
    if L % C:
        raise DimsError(f"chunk_len {C} does not divide seq_len {L}")
    return _native.Shape(heads=h, key_dim=dk, value_dim=dv, chunk_len=C, seq_len=L, dtype=code)


@dataclass
class Geometry:
    h: int
    L: int
    dk: int
    dv: int
    C: int
    dtype: torch.dtype

    @property
    def acc(self):
        return acc_dtype(self.dtype)

    @property
    def N(self):
        return self.L // self.C

    def shape(self) -> _native.Shape:
        return make_shape(self.h, self.L, self.dk, self.dv, self.C, dtype_code(self.dtype))


def geometry(q, v, C) -> Geometry:
    if q.dim() != 3 or v.dim() != 3:
        raise DimsError("q and v must be rank-3 [heads, tokens, channels]")
    h, L, dk = q.shape
    return Geometry(h, L, dk, v.shape[2], C, q.dtype)


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


# ---------------------------------------------------------------- reference function-level API

def check_log_decay(g: torch.Tensor) -> None:
    """DomainError unless every entry is finite and < 0 (glasp/gla.py:106-107)."""
    if g.numel() == 0:
        return
    bad = torch.zeros(1, dtype=torch.int32, device=g.device)
    code = _native.ZGLA_F64 if g.dtype == torch.float64 else _native.ZGLA_F32
    g = g.contiguous()
    if g.dtype not in (torch.float32, torch.float64):
        raise DimsError(f"g must be float32/float64, got {g.dtype}")
    _native.call("zgla_check_log_decay", g.numel(), code, _p(g), _p(bad), _stream())
    if int(bad.item()):
        raise DomainError("log-decay entries must be strictly negative and finite")


def recurrent_forward(q, k, v, g, C, init=None):
    """glasp/gla.py:210-230: token-by-token recurrence -> (o [h,L,dv], bounds [N+1,h,dk,dv], final [h,dk,dv])."""
    geo = geometry(q, v, C)
    s = geo.shape()
    q = _req(q, "q", geo.dtype, (geo.h, geo.L, geo.dk))
    k = _req(k, "k", geo.dtype, (geo.h, geo.L, geo.dk))
    v = _req(v, "v", geo.dtype, (geo.h, geo.L, geo.dv))
    g = _req(g, "g", geo.acc, (geo.h, geo.L, geo.dk))
    if init is not None:
        init = _req(init, "init", geo.acc, (geo.h, geo.dk, geo.dv))
    o = torch.empty((geo.h, geo.L, geo.dv), dtype=geo.dtype, device=q.device)
    bounds = torch.empty((geo.N + 1, geo.h, geo.dk, geo.dv), dtype=geo.acc, device=q.device)
    final = torch.empty((geo.h, geo.dk, geo.dv), dtype=geo.acc, device=q.device)
    _native.call("zgla_recurrent_forward", ctypes.byref(s), _p(q), _p(k), _p(v), _p(g), _p(init), _p(o),
                 _p(bounds), _p(final), _stream())
    return o, bounds, final


def fd_losses(q, k, v, g, probe, which: int, step: float):
    """glasp/gla.py:463-480: sum(probe * recurrent_forward(x +/- step e_i)) for every element i of tensor
    `which` (0 q, 1 k, 2 v, 3 g), float64 -> [numel, 2] (plus, minus); one kernel launch per tensor."""
    h, L, dk = q.shape
    dv = v.shape[2]
    s = make_shape(h, L, dk, dv, 1, _native.ZGLA_F64)
    ts = [_req(x, n, torch.float64, tuple(x.shape)) for x, n in ((q, "q"), (k, "k"), (v, "v"), (g, "g"))]
    probe = _req(probe, "probe", torch.float64, (h, L, dv))
    n = ts[which].numel()
    losses = torch.empty((n, 2), dtype=torch.float64, device=q.device)
    _native.call("zgla_fd_losses", ctypes.byref(s), *(_p(x) for x in ts), _p(probe), int(which), 0, 2 * n,
                 float(step), _p(losses), _stream())
    return losses


def fd_max_state() -> int:
    return int(_native.load().zgla_fd_max_state())


def local_state_scan(k, v, g, C, init=None):
    """glasp/gla.py:248 (init: optional start state, as in recurrent_forward)."""
    geo = geometry(k, v, C)
    s = geo.shape()
    k = _req(k, "k", geo.dtype, (geo.h, geo.L, geo.dk))
    v = _req(v, "v", geo.dtype, (geo.h, geo.L, geo.dv))
    g = _req(g, "g", geo.acc, (geo.h, geo.L, geo.dk))
    if init is not None:
        init = _req(init, "init", geo.acc, (geo.h, geo.dk, geo.dv))
    states = torch.empty((geo.N + 1, geo.h, geo.dk, geo.dv), dtype=geo.acc, device=k.device)
    cum = torch.empty((geo.N + 1, geo.h, geo.dk), dtype=geo.acc, device=k.device)
    ws = _ws(_native.load().zgla_workspace_bytes(ctypes.byref(s)), k.device)
    _native.call("zgla_local_state_scan", ctypes.byref(s), _p(k), _p(v), _p(g), _p(init), _p(states), _p(cum),
                 _p(ws), _stream())
    return states, cum


def forward_outputs(q, k, v, g, states, cum, prev, C):
    """glasp/gla.py:297 (prev None means the zero state)."""
    geo = geometry(q, v, C)
    s = geo.shape()
    q = _req(q, "q", geo.dtype, (geo.h, geo.L, geo.dk))
    k = _req(k, "k", geo.dtype, (geo.h, geo.L, geo.dk))
    v = _req(v, "v", geo.dtype, (geo.h, geo.L, geo.dv))
    g = _req(g, "g", geo.acc, (geo.h, geo.L, geo.dk))
    states = _req(states, "states", geo.acc, (geo.N + 1, geo.h, geo.dk, geo.dv))
    cum = _req(cum, "cumdecay", geo.acc, (geo.N + 1, geo.h, geo.dk))
    if prev is not None:
        prev = _req(prev, "prev", geo.acc, (geo.h, geo.dk, geo.dv))
    o = torch.empty((geo.h, geo.L, geo.dv), dtype=geo.dtype, device=q.device)
    _native.call("zgla_forward_outputs", ctypes.byref(s), _p(q), _p(k), _p(v), _p(g), _p(states), _p(cum), _p(prev),
                 _p(o), _stream())
    return o


def global_correct(states, cum, prev):
    """glasp/gla.py:272: out[n] = e^{cum[n]} (.) prev + states[n]."""
    n, h, dk, dv = states.shape
    code = _native.ZGLA_F64 if states.dtype == torch.float64 else _native.ZGLA_F32
    s = _native.Shape(heads=h, key_dim=dk, value_dim=dv, chunk_len=1, seq_len=1, dtype=code)
    states = _req(states, "states", states.dtype, (n, h, dk, dv))
    cum = _req(cum, "cumdecay", states.dtype, (n, h, dk))
    prev = _req(prev, "prev", states.dtype, (h, dk, dv))
    out = torch.empty_like(states)
    _native.call("zgla_global_correct", ctypes.byref(s), n, _p(states), _p(cum), _p(prev), _p(out), _stream())
    return out


def reverse_boundary_scan(q, g, d_out, C, seed=None):
    """glasp/gla.py:336 -> [N+1, h, dk, dv]."""
    geo = geometry(q, d_out, C)
    s = geo.shape()
    q = _req(q, "q", geo.dtype, (geo.h, geo.L, geo.dk))
    g = _req(g, "g", geo.acc, (geo.h, geo.L, geo.dk))
    d_out = _req(d_out, "d_out", geo.dtype, (geo.h, geo.L, geo.dv))
    if seed is not None:
        seed = _req(seed, "seed", geo.acc, (geo.h, geo.dk, geo.dv))
    rev = torch.empty((geo.N + 1, geo.h, geo.dk, geo.dv), dtype=geo.acc, device=q.device)
    ws = _ws(_native.load().zgla_workspace_bytes(ctypes.byref(s)), q.device)
    _native.call("zgla_reverse_boundary_scan", ctypes.byref(s), _p(q), _p(g), _p(d_out), _p(seed), _p(rev), _p(ws),
                 _stream())
    return rev


def backward(q, k, v, g, d_out, prev, ds_next, C, saved_states=None):
    """glasp/gla.py:359 -> (dq, dk, dv, dg, ds_boundary)."""
    geo = geometry(q, v, C)
    s = geo.shape()
    q = _req(q, "q", geo.dtype, (geo.h, geo.L, geo.dk))
    k = _req(k, "k", geo.dtype, (geo.h, geo.L, geo.dk))
    v = _req(v, "v", geo.dtype, (geo.h, geo.L, geo.dv))
    g = _req(g, "g", geo.acc, (geo.h, geo.L, geo.dk))
    d_out = _req(d_out, "d_out", geo.dtype, (geo.h, geo.L, geo.dv))
    st = (geo.h, geo.dk, geo.dv)
    prev = None if prev is None else _req(prev, "prev", geo.acc, st)
    ds_next = None if ds_next is None else _req(ds_next, "ds_next", geo.acc, st)
    if saved_states is not None:
        saved_states = _req(saved_states, "saved_states", geo.acc, (geo.N + 1,) + st)
    dq, dk = torch.empty_like(q), torch.empty_like(k)
    dv = torch.empty_like(v)
    dg = torch.empty_like(g)
    dsb = torch.empty(st, dtype=geo.acc, device=q.device)
    ws = _ws(_native.load().zgla_workspace_bytes(ctypes.byref(s)), q.device)
    _native.call("zgla_backward", ctypes.byref(s), _p(q), _p(k), _p(v), _p(g), _p(d_out), _p(prev), _p(ds_next),
                 _p(saved_states), _p(dq), _p(dk), _p(dv), _p(dg), _p(dsb), _p(ws), _stream())
    return dq, dk, dv, dg, dsb


def revcum(x):
    """glasp/gla.py:331: inclusive reverse cumsum along axis 1 of [h, L, d]."""
    if x.dim() != 3:
        raise DimsError("revcum expects [h, L, d]")
    if x.dtype not in (torch.float32, torch.float64):
        raise DimsError("revcum expects float32/float64")
    h, L, d = x.shape
    x = x.contiguous()
    code = _native.ZGLA_F64 if x.dtype == torch.float64 else _native.ZGLA_F32
    s = _native.Shape(heads=h, key_dim=d, value_dim=1, chunk_len=1, seq_len=L, dtype=code)
    out = torch.empty_like(x)
    _native.call("zgla_revcum", ctypes.byref(s), d, _p(x), _p(out), _stream())
    return out


def chunk_scalings(g_chunk):
    """glasp/gla.py:233 -> (chunk_decay [h,dk], decay_from_start [h,C,dk], decay_to_end [h,C,dk])."""
    if g_chunk.dim() != 3:
        raise DimsError(f"expected [h, C, e_k], got shape {tuple(g_chunk.shape)}")
    check_log_decay(g_chunk)
    h, C, dk = g_chunk.shape
    g_chunk = g_chunk.contiguous()
    code = _native.ZGLA_F64 if g_chunk.dtype == torch.float64 else _native.ZGLA_F32
    s = _native.Shape(heads=h, key_dim=dk, value_dim=1, chunk_len=C, seq_len=C, dtype=code)
    decay = torch.empty((h, dk), dtype=g_chunk.dtype, device=g_chunk.device)
    fs, te = torch.empty_like(g_chunk), torch.empty_like(g_chunk)
    _native.call("zgla_chunk_scalings", ctypes.byref(s), _p(g_chunk), _p(decay), _p(fs), _p(te), _stream())
    return decay, fs, te


# ---------------------------------------------------------------- ZeCO per-rank hot path

class ZecoShard:
    """One rank's ZeCO GLA work (glasp/engine.py:218-237 forward, 348-364 backward).

    Owns the device workspace that carries the local scan from the forward to
    the backward (segment states, cumulative decays).  Methods map 1:1 onto the
    four ZeCO entry points of the C ABI.
    """

    def __init__(self, heads, seq_len, key_dim, value_dim, chunk_len, dtype, device=None, sms=None, ws=None,
                 watch_domain=True):
        """``ws``: adopt an existing workspace (e.g. one saved for backward by an autograd Function) instead
        of allocating one; such a shard does not register the lazy domain watch.  ``watch_domain=False``
        skips the watch for shards nobody polls (one per layer call)."""
        self.geo = Geometry(heads, seq_len, key_dim, value_dim, chunk_len, dtype)
        self.shape = self.geo.shape()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.sms = int(sms or num_sms(self.device))
        nbytes = _native.load().zgla_zeco_workspace_bytes(ctypes.byref(self.shape), self.sms)
        if nbytes < 0:
            raise DimsError("invalid ZeCO shard geometry")
        if ws is not None and (ws.dtype != torch.uint8 or ws.numel() < nbytes or not ws.is_cuda):
            raise DimsError(f"adopted workspace must be a CUDA uint8 tensor of >= {nbytes} bytes")
        self.ws = _ws(nbytes, self.device) if ws is None else ws
        self.fast = bool(_native.load().zgla_fast_path(ctypes.byref(self.shape)))
        self._dom = None
        if self.fast and ws is None and watch_domain:  # lazy domain reports of the fused segment pass (host-mapped word)
            dom = ctypes.POINTER(ctypes.c_int)()
            _native.call("zgla_zeco_watch_domain", _p(self.ws), ctypes.byref(dom))
            self._dom = dom

    def __del__(self):
        try:
            if getattr(self, "_dom", None) is not None:
                _native.load().zgla_zeco_unwatch_domain(_p(self.ws))
                self._dom = None
        except Exception:
            pass

    def poll_domain(self):
        """Lazy, non-synchronising domain check of the fused path: DomainError if any fwd_local that has
        COMPLETED since the last poll saw a 64-token tile whose log-decay leaves the bf16 exponent domain
        (a host-mapped word the segment pass writes only in that case).  ZecoRank polls at every call, so
        a bad gate surfaces one call late instead of costing a synchronisation per step."""
        if self._dom is not None and self._dom[0]:
            self._dom[0] = 0
            raise DomainError("a log-decay entry is >= 0 or not finite, or a 64-token tile's summed log-decay "
                              "is below -160 (outside the fused bf16 path's exponent domain: use the fp32 mode)")

    def _state(self):
        return torch.empty((self.geo.h, self.geo.dk, self.geo.dv), dtype=self.geo.acc, device=self.device)

    def _chk(self, t, name, width):
        """Validate one operand.  Per-rank [h, L, width] tensors may be strided views (channels contiguous,
        e.g. head slices of a token-major [L, h * width] buffer) on the fused path; the SIMT path gets
        dense copies."""
        if width == 0:
            return _req(t, name, self.geo.acc, (self.geo.h, self.geo.dk, self.geo.dv))
        dt = self.geo.acc if name in ("g", "dg") else self.geo.dtype
        shape = (self.geo.h, self.geo.L, width)
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise DimsError(f"{name} must be a CUDA torch tensor")
        if tuple(t.shape) != shape or t.dtype != dt:
            raise DimsError(f"{name}: expected {dt} {shape}, got {t.dtype} {tuple(t.shape)}")
        if not self.fast or t.stride(2) != 1:
            t = t.contiguous()
        return t

    @staticmethod
    def _ref(t):
        return _native.Tensor(t.data_ptr(), t.stride(1), t.stride(0))

    def fwd_local(self, k, v, g):
        """local scan -> (S_local_final [h,dk,dv], G_tot [h,dk])."""
        geo = self.geo
        k, v, g = self._chk(k, "k", geo.dk), self._chk(v, "v", geo.dv), self._chk(g, "g", geo.dk)
        s_local = self._state()
        g_tot = torch.empty((geo.h, geo.dk), dtype=geo.acc, device=self.device)
        _native.call("zgla_zeco_fwd_local_v", ctypes.byref(self.shape), self.sms, self._ref(k), self._ref(v),
                     self._ref(g), _p(self.ws), _p(s_local), _p(g_tot), _stream())
        return s_local, g_tot

    def check_domain(self):
        """DomainError if the last fwd_local saw a tile whose log-decay overflows the fused path's exponents
        (synchronises; a validation step, not for the timed path)."""
        _native.call("zgla_zeco_domain_check", ctypes.byref(self.shape), self.sms, _p(self.ws), _stream())

    def fwd_output(self, q, k, v, g, s_prev=None, out=None, save_states=True):
        """outputs [h, L, dv]; ``out`` may be a strided view (e.g. of a token-major [L, h * dv] buffer).
        ``save_states=False``: forward only -- the fused path skips the chunk-start states the backward
        reads (ZGLA_FWD_NO_SAVE), and a later bwd_output raises StateError."""
        geo = self.geo
        q, k, v, g = (self._chk(q, "q", geo.dk), self._chk(k, "k", geo.dk), self._chk(v, "v", geo.dv),
                      self._chk(g, "g", geo.dk))
        if s_prev is not None:
            s_prev = self._chk(s_prev, "s_prev", 0)
        o = out if out is not None else torch.empty((geo.h, geo.L, geo.dv), dtype=geo.dtype, device=self.device)
        o_use = self._chk(o, "o", geo.dv)
        _native.call("zgla_zeco_fwd_output_ex_v", ctypes.byref(self.shape), self.sms, self._ref(q), self._ref(k),
                     self._ref(v), self._ref(g), _p(self.ws), _p(s_prev), self._ref(o_use),
                     0 if save_states else _native.ZGLA_FWD_NO_SAVE, _stream())
        self._states_saved = bool(save_states) or not self.fast
        if o_use.data_ptr() != o.data_ptr():
            o.copy_(o_use)
        return o

    def bwd_local(self, q, g, d_out):
        geo = self.geo
        q, g, d_out = self._chk(q, "q", geo.dk), self._chk(g, "g", geo.dk), self._chk(d_out, "d_out", geo.dv)
        ds0 = self._state()
        _native.call("zgla_zeco_bwd_local_v", ctypes.byref(self.shape), self.sms, self._ref(q), self._ref(g),
                     self._ref(d_out), _p(self.ws), _p(ds0), _stream())
        return ds0

    def bwd_output(self, q, k, v, g, d_out, s_prev=None, ds_next=None, grads=None):
        """(dq, dk, dv, dg) [h, L, .]; ``grads`` may be strided views."""
        if not getattr(self, "_states_saved", True):
            raise StateError("bwd_output after a forward run with save_states=False (no saved chunk states)")
        geo = self.geo
        q, k, v, g = (self._chk(q, "q", geo.dk), self._chk(k, "k", geo.dk), self._chk(v, "v", geo.dv),
                      self._chk(g, "g", geo.dk))
        d_out = self._chk(d_out, "d_out", geo.dv)
        if s_prev is not None:
            s_prev = self._chk(s_prev, "s_prev", 0)
        if ds_next is not None:
            ds_next = self._chk(ds_next, "ds_next", 0)
        if grads is None:
            grads = tuple(torch.empty((geo.h, geo.L, w), dtype=dt, device=self.device)
                          for w, dt in ((geo.dk, geo.dtype), (geo.dk, geo.dtype), (geo.dv, geo.dtype),
                                        (geo.dk, geo.acc)))
        use = [self._chk(x, n, w) for x, n, w in zip(grads, ("dq", "dk", "dv", "dg"), (geo.dk, geo.dk, geo.dv, geo.dk))]
        _native.call("zgla_zeco_bwd_output_v", ctypes.byref(self.shape), self.sms, self._ref(q), self._ref(k),
                     self._ref(v), self._ref(g), self._ref(d_out), _p(self.ws), _p(s_prev), _p(ds_next),
                     *(self._ref(x) for x in use), _stream())
        for x, u in zip(grads, use):
            if u.data_ptr() != x.data_ptr():
                x.copy_(u)
        return tuple(grads)


# ---------------------------------------------------------------- All-Scan, list form

def allscan_local(local: torch.Tensor, logdecay: torch.Tensor, num_blocks: int, direction: int):
    """All P ranks on one device: local [P,h,dk,dv] fp32/fp64, logdecay [P,h,dk] -> (recv, scanned)."""
    if local.dim() != 4 or logdecay.dim() != 3 or logdecay.shape != local.shape[:3]:
        raise DimsError(f"all_scan expects [P,h,dk,dv] / [P,h,dk], got {tuple(local.shape)} / {tuple(logdecay.shape)}")
    P, h, dk, dv = local.shape
    if num_blocks < 1 or dk % num_blocks:
        raise ConfigError(f"num_blocks {num_blocks} does not divide key dim {dk}")
    dt = torch.float64 if local.dtype == torch.float64 else torch.float32
    local = local.contiguous().to(dt)
    logdecay = logdecay.contiguous().to(dt)
    recv = torch.empty_like(local)
    scanned = torch.empty_like(local)
    code = _native.ZGLA_F64 if dt == torch.float64 else _native.ZGLA_F32
    _native.call("zgla_allscan_local", P, h, dk, dv, code, num_blocks, direction, _p(local),
                 _p(logdecay), _p(recv), _p(scanned), _stream())
    return recv, scanned


def selftest_mma(a, b, M, N, K, a_mn, b_mn, lane_off=0):
    d = torch.zeros((M, N), dtype=torch.float32, device=a.device)
    _native.call("zgla_selftest_mma", _p(a.contiguous()), _p(b.contiguous()), _p(d), M, N, K, int(a_mn), int(b_mn),
                 lane_off, _stream())
    return d
