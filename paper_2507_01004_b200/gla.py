"""Drop-in for the reference's GLA function-level API (glasp/gla.py).

Same names, argument meaning, return structure and exceptions as
glasp/gla.py:43-444; the arithmetic runs in libzeco_gla.so on the GPU:

  * float64 inputs -> fp64 kernels (reference semantics, ~1e-15 agreement),
  * float32 inputs -> fp32 validation mode,
  * bfloat16 torch tensors -> bf16 storage, fp32 accumulation.

NumPy inputs give NumPy outputs (copied back); torch CUDA tensors stay on the
device.  There is no CPU arithmetic path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from ._convert import acc_of, any_numpy, back, compute_dtype, to_dev
from .errors import DimsError, DomainError, PrecisionError

__all__ = [
    "ModelDims", "ShardLayout", "SeqShard", "State", "CumDecay", "ChunkScalings", "GradShard",
    "recurrent_forward", "chunk_scalings", "local_state_scan", "global_correct", "forward_outputs",
    "revcum", "reverse_boundary_scan", "backward", "finite_diff_grad",
]


@dataclass(frozen=True)
class ModelDims:
    """Per-head sizes (glasp/gla.py:43-56)."""

    heads: int
    key_dim: int
    value_dim: int

    def __post_init__(self):
        if self.heads < 1 or self.key_dim < 1 or self.value_dim < 1:
            raise DimsError(f"dims must be positive, got {self}")

    @property
    def state_elements(self) -> int:
        return self.heads * self.key_dim * self.value_dim


@dataclass(frozen=True)
class ShardLayout:
    """Tokens per rank and chunk length (glasp/gla.py:60-76)."""

    seq_len: int
    chunk_len: int

    def __post_init__(self):
        if self.seq_len < 1 or self.chunk_len < 1:
            raise DimsError(f"layout must be positive, got {self}")
        if self.seq_len % self.chunk_len != 0:
            raise DimsError(f"chunk_len {self.chunk_len} does not divide seq_len {self.seq_len}")

    @property
    def num_chunks(self) -> int:
        return self.seq_len // self.chunk_len


def _finite(x) -> bool:
    if isinstance(x, np.ndarray):
        return bool(np.all(np.isfinite(x)))
    return bool(torch.isfinite(x).all().item())


@dataclass
class SeqShard:
    """One rank's inputs (glasp/gla.py:80-111); q,k,g [h,L,dk], v [h,L,dv]."""

    q: object
    k: object
    v: object
    g: object
    layout: ShardLayout
    dims: ModelDims

    def __post_init__(self):
        h, ek, ev = self.dims.heads, self.dims.key_dim, self.dims.value_dim
        L = self.layout.seq_len
        for name, arr, shape in (("q", self.q, (h, L, ek)), ("k", self.k, (h, L, ek)), ("v", self.v, (h, L, ev)),
                                 ("g", self.g, (h, L, ek))):
            if tuple(arr.shape) != shape:
                raise DimsError(f"{name} has shape {tuple(arr.shape)}, expected {shape}")
        if isinstance(self.g, np.ndarray):
            if not np.all(np.isfinite(self.g)) or not np.all(self.g < 0.0):
                raise DomainError("log-decay entries must be strictly negative and finite")
        else:
            gd = to_dev(self.g)
            ops.check_log_decay(gd if gd.dtype in (torch.float32, torch.float64) else gd.float())

    @property
    def dtype(self):
        return self.q.dtype

    def device_tensors(self):
        """(q, k, v, g) on the device in the compute dtype.  Read from the arrays at every call (no cache):
        the reference recomputes from the arrays each time, so in-place edits between calls must be seen.
        Torch CUDA tensors of the compute dtype are used as they are (no copy)."""
        dt = compute_dtype(self.q)
        acc = acc_of(dt)
        return to_dev(self.q, dt), to_dev(self.k, dt), to_dev(self.v, dt), to_dev(self.g, acc)

    @property
    def _numpy(self) -> bool:
        return isinstance(self.q, np.ndarray)


@dataclass
class State:
    """Per-head state matrix [h, dk, dv] (glasp/gla.py:115-131)."""

    values: object

    def __post_init__(self):
        if self.values.ndim != 3:
            raise DimsError(f"state must be rank-3, got shape {tuple(self.values.shape)}")
        if not _finite(self.values):
            raise DomainError("state entries must be finite")

    @classmethod
    def zeros(cls, dims: ModelDims, dtype=np.float64) -> "State":
        if isinstance(dtype, torch.dtype):
            return cls(torch.zeros((dims.heads, dims.key_dim, dims.value_dim), dtype=dtype, device="cuda"))
        return cls(np.zeros((dims.heads, dims.key_dim, dims.value_dim), dtype=dtype))

    def copy(self) -> "State":
        return State(self.values.copy() if isinstance(self.values, np.ndarray) else self.values.clone())


@dataclass
class CumDecay:
    """Cumulative log decay [h, dk], entries <= 0 (glasp/gla.py:135-149)."""

    log_values: object

    def __post_init__(self):
        if self.log_values.ndim != 2:
            raise DimsError(f"cumdecay must be rank-2, got {tuple(self.log_values.shape)}")
        lv = self.log_values
        ok = (bool(np.all(np.isfinite(lv)) and np.all(lv <= 0.0)) if isinstance(lv, np.ndarray)
              else bool((torch.isfinite(lv) & (lv <= 0)).all().item()))
        if not ok:
            raise DomainError("cumulative log-decay entries must be finite and <= 0")

    @classmethod
    def ones(cls, dims: ModelDims, dtype=np.float64) -> "CumDecay":
        return cls(np.zeros((dims.heads, dims.key_dim), dtype=dtype))


@dataclass
class ChunkScalings:
    """glasp/gla.py:153-167."""

    chunk_decay: object
    decay_from_start: object
    decay_to_end: object


@dataclass
class GradShard:
    """Gradients mirroring SeqShard; dg is w.r.t. the log decay (glasp/gla.py:171-182)."""

    dq: object
    dk: object
    dv: object
    dg: object

    def __post_init__(self):
        for name, arr in (("dq", self.dq), ("dk", self.dk), ("dv", self.dv), ("dg", self.dg)):
            if not _finite(arr):
                raise DomainError(f"{name} contains non-finite entries")


# ---------------------------------------------------------------- helpers

def _states_to_dev(states, acc):
    return torch.stack([to_dev(s.values, acc) for s in states])


def _cum_to_dev(cum, acc):
    return torch.stack([to_dev(c.log_values, acc) for c in cum])


def _state_list(t, as_numpy):
    return [State(back(t[i], as_numpy)) for i in range(t.shape[0])]


def _np_dtype(shard):
    return shard.q.dtype if isinstance(shard.q, np.ndarray) else None


# ---------------------------------------------------------------- API

def recurrent_forward(shard: SeqShard, init: State | None = None):
    """Token-by-token recurrence -> (outputs, N+1 boundary states, final) (glasp/gla.py:210-230).

    Runs ``zgla_recurrent_forward`` (csrc/recurrence.cu): one state update per token, independent of
    every chunkwise kernel, so it can arbitrate them as the reference's does."""
    q, k, v, g = shard.device_tensors()
    acc = acc_of(q.dtype)
    if init is not None:
        expected = (shard.dims.heads, shard.dims.key_dim, shard.dims.value_dim)
        if tuple(init.values.shape) != expected:
            raise DimsError(f"initial state has shape {tuple(init.values.shape)}, expected {expected}")
    init_d = None if init is None else to_dev(init.values, acc)
    o, bounds, final = ops.recurrent_forward(q, k, v, g, shard.layout.chunk_len, init=init_d)
    npo = shard._numpy
    return back(o, npo, _np_dtype(shard)), _state_list(bounds, npo), State(back(final, npo))


def chunk_scalings(g_chunk) -> ChunkScalings:
    """glasp/gla.py:233-245."""
    if g_chunk.ndim != 3:
        raise DimsError(f"expected [h, C, e_k], got shape {tuple(g_chunk.shape)}")
    npo = isinstance(g_chunk, np.ndarray)
    gd = to_dev(g_chunk, acc_of(compute_dtype(g_chunk)))
    d, fs, te = ops.chunk_scalings(gd)
    return ChunkScalings(back(d, npo), back(fs, npo), back(te, npo))


def local_state_scan(shard: SeqShard):
    """N+1 states from zero and N+1 cumulative decays (glasp/gla.py:248-269)."""
    q, k, v, g = shard.device_tensors()
    states, cum = ops.local_state_scan(k, v, g, shard.layout.chunk_len)
    npo = shard._numpy
    return _state_list(states, npo), [CumDecay(back(cum[i], npo)) for i in range(cum.shape[0])]


def global_correct(states, cumdecay, prev: State):
    """out[n] = exp(cumdecay[n]) (.) prev + states[n] (glasp/gla.py:272-287)."""
    if len(states) != len(cumdecay):
        raise DimsError(f"got {len(states)} states but {len(cumdecay)} cumulative decays")
    for st in states:
        if tuple(st.values.shape) != tuple(prev.values.shape):
            raise DimsError(f"state shape {tuple(st.values.shape)} != prev shape {tuple(prev.values.shape)}")
    npo = any_numpy(prev.values)
    acc = acc_of(compute_dtype(prev.values))
    out = ops.global_correct(_states_to_dev(states, acc), _cum_to_dev(cumdecay, acc), to_dev(prev.values, acc))
    return _state_list(out, npo)


def forward_outputs(shard: SeqShard, states, cumdecay, prev: State):
    """Chunkwise outputs with the lazy global correction (glasp/gla.py:297-328)."""
    N = shard.layout.num_chunks
    if len(states) != N + 1 or len(cumdecay) != N + 1:
        raise DimsError(f"expected {N + 1} scan entries, got {len(states)}/{len(cumdecay)}")
    q, k, v, g = shard.device_tensors()
    acc = acc_of(q.dtype)
    o = ops.forward_outputs(q, k, v, g, _states_to_dev(states, acc), _cum_to_dev(cumdecay, acc),
                            to_dev(prev.values, acc), shard.layout.chunk_len)
    return back(o, shard._numpy, _np_dtype(shard))


def revcum(values):
    """Inclusive reverse cumulative sum along axis 1 (glasp/gla.py:331-333)."""
    npo = isinstance(values, np.ndarray)
    x = to_dev(values, acc_of(compute_dtype(values)))
    return back(ops.revcum(x), npo)


def reverse_boundary_scan(shard: SeqShard, d_out):
    """Zero-seeded suffix scan of state cotangents (glasp/gla.py:336-356)."""
    q, k, v, g = shard.device_tensors()
    rev = ops.reverse_boundary_scan(q, g, to_dev(d_out, q.dtype), shard.layout.chunk_len)
    return _state_list(rev, shard._numpy)


def backward(shard: SeqShard, d_out, prev: State, ds_next: State, saved_states=None):
    """Chunkwise backward of one shard -> (GradShard, ds_boundary) (glasp/gla.py:359-444)."""
    C = shard.layout.chunk_len
    N = shard.layout.num_chunks
    h, ek, ev = shard.dims.heads, shard.dims.key_dim, shard.dims.value_dim
    if tuple(d_out.shape) != (h, shard.layout.seq_len, ev):
        raise DimsError(f"d_out has shape {tuple(d_out.shape)}")
    if saved_states is not None and len(saved_states) != N + 1:
        raise DimsError(f"expected {N + 1} saved states, got {len(saved_states)}")
    q, k, v, g = shard.device_tensors()
    acc = acc_of(q.dtype)
    saved = None if saved_states is None else _states_to_dev(saved_states, acc)
    dq, dk, dv, dg, dsb = ops.backward(q, k, v, g, to_dev(d_out, q.dtype), to_dev(prev.values, acc),
                                       to_dev(ds_next.values, acc), C, saved_states=saved)
    npo, ndt = shard._numpy, _np_dtype(shard)
    grads = GradShard(dq=back(dq, npo, ndt), dk=back(dk, npo, ndt), dv=back(dv, npo, ndt), dg=back(dg, npo, ndt))
    return grads, State(back(dsb, npo))


def finite_diff_grad(shard: SeqShard, probe, step: float) -> GradShard:
    """Central differences of <probe, recurrent_forward(shard)> (glasp/gla.py:447-480), float64 only.

    Every perturbed loss is a token recurrence (csrc/recurrence.cu ``fd_loss_kernel``, one CTA per
    perturbation, one launch per tensor); grad[i] = (plus_i - minus_i) / (2 step) as in the reference.
    States larger than the kernel's shared-memory budget take one ``recurrent_forward`` per perturbation."""
    if step <= 0.0:
        raise DomainError(f"step must be positive, got {step}")
    for name, arr in (("q", shard.q), ("k", shard.k), ("v", shard.v), ("g", shard.g), ("probe", probe)):
        dt = arr.dtype
        if not (dt == np.float64 or dt == torch.float64):
            raise PrecisionError(f"{name} must be float64 for finite differences, got {dt}")
    npo = shard._numpy
    base = [to_dev(getattr(shard, n), torch.float64) for n in ("q", "k", "v", "g")]
    pr = to_dev(probe, torch.float64)
    h, ek, ev = shard.dims.heads, shard.dims.key_dim, shard.dims.value_dim
    grads = {}
    for which, name in enumerate(("q", "k", "v", "g")):
        if h * ek * ev <= ops.fd_max_state():
            pm = ops.fd_losses(*base, pr, which, step).cpu().numpy()
        else:
            pm = _fd_losses_by_recurrence(base, pr, which, step, shard.layout.chunk_len)
        grad = ((pm[:, 0] - pm[:, 1]) / (2.0 * step)).reshape(tuple(base[which].shape))
        grads[name] = grad if npo else torch.from_numpy(grad).to(base[which].device)
    return GradShard(dq=grads["q"], dk=grads["k"], dv=grads["v"], dg=grads["g"])


def _fd_losses_by_recurrence(base, probe, which, step, C):
    x = base[which].clone()
    flat = x.view(-1)
    out = np.empty((flat.numel(), 2))
    args = list(base)
    args[which] = x
    for i in range(flat.numel()):
        orig = flat[i].item()
        for col, bump in ((0, step), (1, -step)):
            flat[i] = orig + bump
            o, _, _ = ops.recurrent_forward(*args, C)
            out[i, col] = float((probe * o).sum().item())
        flat[i] = orig
    return out
