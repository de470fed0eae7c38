"""GLA layer and model on top of the ZeCO kernels (BASELINE config 5).

The reference lab consumes q, k, v, g directly and has no model;
this module is the wrapper a training stack needs around the hot path:

* ``ZecoGLAFunction`` -- torch.autograd.Function over the per-rank ZeCO entry
  points (glasp/engine.py:218-237 forward, 348-364 backward): local scan ->
  All-Scan FWD -> outputs with the fused correction; local reverse scan ->
  All-Scan BWD -> gradients with the fused corrections.  Tensors are
  ``[h, L, d]`` (the reference layout, glasp/gla.py:29-30) and may be strided views of
  token-major buffers (zgla_tensor strides, no transposing copies); the per-call ZecoShard workspace (segment
  states, saved chunk states) is a saved tensor, so activation recompute drops and regenerates it.
* ``GatedLinearAttention`` -- hidden -> q, k, v, r (one GEMM; the kernels read its head slices in place),
  low-rank log-sigmoid gate (g < 0 by construction), ZeCO GLA core, per-head
  RMS norm, swish output gate, output projection.
* ``GLAModel`` -- embedding, N x (RMSNorm -> GLA -> residual, RMSNorm ->
  SwiGLU MLP -> residual), final norm, LM head, cross-entropy loss; optional
  per-block activation recompute (torch.utils.checkpoint).

Head geometry: the fused tcgen05 kernels serve d_k = d_v = 128, so the
1.3B configuration (hidden 2048, 24 layers) uses 16 heads of 128 (the paper's
operator setting) rather than the 32 x 64 of its model runs
(PAPER.md:437); other head sizes run the fp32/fp64 SIMT kernels.  GEMMs are
cuBLAS through torch (plain library GEMMs); the only non-library kernels on
the path are this package's.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import _native, ops
from .errors import ConfigError


class ZecoGLAFunction(torch.autograd.Function):
    """o = GLA(q, k, v, g) over this rank's shard, sequence-parallel through ``comm`` (or single rank)."""

    @staticmethod
    def forward(ctx, q, k, v, g, chunk_len, comm, num_blocks):
        h, L, dk = q.shape
        dv = v.shape[2]
        # strided [h, L, d] views (e.g. head slices of token-major projections) are read in place
        q, k, v, g = (x if x.stride(2) == 1 else x.contiguous() for x in (q, k, v, g))
        shard = ops.ZecoShard(h, L, dk, dv, chunk_len, q.dtype, device=q.device, watch_domain=False)
        s_loc, g_tot = shard.fwd_local(k, v, g)
        prev = None
        world = comm.world if comm is not None else 1
        rank = comm.rank if comm is not None else 0
        if world > 1:
            recv, _ = comm(s_loc, g_tot, num_blocks, _native.ZGLA_FWD)
            prev = recv if rank > 0 else None
        # outputs and gradients are produced token-major ([L, h, d] storage, [h, L, d] views), the layout the
        # surrounding GEMMs consume: the runtime-stride kernel variant costs ~10 % of the core
        # (scripts/strided_bench.py) but saves the transposing copies (GLA-1.3B step 2.06 -> 1.87 s)
        # forward-only calls (no input needs a gradient: torch.no_grad() evaluation) skip the chunk-start
        # states that only the backward reads
        o = shard.fwd_output(q, k, v, g, prev, out=_token_major(h, L, dv, q.dtype, q.device),
                             save_states=any(ctx.needs_input_grad[:4]))
        # everything the backward needs goes through save_for_backward -- including the shard's workspace
        # (segment states, saved chunk states) -- so activation checkpointing can drop and regenerate it
        none = torch.empty(0, device=q.device)
        ctx.save_for_backward(q, k, v, g, shard.ws, g_tot, prev if prev is not None else none)
        ctx.geom = (h, L, dk, dv, chunk_len, q.dtype, shard.sms)
        ctx.comm, ctx.K, ctx.world, ctx.rank = comm, num_blocks, world, rank
        return o

    @staticmethod
    def backward(ctx, d_out):
        q, k, v, g, ws, g_tot, prev = ctx.saved_tensors
        h, L, dk, dv, C, dt, sms = ctx.geom
        shard = ops.ZecoShard(h, L, dk, dv, C, dt, device=q.device, sms=sms, ws=ws)
        prev = prev if prev.numel() else None
        d_out = d_out.to(q.dtype)
        if d_out.stride(2) != 1:
            d_out = d_out.contiguous()
        ds0 = shard.bwd_local(q, g, d_out)
        ds_next = None
        if ctx.world > 1:
            recv, _ = ctx.comm(ds0, g_tot, ctx.K, _native.ZGLA_BWD)
            ds_next = recv if ctx.rank < ctx.world - 1 else None
        h, L, dk_, dv_ = q.shape[0], q.shape[1], q.shape[2], v.shape[2]
        grads = (_token_major(h, L, dk_, q.dtype, q.device), _token_major(h, L, dk_, q.dtype, q.device),
                 _token_major(h, L, dv_, q.dtype, q.device), _token_major(h, L, dk_, g.dtype, q.device))
        dq, dk, dv, dg = shard.bwd_output(q, k, v, g, d_out, prev, ds_next, grads=grads)
        return dq, dk, dv, dg, None, None, None


def _token_major(h, L, d, dtype, device):
    """[h, L, d] view over [L, h, d] storage."""
    return torch.empty((L, h, d), dtype=dtype, device=device).transpose(0, 1)


def zeco_gla(q, k, v, g, chunk_len=64, comm=None, num_blocks=4):
    """Functional form: q, k [h, L, dk], v [h, L, dv] (bf16/fp32/fp64), g [h, L, dk] log gates < 0 (fp32/fp64)."""
    return ZecoGLAFunction.apply(q, k, v, g, chunk_len, comm, num_blocks)


class RMSNorm(nn.Module):
    def __init__(self, dim, eps=1e-6):
        super().__init__()
        self.eps = eps
        self.weight = nn.Parameter(torch.ones(dim))

    def forward(self, x):
        return F.rms_norm(x, (x.shape[-1],), self.weight.to(x.dtype), self.eps)


class GatedLinearAttention(nn.Module):
    """One GLA token mixer over a [L, hidden] sequence shard (batch 1, like the reference)."""

    def __init__(self, hidden_size=2048, num_heads=16, gate_low_rank_dim=16, gate_logit_normalizer=16.0,
                 chunk_len=64, comm=None, num_blocks=4, norm_eps=1e-6, dtype=torch.bfloat16, device=None):
        super().__init__()
        if hidden_size % num_heads:
            raise ConfigError(f"hidden_size {hidden_size} not divisible by num_heads {num_heads}")
        self.hidden, self.H = hidden_size, num_heads
        self.d = hidden_size // num_heads
        self.C, self.comm, self.K = chunk_len, comm, num_blocks
        self.normalizer = gate_logit_normalizer
        kw = dict(device=device, dtype=dtype)
        std = hidden_size ** -0.5
        # one GEMM for q, k, v and the output-gate input r: x [L, hidden] @ w_qkvr [hidden, 4 H d]
        self.w_qkvr = nn.Parameter(torch.randn(hidden_size, 4 * hidden_size, **kw) * std)
        self.wg1 = nn.Parameter(torch.randn(hidden_size, gate_low_rank_dim, **kw) * std)
        self.wg2 = nn.Parameter(torch.randn(gate_low_rank_dim, hidden_size, **kw) * gate_low_rank_dim ** -0.5)
        self.bg = nn.Parameter(torch.zeros(hidden_size, device=device, dtype=torch.float32))
        self.wo = nn.Parameter(torch.randn(hidden_size, hidden_size, **kw) * std)
        self.norm = RMSNorm(self.d, norm_eps)
        if device is not None:
            self.norm.to(device)

    def _heads(self, t):
        """[L, H d] -> [H, L, d] VIEW (no copy): the fused kernels read strided head slices in place."""
        return t.view(t.shape[0], self.H, self.d).transpose(0, 1)

    def project(self, x):
        """x [L, hidden] -> q, k, v, g [H, L, d] strided views of token-major buffers (g fp32 log gates < 0),
        r [L, H, d]."""
        qkvr = torch.matmul(x, self.w_qkvr)
        q, k, v, r = qkvr.split(self.hidden, dim=1)
        z = torch.matmul(torch.matmul(x, self.wg1), self.wg2).float() + self.bg
        g = F.logsigmoid(z) / self.normalizer
        return self._heads(q), self._heads(k), self._heads(v), self._heads(g), r.view(-1, self.H, self.d)

    def finish(self, o, r):
        """per-head RMS norm, swish output gate, output projection -> [L, hidden]."""
        y = self.norm(o.transpose(0, 1)) * F.silu(r)
        return torch.matmul(y.reshape(y.shape[0], self.hidden), self.wo)

    def forward(self, x, core=None):
        q, k, v, g, r = self.project(x)
        o = (core or zeco_gla)(q, k, v, g, self.C, self.comm, self.K)
        return self.finish(o, r)


class SwiGLU(nn.Module):
    def __init__(self, hidden, inter, dtype, device):
        super().__init__()
        self.gate_up = nn.Linear(hidden, 2 * inter, bias=False, dtype=dtype, device=device)
        self.down = nn.Linear(inter, hidden, bias=False, dtype=dtype, device=device)

    def forward(self, x):
        a, b = self.gate_up(x).chunk(2, dim=-1)
        return self.down(F.silu(a) * b)


class GLABlock(nn.Module):
    def __init__(self, cfg, comm, device):
        super().__init__()
        self.n1 = RMSNorm(cfg.hidden, cfg.norm_eps)
        self.attn = GatedLinearAttention(cfg.hidden, cfg.heads, cfg.gate_low_rank_dim, cfg.gate_logit_normalizer,
                                         cfg.chunk_len, comm, cfg.num_blocks, cfg.norm_eps, cfg.dtype, device)
        self.n2 = RMSNorm(cfg.hidden, cfg.norm_eps)
        self.mlp = SwiGLU(cfg.hidden, cfg.intermediate, cfg.dtype, device)
        if device is not None:
            self.n1.to(device)
            self.n2.to(device)

    def forward(self, x, core=None):
        x = x + self.attn(self.n1(x), core)
        return x + self.mlp(self.n2(x))


@dataclass
class GLAConfig:
    vocab: int = 32000
    hidden: int = 2048
    layers: int = 24
    heads: int = 16
    intermediate: int = 5632
    gate_low_rank_dim: int = 16
    gate_logit_normalizer: float = 16.0
    chunk_len: int = 64
    num_blocks: int = 4
    norm_eps: float = 1e-6
    recompute: bool = True
    dtype: torch.dtype = torch.bfloat16


GLA_1P3B = GLAConfig()  # BASELINE config 5: 24 layers, hidden 2048 (16 heads of 128)


class GLAModel(nn.Module):
    """Decoder-only GLA language model over one rank's contiguous token shard."""

    def __init__(self, cfg: GLAConfig = GLA_1P3B, comm=None, device=None):
        super().__init__()
        self.cfg = cfg
        self.embed = nn.Embedding(cfg.vocab, cfg.hidden, dtype=cfg.dtype, device=device)
        self.blocks = nn.ModuleList([GLABlock(cfg, comm, device) for _ in range(cfg.layers)])
        self.norm = RMSNorm(cfg.hidden, cfg.norm_eps)
        if device is not None:
            self.norm.to(device)
        self.head = nn.Linear(cfg.hidden, cfg.vocab, bias=False, dtype=cfg.dtype, device=device)

    def forward(self, tokens, labels=None, core=None):
        """tokens, labels [L] (this rank's shard; labels already shifted) -> mean CE loss (or logits)."""
        x = self.embed(tokens)
        for blk in self.blocks:
            if self.cfg.recompute and self.training and torch.is_grad_enabled():
                x = torch.utils.checkpoint.checkpoint(blk, x, core, use_reentrant=False)
            else:
                x = blk(x, core)
        logits = self.head(self.norm(x))
        if labels is None:
            return logits
        return F.cross_entropy(logits.float(), labels)


def num_params(model: nn.Module) -> int:
    return sum(p.numel() for p in model.parameters())


def model_flops_per_token(cfg: GLAConfig) -> float:
    """fwd+bwd FLOPs per token: 6 x (matmul params) + the GLA core (SURVEY 8(d) per token-head counts)."""
    d = cfg.hidden // cfg.heads
    per_layer = (4 * cfg.hidden * cfg.hidden + cfg.hidden * cfg.gate_low_rank_dim
                 + cfg.gate_low_rank_dim * cfg.hidden + cfg.hidden * cfg.hidden + 3 * cfg.hidden * cfg.intermediate)
    mm = 6 * (cfg.layers * per_layer + cfg.vocab * cfg.hidden)
    C = cfg.chunk_len
    core = cfg.layers * cfg.heads * ((2 * C * (d + d) + 4 * d * d) + (2 * C * (3 * d + 2 * d) + 12 * d * d))
    return float(mm + core)


def gla_reference(q, k, v, g, chunk_len=64, comm=None, num_blocks=4):
    """Plain-torch O(L^2 d) GLA in float64 (test reference only, single rank):
    O_t = sum_{j<=t} (q_t e^{G_t - G_j} . k_j) v_j  (reference recurrence, glasp/gla.py:210-230)."""
    if comm is not None and comm.world > 1:
        raise ConfigError("gla_reference is single-rank")
    qd, kd, vd, gd = (x.double() for x in (q, k, v, g))
    G = torch.cumsum(gd, dim=1)
    L = q.shape[1]
    mask = torch.tril(torch.ones(L, L, dtype=torch.bool, device=q.device))
    expo = (G[:, :, None, :] - G[:, None, :, :]).masked_fill(~mask[None, :, :, None], -math.inf)
    A = torch.einsum("htc,hjc,htjc->htj", qd, kd, torch.exp(expo))
    return torch.einsum("htj,hjv->htv", A, vd).to(q.dtype)
