"""GLA layer / model wrapper on the ZeCO kernels vs a plain-torch float64 GLA.
Tolerances: bf16 rtol 1e-2 (relative Frobenius), fp32 mode 1e-4."""

import math

import pytest
import torch

from tests.helpers import TOL_BF16, TOL_F32

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double(), b.double()
    s = max(a.norm().item(), b.norm().item())
    return 0.0 if s == 0 else (a - b).norm().item() / s


def _inputs(h, L, d, dtype, seed=0, lo=math.log(0.9), hi=math.log(0.999)):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    u = lambda a, b, dt: (torch.rand((h, L, d), device="cuda", generator=gen) * (b - a) + a).to(dt)  # noqa: E731
    q, k, v = (u(-1, 1, dtype) for _ in range(3))
    g = u(lo, hi, torch.float32 if dtype != torch.float64 else torch.float64)
    w = u(-1, 1, torch.float64)
    return q, k, v, g, w


@pytest.mark.parametrize("dtype,tol,D", [(torch.bfloat16, TOL_BF16, 128), (torch.float32, TOL_F32, 128),
                                         (torch.bfloat16, TOL_BF16, 64)])
def test_autograd_function_vs_torch_reference(dtype, tol, D):
    from paper_2507_01004_b200.layer import gla_reference, zeco_gla
    q, k, v, g, w = _inputs(2, 256, D, dtype)
    leaves = [x.clone().requires_grad_(True) for x in (q, k, v, g)]
    o = zeco_gla(*leaves)
    (o.double() * w).sum().backward()
    ref = [x.detach().double().requires_grad_(True) for x in (q, k, v, g)]
    o_ref = gla_reference(*ref)
    (o_ref * w).sum().backward()
    assert rel(o.detach(), o_ref.detach()) <= tol
    for name, a, b in zip(("dq", "dk", "dv", "dg"), leaves, ref):
        err = rel(a.grad, b.grad)
        assert err <= tol, f"{name}: {err:.3e}"


def test_layer_matches_reference_core():
    from paper_2507_01004_b200.layer import GatedLinearAttention, gla_reference
    torch.manual_seed(0)
    layer = GatedLinearAttention(hidden_size=256, num_heads=2, device="cuda")
    x = (torch.randn(512, 256, device="cuda") * 0.5).to(torch.bfloat16)
    outs, grads = [], []
    for core in (None, gla_reference):
        layer.zero_grad()
        xx = x.clone().requires_grad_(True)
        y = layer(xx, core)
        y.float().square().mean().backward()
        outs.append(y.detach())
        grads.append([xx.grad] + [p.grad.clone() for p in layer.parameters()])
    assert rel(outs[0], outs[1]) <= TOL_BF16
    for a, b in zip(*grads):
        assert rel(a, b) <= 2 * TOL_BF16


def test_model_step_and_recompute_equivalence():
    from paper_2507_01004_b200.layer import GLAConfig, GLAModel
    torch.manual_seed(0)
    cfg = GLAConfig(vocab=512, hidden=256, layers=2, heads=2, intermediate=512)
    model = GLAModel(cfg, device="cuda")
    tok = torch.randint(0, cfg.vocab, (1024,), device="cuda")
    lab = torch.roll(tok, -1)
    res = []
    for rc in (True, False):
        model.cfg.recompute = rc
        model.zero_grad()
        loss = model(tok, lab)
        loss.backward()
        res.append((loss.item(), [p.grad.clone() for p in model.parameters()]))
    assert math.isfinite(res[0][0]) and abs(res[0][0] - math.log(cfg.vocab)) < 1.0
    assert res[0][0] == res[1][0]
    for a, b in zip(res[0][1], res[1][1]):
        assert torch.equal(a, b)


def test_layer_d64_heads_strided_plumbing():
    """32 x 64-style heads (4 x 64 here) through the layer: the zero-copy strided path (projection head
    slices in, token-major outputs / gradients) must give exactly what dense copies give, and the output
    must match the float64 reference core.  (x.grad is not compared against the reference: the per-head
    RMS norm of rows with |o| ~1e-3 of the median amplifies bf16 rounding of the core output -- the
    core's own gradients are checked against the reference in test_autograd_function_vs_torch_reference.)"""
    from paper_2507_01004_b200.layer import GatedLinearAttention, gla_reference, zeco_gla
    torch.manual_seed(1)
    layer = GatedLinearAttention(hidden_size=256, num_heads=4, device="cuda")
    x = (torch.randn(512, 256, device="cuda") * 0.5).to(torch.bfloat16)

    def dense(q, k, v, g, *a):
        return zeco_gla(q.contiguous(), k.contiguous(), v.contiguous(), g.contiguous()).contiguous()
    outs = []
    for core in (None, dense, gla_reference):
        layer.zero_grad()
        xx = x.clone().requires_grad_(True)
        y = layer(xx, core)
        y.float().square().mean().backward()
        outs.append((y.detach(), xx.grad.clone(), [p.grad.clone() for p in layer.parameters()]))
    assert torch.equal(outs[0][0], outs[1][0])
    assert rel(outs[0][1], outs[1][1]) <= 1e-6
    for a, b in zip(outs[0][2], outs[1][2]):
        assert rel(a, b) <= 1e-6
    assert rel(outs[0][0], outs[2][0]) <= TOL_BF16


def test_layer_shards_do_not_watch_the_domain():
    """The layer builds one shard per call and never polls it: no host-mapped domain word per call (a
    cudaHostAlloc / cudaFreeHost pair per shard synchronised the device and slowed GLA-1.3B by ~50 %)."""
    import torch
    from paper_2507_01004_b200 import ops
    a = ops.ZecoShard(2, 256, 128, 128, 64, torch.bfloat16, watch_domain=False)
    b = ops.ZecoShard(2, 256, 128, 128, 64, torch.bfloat16)
    assert a._dom is None and b._dom is not None


def test_layer_no_grad_forward_matches():
    """Under torch.no_grad() the layer skips the saved chunk states (forward only); outputs are bit-identical."""
    from paper_2507_01004_b200.layer import zeco_gla
    q, k, v, g, _ = _inputs(2, 512, 128, torch.bfloat16)
    a = zeco_gla(*(x.clone().requires_grad_(True) for x in (q, k, v, g))).detach()
    with torch.no_grad():
        b = zeco_gla(q, k, v, g)
    assert torch.equal(a, b)
