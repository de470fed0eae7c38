"""The host-buffer layer call (zgla_zeco_fwd_bwd_host, via ZecoRank.forward_backward_host):
head groups pipelined H2D -> kernels -> D2H must give the device path's results.

* head_groups = 1 runs exactly the device path's plan: bitwise equal;
* head_groups > 1 re-plans the segments per group (different fp32 summation order): checked
  against the CPU oracle at the north-star tolerance (bf16 rtol 1e-2, fp32 mode 1e-4)."""

import numpy as np
import pytest
import torch

from oracle import gla_oracle as orc
from tests.helpers import TOL_BF16, TOL_F32, rel

pytestmark = pytest.mark.gpu


def _case(h, L, D, dtype, seed=3):
    q, k, v, g = orc.make_inputs(1, L, h, D, D, seed, orc.LONG_DECAY_LOW, orc.LONG_DECAY_HIGH)
    do = orc.make_cotangent(seed, h, L, D)
    acc = torch.float32
    host = [torch.from_numpy(np.ascontiguousarray(x)).to(dt).pin_memory()
            for x, dt in ((q, dtype), (k, dtype), (v, dtype), (g, acc), (do, dtype))]
    return host


def _outs(h, L, D, dtype):
    return [torch.empty((h, L, D), dtype=dt).pin_memory() for dt in (dtype, dtype, dtype, dtype, torch.float32)]


def _device_path(host, h, L, D, dtype):
    from paper_2507_01004_b200 import distributed as zd
    layer = zd.ZecoRank(h, L, D, 64, dtype)
    q, k, v, g, do = (x.cuda() for x in host)
    o = layer.forward(q, k, v, g)
    grads = layer.backward(q, k, v, g, do)
    torch.cuda.synchronize()
    return [o.cpu()] + [x.cpu() for x in grads]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_host_call_one_group_bitwise(dtype):
    from paper_2507_01004_b200 import distributed as zd
    h, L, D = 4, 512, 128
    host = _case(h, L, D, dtype)
    want = _device_path(host, h, L, D, dtype)
    layer = zd.ZecoRank(h, L, D, 64, dtype)
    out = _outs(h, L, D, dtype)
    layer.forward_backward_host(host, out, head_groups=1)
    torch.cuda.current_stream().synchronize()
    for name, a, b in zip(("o", "dq", "dk", "dv", "dg"), out, want):
        assert torch.equal(a, b), name


@pytest.mark.parametrize("dtype,groups,h", [(torch.bfloat16, 2, 4), (torch.bfloat16, 4, 4), (torch.float32, 4, 4),
                                           (torch.bfloat16, 3, 6), (torch.bfloat16, 4, 7)])
def test_host_call_groups_vs_oracle(dtype, groups, h):
    """groups of 1 head at both ends (tapered split) when heads > groups, uniform otherwise"""
    from paper_2507_01004_b200 import distributed as zd
    L, D = 512, 128
    host = _case(h, L, D, dtype)
    layer = zd.ZecoRank(h, L, D, 64, dtype)
    out = _outs(h, L, D, dtype)
    # run twice: the second call reuses streams, events and the device buffer
    for _ in range(2):
        for t in out:
            t.zero_()
        layer.forward_backward_host(host, out, head_groups=groups)
        torch.cuda.current_stream().synchronize()
    q, k, v, g, do = (x.double().numpy() for x in host)
    want_o, saved, _ = orc.zeco_forward(q, k, v, g, 1, 64)
    want_g, _ = orc.zeco_backward(q, k, v, g, do, 1, 64, saved)
    tol = TOL_BF16 if dtype == torch.bfloat16 else TOL_F32
    for name, a, b in zip(("o", "dq", "dk", "dv", "dg"), out, [want_o] + list(want_g)):
        err = rel(a.double().numpy(), b)
        assert err <= tol, f"{name}: rel err {err:.3e} > {tol}"


def test_host_call_rejects_bad_args():
    from paper_2507_01004_b200 import distributed as zd
    from paper_2507_01004_b200.errors import ConfigError
    h, L, D = 4, 256, 128
    host = _case(h, L, D, torch.bfloat16)
    layer = zd.ZecoRank(h, L, D, 64, torch.bfloat16)
    out = _outs(h, L, D, torch.bfloat16)
    with pytest.raises(ConfigError):
        layer.forward_backward_host(host, out, head_groups=5)
    with pytest.raises(ConfigError):
        layer.forward_backward_host([x.cuda() for x in host], out, head_groups=1)


def test_host_call_overlap_chain_matches():
    """overlap=True: consecutive calls chained through per-group events give the same results as the
    stream-ordered call once host_wait() has been honoured (inputs changed between calls)."""
    from paper_2507_01004_b200 import distributed as zd
    h, L, D = 4, 512, 128
    layer = zd.ZecoRank(h, L, D, 64, torch.bfloat16)
    cases = [_case(h, L, D, torch.bfloat16, seed=s) for s in (1, 2, 3)]
    want = []
    for host in cases:
        out = _outs(h, L, D, torch.bfloat16)
        layer.forward_backward_host(host, out, head_groups=2)
        torch.cuda.current_stream().synchronize()
        want.append(out)
    outs = [_outs(h, L, D, torch.bfloat16) for _ in cases]
    for host, out in zip(cases, outs):
        layer.forward_backward_host(host, out, head_groups=2, overlap=True)
    layer.host_wait()
    torch.cuda.current_stream().synchronize()
    for a_set, b_set in zip(outs, want):
        for a, b in zip(a_set, b_set):
            assert torch.equal(a, b)


def test_host_call_d64_vs_oracle():
    """The host-buffer call on d = 64 heads (fused path with zero-filled channels)."""
    from paper_2507_01004_b200 import distributed as zd
    h, L, D = 4, 512, 64
    host = _case(h, L, D, torch.bfloat16, seed=9)
    layer = zd.ZecoRank(h, L, D, 64, torch.bfloat16)
    assert layer.shard.fast
    out = _outs(h, L, D, torch.bfloat16)
    layer.forward_backward_host(host, out, head_groups=2)
    torch.cuda.current_stream().synchronize()
    q, k, v, g, do = (x.double().numpy() for x in host)
    want_o, saved, _ = orc.zeco_forward(q, k, v, g, 1, 64)
    want_g, _ = orc.zeco_backward(q, k, v, g, do, 1, 64, saved)
    for name, a, b in zip(("o", "dq", "dk", "dv", "dg"), out, [want_o] + list(want_g)):
        err = rel(a.double().numpy(), b)
        assert err <= TOL_BF16, f"{name}: rel err {err:.3e}"


def _arena(tensors, gap=256):
    """pinned tensors carved back to back from one buffer (equal pitch for equal sizes): the layout whose
    equal-sized head-group slices the host call moves with one 2-D copy per direction"""
    sizes = [x.numel() * x.element_size() for x in tensors]
    offs = [0]
    for b in sizes[:-1]:
        offs.append(offs[-1] + (b + gap - 1) // gap * gap)
    buf = torch.empty(offs[-1] + sizes[-1], dtype=torch.uint8).pin_memory()
    out = [buf[o:o + b].view(x.dtype).view(x.shape) for o, b, x in zip(offs, sizes, tensors)]
    for a, x in zip(out, tensors):
        a.copy_(x)
    return out


@pytest.mark.parametrize("groups,h", [(1, 4), (2, 4), (4, 7)])
def test_host_call_arena_layout_bitwise(groups, h):
    """inputs q k v dO g and outputs o dq dk dv dg carved from one pinned arena each (2-D copies of the
    equal-sized tensors) give bit-identical results to separate pinned buffers (one copy per tensor)"""
    from paper_2507_01004_b200 import distributed as zd
    L, D, dt = 512, 128, torch.bfloat16
    host = _case(h, L, D, dt)
    layer = zd.ZecoRank(h, L, D, 64, dt)
    out_sep = _outs(h, L, D, dt)
    layer.forward_backward_host(host, out_sep, head_groups=groups)
    torch.cuda.current_stream().synchronize()
    q, k, v, g, do = host
    aq, ak, av, ado, ag = _arena([q, k, v, do, g])
    out_ar = _arena([torch.zeros_like(x) for x in out_sep])
    layer.forward_backward_host([aq, ak, av, ag, ado], out_ar, head_groups=groups)
    torch.cuda.current_stream().synchronize()
    for name, a, b in zip(("o", "dq", "dk", "dv", "dg"), out_ar, out_sep):
        assert torch.equal(a, b), name
