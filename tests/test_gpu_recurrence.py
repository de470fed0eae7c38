"""The drop-in's independent oracles on the GPU: recurrent_forward (token recurrence kernel,
csrc/recurrence.cu) against the CPU oracle's recurrence, and finite_diff_grad (one launch per tensor of
perturbed recurrences) against the oracle's analytic gradients -- glasp/gla.py:210-230, 447-480."""

import numpy as np
import pytest

from oracle import gla_oracle as orc
from tests.helpers import rel

pytestmark = pytest.mark.gpu


def shard_of(rng, h, L, C, ek, ev, dtype=np.float64):
    from paper_2507_01004_b200 import ModelDims, SeqShard, ShardLayout
    q, k = rng.uniform(-1, 1, (h, L, ek)), rng.uniform(-1, 1, (h, L, ek))
    v = rng.uniform(-1, 1, (h, L, ev))
    g = rng.uniform(orc.DECAY_LOW, orc.DECAY_HIGH, (h, L, ek))
    return SeqShard(q=q.astype(dtype), k=k.astype(dtype), v=v.astype(dtype), g=g.astype(dtype),
                    layout=ShardLayout(L, C), dims=ModelDims(h, ek, ev))


@pytest.mark.parametrize("h,L,C,ek,ev", [(1, 64, 1, 3, 2), (2, 128, 16, 8, 5), (4, 512, 64, 64, 64),
                                         (2, 256, 64, 128, 128), (3, 96, 96, 1, 300)])
def test_recurrent_forward_matches_oracle(h, L, C, ek, ev):
    from paper_2507_01004_b200 import State, recurrent_forward
    rng = np.random.default_rng(h * 1000 + L)
    sh = shard_of(rng, h, L, C, ek, ev)
    init = State(rng.uniform(-1, 1, (h, ek, ev)))
    o, bounds, final = recurrent_forward(sh, init)
    o_ref, b_ref = orc.recurrence(sh.q, sh.k, sh.v, sh.g, C, init=init.values)
    assert rel(o, o_ref) <= 1e-12
    assert len(bounds) == L // C + 1
    for got, want in zip(bounds, b_ref):
        assert rel(got.values, want) <= 1e-12
    assert rel(final.values, b_ref[-1]) <= 1e-12
    np.testing.assert_array_equal(bounds[0].values, init.values)


def test_recurrent_forward_fp32_mode():
    from paper_2507_01004_b200 import recurrent_forward
    sh = shard_of(np.random.default_rng(7), 2, 256, 64, 64, 64, np.float32)
    o, _, _ = recurrent_forward(sh)
    o_ref, _ = orc.recurrence(*(x.astype(np.float64) for x in (sh.q, sh.k, sh.v, sh.g)), 64)
    assert o.dtype == np.float32 and rel(o, o_ref) <= 1e-5


def test_finite_diff_grad_matches_analytic():
    from paper_2507_01004_b200 import finite_diff_grad
    for seed in range(4):
        rng = np.random.default_rng(2000 + seed)
        sh = shard_of(rng, 2, 8, 4, 3, 2)
        probe = rng.uniform(-1, 1, (2, 8, 2))
        fd = finite_diff_grad(sh, probe, step=1e-5)
        o, saved, _ = orc.zeco_forward(sh.q, sh.k, sh.v, sh.g, 1, 4)
        (dq, dk, dv, dg), _ = orc.zeco_backward(sh.q, sh.k, sh.v, sh.g, probe, 1, 4, saved)
        for got, want in ((fd.dq, dq), (fd.dk, dk), (fd.dv, dv), (fd.dg, dg)):
            assert rel(got, want) <= 1e-7


def test_finite_diff_grad_causality_and_large_state_path():
    """probe on the first token only: later tokens get exactly zero; a state above the shared-memory budget
    takes the per-perturbation recurrence path and agrees with the batched kernel."""
    from paper_2507_01004_b200 import finite_diff_grad, ops
    rng = np.random.default_rng(11)
    sh = shard_of(rng, 1, 4, 2, 2, 2)
    probe = np.zeros((1, 4, 2))
    probe[:, 0, :] = 1.0
    fd = finite_diff_grad(sh, probe, step=1e-5)
    for arr in (fd.dq, fd.dk, fd.dv, fd.dg):
        np.testing.assert_allclose(arr[:, 1:, :], 0.0, atol=1e-9)
    import torch
    base = [torch.from_numpy(x).cuda() for x in (sh.q, sh.k, sh.v, sh.g)]
    pr = torch.from_numpy(rng.uniform(-1, 1, (1, 4, 2))).cuda()
    from paper_2507_01004_b200.gla import _fd_losses_by_recurrence
    for which in range(4):
        a = ops.fd_losses(*base, pr, which, 1e-5).cpu().numpy()
        b = _fd_losses_by_recurrence(base, pr, which, 1e-5, 2)
        np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-15)
