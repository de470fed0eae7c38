"""Drop-in behaviour of the strategy engine on the GPU, in the reference's own terms
(reference tests/test_engine.py, tests/test_collectives.py, cli verify): float64 inputs
run the exact kernels, so the reference's f64 tolerances apply unchanged."""

import math

import numpy as np
import pytest
import torch

from oracle import gla_oracle as orc
from tests.helpers import TOL_BF16, rel

pytestmark = pytest.mark.gpu

DISTRIBUTED = ["ZECO", "LASP1", "LASP2"]


def make_seq(seed, P=4, L=32, C=8, h=2, ek=4, ev=4, **kw):
    from paper_2507_01004_b200 import ModelDims, generate_sequence
    return generate_sequence(num_ranks=P, tokens_per_rank=L, chunk_len=C,
                             dims=ModelDims(heads=h, key_dim=ek, value_dim=ev), seed=seed, **kw)


def fwd(seq, strategy, K=2):
    from paper_2507_01004_b200 import PipelineConfig, StrategyKind, create_cluster, run_forward
    st = getattr(StrategyKind, strategy)
    P = 1 if st is StrategyKind.SINGLE_DEVICE else seq.num_ranks
    cl = create_cluster(P)
    return run_forward(seq, st, cl, PipelineConfig(K)), cl


def bwd(seq, do, strategy, art, cl, K=2):
    from paper_2507_01004_b200 import PipelineConfig, StrategyKind, run_backward
    return run_backward(seq, do, getattr(StrategyKind, strategy), cl, PipelineConfig(K), art)


@pytest.mark.parametrize("strategy", DISTRIBUTED)
def test_forward_matches_single_device(strategy):
    seq = make_seq(10, P=4, L=128, C=32, h=2, ek=8, ev=8)
    want = fwd(seq, "SINGLE_DEVICE")[0].outputs
    got = fwd(seq, strategy)[0].outputs
    assert isinstance(got, np.ndarray) and got.dtype == np.float64
    assert rel(got, want) <= 1e-10


def test_forward_matches_oracle_and_recurrence():
    seq = make_seq(11, P=2, L=32, C=8)
    o_ref, _ = orc.recurrence(seq.q, seq.k, seq.v, seq.g, 8)
    for strategy in DISTRIBUTED:
        assert rel(fwd(seq, strategy)[0].outputs, o_ref) <= 1e-10


def test_p1_zeco_bitwise_equals_single():
    seq = make_seq(12, P=1, L=64, C=16)
    a = fwd(seq, "ZECO")[0].outputs
    b = fwd(seq, "SINGLE_DEVICE")[0].outputs
    assert a.tobytes() == b.tobytes()


def test_p1_zeco_zero_communication():
    art, _ = fwd(make_seq(13, P=1), "ZECO")
    assert art.ledger.total_sent == 0 and art.ledger.total_received == 0


def test_boundary_states_match_recurrence():
    seq = make_seq(14, P=4, L=32, C=8)
    _, bounds = orc.recurrence(seq.q, seq.k, seq.v, seq.g, 8)
    art, _ = fwd(seq, "ZECO")
    N = seq.layout.num_chunks
    for r, states in enumerate(art.boundary_states):
        for n, st in enumerate(states):
            assert rel(st.values, bounds[r * N + n]) <= 1e-12


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("strategy", DISTRIBUTED + ["SINGLE_DEVICE"])
def test_backward_matches_oracle(P, strategy):
    """Every strategy's gradients against the f64 CPU oracle (oracle/gla_oracle.py, pinned to the reference)."""
    seq = make_seq(20 + P, P=P, L=64, C=16, h=2, ek=4, ev=3)
    do = np.random.default_rng(99).uniform(-1, 1, (2, P * 64, 3))
    o_want, saved, _ = orc.zeco_forward(seq.q, seq.k, seq.v, seq.g, P, 16)
    want, _ = orc.zeco_backward(seq.q, seq.k, seq.v, seq.g, do, P, 16, saved)
    a1, c1 = fwd(seq, strategy)
    assert rel(a1.outputs, o_want) <= 1e-10
    got = bwd(seq, do, strategy, a1, c1).grads
    for name, w in zip(("dq", "dk", "dv", "dg"), want):
        assert rel(getattr(got, name), w) <= 1e-10, name


def test_zeco_volume_contract():
    seq = make_seq(30, P=4, L=32, C=8, h=1, ek=128, ev=128)
    art, cl = fwd(seq, "ZECO")
    led = art.ledger
    for r in range(3):
        assert led.sent(rank=r, primitive="all_scan") == 16384
    assert led.sent(rank=3, primitive="all_scan") == 0
    do = np.zeros((1, 4 * 32, 128))
    back = bwd(seq, do, "ZECO", art, cl)
    # zero cotangent still runs the backward All-Scan: 3 more states sent (reference tests/test_engine.py:155-166)
    assert back.ledger.total_sent == 6 * 16384
    for name in ("dq", "dk", "dv", "dg"):
        assert np.all(getattr(back.grads, name) == 0.0)


def test_state_errors():
    from paper_2507_01004_b200 import StateError
    seq = make_seq(31, P=2)
    art, cl = fwd(seq, "ZECO")
    with pytest.raises(StateError):
        bwd(seq, np.zeros((2, 64, 4)), "LASP2", art, cl)


def test_engine_bf16_fast_path_long_memory():
    """bf16 torch inputs through the drop-in engine select the tcgen05 kernels (P=4 ranks on one GPU)."""
    seq = make_seq(40, P=4, L=512, C=64, h=2, ek=128, ev=128, precision="bf16",
                   decay_low=math.log(0.9999), decay_high=math.log(0.99999))
    do = torch.rand(2, 4 * 512, 128, device="cuda", dtype=torch.float32).mul(2).sub(1).to(torch.bfloat16)
    from paper_2507_01004_b200 import ops
    assert ops.ZecoShard(2, 512, 128, 128, 64, torch.bfloat16).fast
    art, cl = fwd(seq, "ZECO", K=4)
    grads = bwd(seq, do, "ZECO", art, cl, K=4).grads
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    q, k, v, g = f(seq.q), f(seq.k), f(seq.v), f(seq.g)
    o, saved, _ = orc.zeco_forward(q, k, v, g, 4, 64)
    (dq, dk, dv, dg), _ = orc.zeco_backward(q, k, v, g, f(do), 4, 64, saved)
    assert rel(f(art.outputs), o) <= TOL_BF16
    for got, want in ((grads.dq, dq), (grads.dk, dk), (grads.dv, dv), (grads.dg, dg)):
        assert rel(f(got), want) <= TOL_BF16


def test_engine_bf16_any_gate_the_reference_accepts():
    """Gates far outside the fused path's exponent domain (per-token decay 0.02-0.05: a 64-token tile's
    log-decay near -200) are accepted by the drop-in engine like the reference accepts them: the call
    widens to the fp32 kernels (exact token recurrence) and returns bf16 outputs/gradients."""
    seq = make_seq(41, P=2, L=256, C=64, h=2, ek=128, ev=128, precision="bf16",
                   decay_low=math.log(0.02), decay_high=math.log(0.05))
    do = torch.rand(2, 2 * 256, 128, device="cuda", dtype=torch.float32).mul(2).sub(1).to(torch.bfloat16)
    art, cl = fwd(seq, "ZECO", K=4)
    grads = bwd(seq, do, "ZECO", art, cl, K=4).grads
    assert art.outputs.dtype == torch.bfloat16 and grads.dq.dtype == torch.bfloat16
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    q, k, v, g = f(seq.q), f(seq.k), f(seq.v), f(seq.g)
    o, saved, _ = orc.zeco_forward(q, k, v, g, 2, 64)
    (dq, dk, dv, dg), _ = orc.zeco_backward(q, k, v, g, f(do), 2, 64, saved)
    assert rel(f(art.outputs), o) <= TOL_BF16
    for got, want in ((grads.dq, dq), (grads.dk, dk), (grads.dv, dv), (grads.dg, dg)):
        assert rel(f(got), want) <= TOL_BF16


@pytest.mark.parametrize("G", [2, 4])
def test_overlap_schedule_matches_serial(G):
    """ZecoRank(overlap_groups=G) -- All-Scan per head group on a communication stream, here an injected-
    latency stand-in (LatencyChain: recv = 0) -- gives the serial schedule's results within the bf16
    tolerance, eagerly and replayed from a CUDA graph."""
    from paper_2507_01004_b200 import distributed as zd
    torch.manual_seed(1)
    H, L, D = 8, 2048, 128
    q, k, v, do = ((torch.rand(H, L, D, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(4))
    g = torch.rand(H, L, D, device="cuda") * (math.log(0.999) - math.log(0.9)) + math.log(0.9)

    def run(groups, graph=False):
        layer = zd.ZecoRank(H, L, D, 64, torch.bfloat16, comm=zd.LatencyChain(5000), overlap_groups=groups)
        o = torch.empty_like(q)
        grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty_like(g))

        def step():
            layer.forward(q, k, v, g, out=o)
            layer.backward(q, k, v, g, do, grads=grads)
        step()
        if graph:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream().wait_stream(side)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                step()
            for t in (o,) + grads:
                t.zero_()
            gr.replay()
        torch.cuda.synchronize()
        return [t.double().cpu().numpy() for t in (o,) + grads]

    a = run(1)
    for graph in (False, True):
        b = run(G, graph)
        for x, y in zip(a, b):
            assert rel(y, x) <= 5e-3
