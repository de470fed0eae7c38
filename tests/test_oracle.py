"""Pin the CPU oracle (oracle/gla_oracle.py) before trusting it.

1. Known-answer tests copied from the reference's own test values
   (reference tests/test_gla.py, tests/test_collectives.py).
2. Every golden vector in tests/golden/ (frozen from the reference itself by
   tests/golden/make_golden.py).
3. When /root/reference is present: the live reference on extra seeds.
"""

import math
import sys

import numpy as np
import pytest

from oracle import gla_oracle as orc
from tests.helpers import bf16_bits_to_f64, rel


# ---------------------------------------------------------------- known answers

def scalar(alphas, qs, ks, vs):
    L = len(alphas)
    g = np.log(np.asarray(alphas, dtype=np.float64)).reshape(1, L, 1)
    f = lambda x: np.asarray(x, dtype=np.float64).reshape(1, L, 1)  # noqa: E731
    return f(qs), f(ks), f(vs), g


def test_kat_recurrence_hand_example():
    # reference tests/test_gla.py:53-59
    q, k, v, g = scalar([0.5, 0.5], [1, 1], [1, 2], [1, 1])
    o, bounds = orc.recurrence(q, k, v, g, chunk_len=2)
    np.testing.assert_allclose(o.ravel(), [1.0, 2.5])
    assert bounds[1].item() == pytest.approx(2.5)


def test_kat_single_token():
    # reference tests/test_gla.py:69-72
    q, k, v, g = scalar([1 - 1e-12], [2], [3], [5])
    o, _ = orc.recurrence(q, k, v, g, chunk_len=1)
    assert o.item() == pytest.approx(30.0)


def test_kat_chunk_scalings():
    # reference tests/test_gla.py:89-94
    gam, lam, tail = orc.chunk_scalings(np.log(np.array([[[0.5], [0.5]]])))
    assert gam.item() == pytest.approx(0.25)
    np.testing.assert_allclose(lam.ravel(), [0.5, 0.25])
    np.testing.assert_allclose(tail.ravel(), [0.5, 1.0])


def test_kat_local_scan():
    # reference tests/test_gla.py:136-140
    q, k, v, g = scalar([0.5, 0.5], [1, 1], [1, 2], [1, 1])
    states, cum = orc.local_scan(k, v, g, 2)
    assert states[0, 1].item() == pytest.approx(2.5)
    assert cum[0, 1].item() == pytest.approx(math.log(0.25))


def test_kat_global_correct():
    # reference tests/test_gla.py:168-173: log .25, prev 4, local 1 -> 2
    out = orc.lift_states(np.ones((1, 1, 1, 1)), np.full((1, 1, 1), math.log(0.25)),
                          np.full((1, 1, 1), 4.0))
    assert out.item() == pytest.approx(2.0)


def test_kat_revcum():
    # reference tests/test_gla.py:182-184
    np.testing.assert_array_equal(orc.rev_cumsum(np.array([[[1.0], [2.0], [3.0]]])).ravel(), [6, 5, 3])


def test_kat_allscan_scalar():
    # reference tests/test_collectives.py:55-62
    local = [np.full((1, 1, 1), x) for x in (1.0, 2.0, 3.0)]
    logs = [np.full((1, 1), x) for x in (0.0, math.log(0.5), math.log(0.5))]
    recv, scanned = orc.scan_ranks(local, logs)
    assert [s.item() for s in scanned] == pytest.approx([1.0, 2.5, 4.25])
    assert recv[2].item() == pytest.approx(2.5)


# ---------------------------------------------------------------- golden vectors

def _inputs(case):
    if "q_bits" in case:
        q, k, v, do = (bf16_bits_to_f64(case[f"{n}_bits"]) for n in ("q", "k", "v", "do"))
        return q, k, v, case["g"].astype(np.float64), do
    return case["q"], case["k"], case["v"], case["g"], case["do"]


@pytest.mark.parametrize("name", ["zeco_f64_p4", "zeco_bf16_d64_p2", "zeco_bf16_d128_p2_long"])
def test_oracle_matches_golden_strategy(golden, name):
    case = golden(name)
    P, C = int(case["P"]), int(case["C"])
    q, k, v, g, do = _inputs(case)
    o, saved, bounds = orc.zeco_forward(q, k, v, g, P, C)
    tol = 1e-12 if name.endswith("p4") else 1e-6  # bf16 fixtures stored as float32
    assert rel(o, case["o"]) <= tol
    assert rel(np.stack(saved["prev"]), case["prev"]) <= 1e-12
    assert rel(np.stack(bounds).transpose(0, 2, 1, 3, 4), case["bounds"]) <= tol
    (dq, dk, dv, dg), _ = orc.zeco_backward(q, k, v, g, do, P, C, saved)
    for got, key in ((dq, "dq"), (dk, "dk_"), (dv, "dv_"), (dg, "dg")):
        assert rel(got, case[key]) <= tol, key


def test_oracle_matches_golden_functions(golden):
    c = golden("gla_functions")
    C = int(c["C"])
    states, cum = orc.local_scan(c["k"], c["v"], c["g"], C)
    assert rel(states, c["states"]) <= 1e-13
    assert rel(cum, c["cum"]) <= 1e-13
    o = orc.chunk_outputs(c["q"], c["k"], c["v"], c["g"], states, cum, c["prev"], C)
    assert rel(o, c["o"]) <= 1e-13
    assert rel(orc.lift_states(states, cum, c["prev"]), c["corrected"]) <= 1e-13
    assert rel(orc.boundary_cotangents(c["q"], c["g"], c["do"], C), c["rev"]) <= 1e-13
    dq, dk, dv, dg, dsb = orc.chunk_backward(c["q"], c["k"], c["v"], c["g"], c["do"],
                                             c["prev"], c["ds_next"], C)
    for got, key in ((dq, "dq"), (dk, "dk_"), (dv, "dv_"), (dg, "dg"), (dsb, "ds_boundary")):
        assert rel(got, c[key]) <= 1e-12, key
    ro, rb = orc.recurrence(c["q"], c["k"], c["v"], c["g"], C, init=c["prev"])
    assert rel(ro, c["rec_o"]) <= 1e-13
    assert rel(np.stack(rb, axis=1), c["rec_bounds"]) <= 1e-13
    np.testing.assert_allclose(orc.rev_cumsum(c["revcum_in"][None])[0], c["revcum_out"])


@pytest.mark.parametrize("name", ["allscan_f64_p5", "allscan_f32_p8"])
def test_oracle_matches_golden_allscan(golden, name):
    c = golden(name)
    local, logs = list(c["local"]), list(c["logdecay"])
    recv, scanned = orc.scan_ranks(local, logs)
    np.testing.assert_allclose(np.stack(recv), c["recv_fwd"], rtol=1e-6 if "f32" in name else 0)
    np.testing.assert_allclose(np.stack(scanned), c["scanned_fwd"], rtol=1e-6 if "f32" in name else 0)
    recv_b, scanned_b = orc.scan_ranks(local[::-1], logs[::-1])
    np.testing.assert_allclose(np.stack(recv_b[::-1]), c["recv_bwd"], rtol=1e-6 if "f32" in name else 0)
    np.testing.assert_allclose(np.stack(scanned_b[::-1]), c["scanned_bwd"],
                               rtol=1e-6 if "f32" in name else 0)


def test_golden_ledger_contract(golden):
    # ZeCO: every non-terminal rank sends one state per direction (tests/test_engine.py:111-122)
    c = golden("zeco_f64_p4")
    state_el = int(c["h"]) * int(c["dk"]) * int(c["dv"])
    # fwd chain 0->3 (ranks 0..2 send), bwd chain 3->0 (ranks 1..3 send)
    np.testing.assert_array_equal(c["sent_per_rank"], [state_el, 2 * state_el, 2 * state_el, state_el])
    a = golden("allscan_f64_p5")
    el = a["local"][0].size
    np.testing.assert_array_equal(a["sent_fwd"], [el] * 4 + [0])
    np.testing.assert_array_equal(a["sent_bwd"], [0] + [el] * 4)


# ---------------------------------------------------------------- live reference

@pytest.mark.reference
@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("P,L,C", [(1, 64, 16), (2, 48, 16), (4, 32, 8)])
def test_oracle_matches_live_reference(seed, P, L, C):
    sys.path.insert(0, "/root/reference/pkg/src")
    from glasp import ModelDims, generate_sequence
    from glasp.cluster import NetConfig, create_cluster
    from glasp.collectives import PipelineConfig
    from glasp.engine import StrategyKind, run_backward, run_forward

    seq = generate_sequence(P, L, C, ModelDims(3, 5, 4), seed)
    do = orc.make_cotangent(seed, 3, P * L, 4)
    cl = create_cluster(P, NetConfig())
    f = run_forward(seq, StrategyKind.ZECO, cl, PipelineConfig(1))
    b = run_backward(seq, do, StrategyKind.ZECO, cl, PipelineConfig(1), f)
    q, k, v, g = orc.make_inputs(P, L, 3, 5, 4, seed)
    np.testing.assert_array_equal(q, seq.q)
    np.testing.assert_array_equal(g, seq.g)
    o, saved, _ = orc.zeco_forward(q, k, v, g, P, C)
    assert rel(o, f.outputs) <= 1e-12
    (dq, dk, dv, dg), _ = orc.zeco_backward(q, k, v, g, do, P, C, saved)
    for got, want in ((dq, b.grads.dq), (dk, b.grads.dk), (dv, b.grads.dv), (dg, b.grads.dg)):
        assert rel(got, want) <= 1e-12
