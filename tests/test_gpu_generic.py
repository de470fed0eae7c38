"""Generic CUDA kernels (fp64 exact mode, fp32 validation mode) against the golden vectors
frozen from the reference, through the C ABI (paper_2507_01004_b200.ops)."""

import numpy as np
import pytest
import torch

from tests.helpers import TOL_F32, bf16_bits_to_f64, rel

pytestmark = pytest.mark.gpu


def dev(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype)


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-12), (torch.float32, TOL_F32)])
def test_function_level_api(golden, dtype, tol):
    from paper_2507_01004_b200 import ops

    c = golden("gla_functions")
    C = int(c["C"])
    q, k, v, g, do = (dev(c[n], dtype) for n in ("q", "k", "v", "g", "do"))
    prev, dsn = dev(c["prev"], dtype), dev(c["ds_next"], dtype)
    states, cum = ops.local_state_scan(k, v, g, C)
    assert rel(states.permute(1, 0, 2, 3).cpu(), c["states"]) <= tol
    assert rel(cum.permute(1, 0, 2).cpu(), c["cum"]) <= tol
    o = ops.forward_outputs(q, k, v, g, states, cum, prev, C)
    assert rel(o.cpu(), c["o"]) <= tol
    corr = ops.global_correct(states, cum, prev)
    assert rel(corr.permute(1, 0, 2, 3).cpu(), c["corrected"]) <= tol
    rev = ops.reverse_boundary_scan(q, g, do, C)
    assert rel(rev.permute(1, 0, 2, 3).cpu(), c["rev"]) <= tol
    dq, dk, dv, dg, dsb = ops.backward(q, k, v, g, do, prev, dsn, C)
    for got, key in ((dq, "dq"), (dk, "dk_"), (dv, "dv_"), (dg, "dg"), (dsb, "ds_boundary")):
        assert rel(got.cpu(), c[key]) <= tol, key
    # saved-states variant (glasp/gla.py:398-404)
    dq2, dk2, dv2, dg2, _ = ops.backward(q, k, v, g, do, prev, dsn, C, saved_states=states)
    for got, key in ((dq2, "dq"), (dk2, "dk_"), (dv2, "dv_"), (dg2, "dg")):
        assert rel(got.cpu(), c[key]) <= tol, key
    rc = ops.revcum(dev(c["revcum_in"][None], dtype))
    assert rel(rc.cpu()[0], c["revcum_out"]) <= tol


def _zeco_case(golden, name, dtype, device_dtype_g):
    c = golden(name)
    if "q_bits" in c:
        q, k, v, do = (bf16_bits_to_f64(c[f"{n}_bits"]) for n in ("q", "k", "v", "do"))
        g = c["g"].astype(np.float64)
    else:
        q, k, v, g, do = c["q"], c["k"], c["v"], c["g"], c["do"]
    return c, [dev(x, dtype) for x in (q, k, v)] + [dev(g, device_dtype_g), dev(do, dtype)]


@pytest.mark.parametrize("name", ["zeco_f64_p4", "zeco_bf16_d64_p2", "zeco_bf16_d128_p2_long"])
@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-10), (torch.float32, TOL_F32)])
def test_zeco_ranks_generic_modes(golden, name, dtype, tol):
    """Per-rank ZeCO entry points + list-form All-Scan kernel reproduce the reference run."""
    from paper_2507_01004_b200 import ops

    c, (q, k, v, g, do) = _zeco_case(golden, name, dtype, dtype)
    P, C, K = int(c["P"]), int(c["C"]), int(c["K"])
    h, T, dk = q.shape
    L = T // P
    sl = [slice(p * L, (p + 1) * L) for p in range(P)]
    shards = [ops.ZecoShard(h, L, dk, v.shape[2], C, dtype) for _ in range(P)]
    loc = [shards[p].fwd_local(k[:, s], v[:, s], g[:, s]) for p, s in enumerate(sl)]
    recv, scanned = ops.allscan_local(torch.stack([x[0] for x in loc]), torch.stack([x[1] for x in loc]), K,
                                      0)
    assert rel(recv.cpu(), c["prev"]) <= tol
    assert rel(scanned.cpu(), c["scanned"]) <= tol
    o = torch.cat([shards[p].fwd_output(q[:, s], k[:, s], v[:, s], g[:, s], recv[p]) for p, s in enumerate(sl)], 1)
    assert rel(o.cpu(), c["o"]) <= max(tol, 2e-7)
    d0 = torch.stack([shards[p].bwd_local(q[:, s], g[:, s], do[:, s]) for p, s in enumerate(sl)])
    ds_next, _ = ops.allscan_local(d0, torch.stack([x[1] for x in loc]), K, 1)
    grads = [shards[p].bwd_output(q[:, s], k[:, s], v[:, s], g[:, s], do[:, s], recv[p], ds_next[p])
             for p, s in enumerate(sl)]
    for i, key in enumerate(("dq", "dk_", "dv_", "dg")):
        got = torch.cat([gr[i] for gr in grads], 1)
        assert rel(got.cpu(), c[key]) <= max(tol, 2e-7), key


@pytest.mark.parametrize("name", ["allscan_f64_p5", "allscan_f32_p8"])
@pytest.mark.parametrize("K", [1, 2])
def test_allscan_local_matches_reference(golden, name, K):
    from paper_2507_01004_b200 import ops

    c = golden(name)
    dt = torch.float64 if "f64" in name else torch.float32
    local, logs = dev(c["local"], dt), dev(c["logdecay"], dt)
    for direction, tag in ((0, "fwd"), (1, "bwd")):
        recv, scanned = ops.allscan_local(local, logs, K, direction)
        np.testing.assert_allclose(recv.cpu().numpy(), c[f"recv_{tag}"], rtol=1e-6 if dt == torch.float32 else 1e-14,
                                   atol=1e-7 if dt == torch.float32 else 1e-15)
        np.testing.assert_allclose(scanned.cpu().numpy(), c[f"scanned_{tag}"],
                                   rtol=1e-6 if dt == torch.float32 else 1e-14,
                                   atol=1e-7 if dt == torch.float32 else 1e-15)


def test_allscan_k_invariance_bitwise():
    from paper_2507_01004_b200 import ops

    gen = torch.Generator(device="cuda").manual_seed(3)
    local = torch.rand(4, 2, 8, 3, device="cuda", generator=gen) * 2 - 1
    logs = -2 * torch.rand(4, 2, 8, device="cuda", generator=gen)
    base = ops.allscan_local(local, logs, 1, 0)
    for K in (2, 4, 8):
        got = ops.allscan_local(local, logs, K, 0)
        assert torch.equal(got[0], base[0]) and torch.equal(got[1], base[1])
