"""Parity of the fused tcgen05 ZeCO path (bf16, D=128) against the CPU oracle and the
reference golden vectors.  Tolerance: north-star rtol 1e-2 (relative Frobenius) for bf16."""

import math

import numpy as np
import pytest
import torch

from oracle import gla_oracle as orc
from tests.helpers import TOL_BF16, bf16_bits_to_f64, rel

pytestmark = pytest.mark.gpu


def bf16_round(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).to(torch.float64).numpy()


def make_case(h, P, L, seed, long_memory=False, D=128):
    lo, hi = (orc.LONG_DECAY_LOW, orc.LONG_DECAY_HIGH) if long_memory else (orc.DECAY_LOW, orc.DECAY_HIGH)
    q, k, v, g = orc.make_inputs(P, L, h, D, D, seed, lo, hi)
    do = orc.make_cotangent(seed, h, P * L, D)
    q, k, v, do = (bf16_round(x) for x in (q, k, v, do))
    g = g.astype(np.float32).astype(np.float64)
    return q, k, v, g, do


def run_fast(q, k, v, g, do, P, sms=None, K=4):
    """Per-rank ZeCO entry points on the device + the list-form All-Scan kernel."""
    from paper_2507_01004_b200 import ops

    h, T, D = q.shape
    L = T // P
    dev = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)  # noqa: E731
    Q, Kt, V, G, DO = (dev(q, torch.bfloat16), dev(k, torch.bfloat16), dev(v, torch.bfloat16), dev(g, torch.float32),
                       dev(do, torch.bfloat16))
    sl = [slice(p * L, (p + 1) * L) for p in range(P)]
    part = lambda X, p: X[:, sl[p]].contiguous()  # noqa: E731
    shards = [ops.ZecoShard(h, L, D, D, 64, torch.bfloat16, sms=sms) for _ in range(P)]
    assert all(s.fast for s in shards)
    loc = [shards[p].fwd_local(part(Kt, p), part(V, p), part(G, p)) for p in range(P)]
    S_loc = torch.stack([x[0] for x in loc])
    G_tot = torch.stack([x[1] for x in loc])
    recv, scanned = ops.allscan_local(S_loc, G_tot, K, 0)
    o = torch.cat([shards[p].fwd_output(part(Q, p), part(Kt, p), part(V, p), part(G, p), recv[p] if p else None)
                   for p in range(P)], 1)
    d0 = torch.stack([shards[p].bwd_local(part(Q, p), part(G, p), part(DO, p)) for p in range(P)])
    ds_next, _ = ops.allscan_local(d0, G_tot, K, 1)
    grads = [shards[p].bwd_output(part(Q, p), part(Kt, p), part(V, p), part(G, p), part(DO, p),
                                  recv[p] if p else None, ds_next[p] if p < P - 1 else None) for p in range(P)]
    cat = lambda i: torch.cat([gr[i] for gr in grads], 1).double().cpu().numpy()  # noqa: E731
    torch.cuda.synchronize()
    return {"o": o.double().cpu().numpy(), "dq": cat(0), "dk": cat(1), "dv": cat(2), "dg": cat(3),
            "prev": recv.double().cpu().numpy(), "scanned": scanned.double().cpu().numpy(),
            "s_local": S_loc.double().cpu().numpy(), "d0": d0.double().cpu().numpy()}


def oracle(q, k, v, g, do, P, C=64):
    o, saved, _ = orc.zeco_forward(q, k, v, g, P, C)
    (dq, dk, dv, dg), ds_next = orc.zeco_backward(q, k, v, g, do, P, C, saved)
    return {"o": o, "dq": dq, "dk": dk, "dv": dv, "dg": dg, "prev": np.stack(saved["prev"]),
            "scanned": np.stack(saved["scanned"])}


def check(got, want, tol=TOL_BF16, keys=("o", "dq", "dk", "dv", "dg")):
    errs = {kk: rel(got[kk], want[kk]) for kk in keys}
    bad = {kk: e for kk, e in errs.items() if not e <= tol}
    print("rel errors", {kk: f"{e:.2e}" for kk, e in errs.items()})
    assert not bad, f"rel errors {errs}"
    return errs


def test_fast_golden_long_memory(golden):
    """Reference run (glasp ZeCO, P=2, long-memory gates) on bit-identical bf16 inputs."""
    c = golden("zeco_bf16_d128_p2_long")
    q, k, v, do = (bf16_bits_to_f64(c[f"{n}_bits"]) for n in ("q", "k", "v", "do"))
    g = c["g"].astype(np.float64)
    got = run_fast(q, k, v, g, do, int(c["P"]), K=int(c["K"]))
    want = {"o": c["o"], "dq": c["dq"], "dk": c["dk_"], "dv": c["dv_"], "dg": c["dg"], "prev": c["prev"],
            "scanned": c["scanned"]}
    check(got, want)
    assert rel(got["prev"], want["prev"]) <= TOL_BF16
    assert rel(got["scanned"], want["scanned"]) <= TOL_BF16


@pytest.mark.parametrize("P,L,h,long_memory,sms", [
    (1, 2048, 2, False, None),
    (1, 2048, 2, True, None),
    (2, 1024, 2, True, None),
    (1, 1024, 1, True, 1),       # one segment: a single CTA walks all 16 tiles
    (2, 512, 3, False, 4),       # ragged segment split (8 tiles over 1 segment / head)
    (4, 256, 2, True, 148),      # 4 ranks, every tile its own segment
])
def test_fast_matches_oracle(P, L, h, long_memory, sms):
    q, k, v, g, do = make_case(h, P, L, seed=100 + P + L + h, long_memory=long_memory)
    got = run_fast(q, k, v, g, do, P, sms=sms)
    want = oracle(q, k, v, g, do, P)
    check(got, want)
    assert rel(got["prev"], want["prev"]) <= TOL_BF16


def test_fast_segmentation_invariance():
    """Results do not depend on how a head is cut into segments (nseg = 1 vs one per tile)."""
    q, k, v, g, do = make_case(1, 1, 1024, seed=7, long_memory=True)
    a = run_fast(q, k, v, g, do, 1, sms=1)
    b = run_fast(q, k, v, g, do, 1, sms=16)
    for key in ("o", "dq", "dk", "dv", "dg"):
        assert rel(a[key], b[key]) <= 5e-3, key


def test_fast_cfg2_heads_against_oracle():
    """BASELINE config 2 shape (H=16, d=128, 16K tokens, 1 GPU); heads 0 and 15 checked in f64."""
    h, L = 16, 16384
    q, k, v, g, do = make_case(h, 1, L, seed=2)
    got = run_fast(q, k, v, g, do, 1)
    for hh in (0, h - 1):
        sl = slice(hh, hh + 1)
        want = oracle(q[sl], k[sl], v[sl], g[sl], do[sl], 1)
        check({kk: got[kk][sl] for kk in ("o", "dq", "dk", "dv", "dg")}, want)


def test_fast_zero_cotangent_gives_zero_grads():
    q, k, v, g, do = make_case(2, 2, 256, seed=3)
    got = run_fast(q, k, v, g, np.zeros_like(do), 2)
    for key in ("dq", "dk", "dv", "dg"):
        assert np.all(got[key] == 0.0), key


@pytest.mark.parametrize("h,L", [(160, 128), (37, 192)])
def test_fast_more_heads_than_sms(h, L):
    """h > #SMs: one segment per head, more than one CTA wave; odd head count / tile count."""
    q, k, v, g, do = make_case(h, 1, L, seed=11, long_memory=True)
    got = run_fast(q, k, v, g, do, 1)
    for hh in (0, h // 2, h - 1):
        sl = slice(hh, hh + 1)
        want = oracle(q[sl], k[sl], v[sl], g[sl], do[sl], 1)
        check({kk: got[kk][sl] for kk in ("o", "dq", "dk", "dv", "dg")}, want)


def test_fast_deterministic_and_linear_in_v_at_cfg2():
    """Full BASELINE config-2 size: bitwise-deterministic reruns, and o / dq linear in v (fp32-accumulated
    bf16 path: o(v1) + o(v2) vs o(v1 + v2) within the bf16 tolerance)."""
    from paper_2507_01004_b200 import ops
    torch.manual_seed(0)
    h, L, D = 16, 16384, 128
    sh = ops.ZecoShard(h, L, D, D, 64, torch.bfloat16)
    q, k, v1, v2 = ((torch.rand(h, L, D, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(4))
    g = torch.rand(h, L, D, device="cuda") * (math.log(0.999) - math.log(0.9)) + math.log(0.9)

    def fwd(v):
        sh.fwd_local(k, v, g)
        return sh.fwd_output(q, k, v, g).float()
    a1, a2 = fwd(v1), fwd(v1)
    assert torch.equal(a1, a2)
    s = fwd((v1.float() + v2.float()).to(torch.bfloat16))
    lin = a1 + fwd(v2)
    err = ((s - lin).norm() / lin.norm()).item()
    assert err <= TOL_BF16, err


def test_fast_causality_bitwise_at_cfg2():
    """Full BASELINE config-2 size, exact (bitwise) causality of the segment-parallel kernels.
    Forward: changing k / v of token t leaves o[:t] and every other head bit-identical.
    Backward: changing dO of token t leaves dq everywhere but at t, dk / dv after t and dg after t's
    64-token tile bit-identical (dq_i needs dO_i only; dk_j, dv_j, dg_j need dO_i for i >= j)."""
    from paper_2507_01004_b200 import ops
    torch.manual_seed(5)
    h, L, D, hp = 16, 16384, 128, 5
    t = 9 * 1024 + 64 * 7 + 17  # inside a tile, inside a segment (not a boundary)
    sh = ops.ZecoShard(h, L, D, D, 64, torch.bfloat16)
    q, k, v, do = ((torch.rand(h, L, D, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(4))
    g = torch.rand(h, L, D, device="cuda") * (math.log(0.999) - math.log(0.9)) + math.log(0.9)

    def step(k, v, do):
        sh.fwd_local(k, v, g)
        o = sh.fwd_output(q, k, v, g).clone()
        sh.bwd_local(q, g, do)
        return o, [x.clone() for x in sh.bwd_output(q, k, v, g, do, None, None)]

    o0, (dq0, dk0, dv0, dg0) = step(k, v, do)
    k1, v1 = k.clone(), v.clone()
    k1[hp, t] = -k1[hp, t]
    v1[hp, t] = v1[hp, t] * 2 + 0.5
    o1, _ = step(k1, v1, do)
    others = [x for x in range(h) if x != hp]
    assert torch.equal(o1[others], o0[others])
    assert torch.equal(o1[hp, :t], o0[hp, :t])
    assert not torch.equal(o1[hp, t:], o0[hp, t:])

    do1 = do.clone()
    do1[hp, t] = -do1[hp, t] + 0.25
    _, (dq1, dk1, dv1, dg1) = step(k, v, do1)
    for a, b in ((dq1, dq0), (dk1, dk0), (dv1, dv0), (dg1, dg0)):
        assert torch.equal(a[others], b[others])
    assert torch.equal(dq1[hp, :t], dq0[hp, :t]) and torch.equal(dq1[hp, t + 1:], dq0[hp, t + 1:])
    for a, b in ((dk1, dk0), (dv1, dv0), (dg1, dg0)):
        assert not torch.equal(a[hp, :t + 1], b[hp, :t + 1])
    for a, b in ((dk1, dk0), (dv1, dv0)):
        assert torch.equal(a[hp, t + 1:], b[hp, t + 1:])
    # dg inside a tile is the tile's suffix sum taken as (tile total - prefix): bit-identical from the
    # next tile on, equal up to fp32 rounding between t and the end of its tile
    te = (t // 64 + 1) * 64
    assert torch.equal(dg1[hp, te:], dg0[hp, te:])
    torch.testing.assert_close(dg1[hp, t + 1:te], dg0[hp, t + 1:te], rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("lo,hi", [(math.log(0.5), math.log(0.9)), (math.log(0.2), math.log(0.5))])
def test_fast_strong_decay_inside_domain(lo, hi):
    """Strong gates (per-token decay down to 0.2: 64-token tile log-decay down to about -103, in-tile
    exponents up to ~52) stay inside the fast path's overflow-free domain (tile log-decay > -170)."""
    h, P, L = 2, 2, 512
    q, k, v, g = orc.make_inputs(P, L, h, 128, 128, 5, lo, hi)
    do = orc.make_cotangent(5, h, P * L, 128)
    q, k, v, do = (bf16_round(x) for x in (q, k, v, do))
    g = g.astype(np.float32).astype(np.float64)
    got = run_fast(q, k, v, g, do, P)
    for key in ("o", "dq", "dk", "dv", "dg"):
        assert np.all(np.isfinite(got[key])), key
    check(got, oracle(q, k, v, g, do, P))


@pytest.mark.parametrize("D", [128, 64])
def test_fast_strided_views_bitwise(D):
    """zgla_tensor strides: q/k/v/g/dO as head slices of token-major buffers and o/dq/dk/dv/dg written
    into token-major buffers give bitwise the same results as dense [h, L, d] tensors."""
    from paper_2507_01004_b200 import ops
    torch.manual_seed(3)
    h, L = 3, 1024
    dense = [(torch.rand(h, L, D, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(3)]
    g = torch.rand(h, L, D, device="cuda") * (math.log(0.999) - math.log(0.9)) + math.log(0.9)
    do = (torch.rand(h, L, D, device="cuda") * 2 - 1).to(torch.bfloat16)

    def token_major(x, pad=0):  # [L, h * D + pad] storage, [h, L, D] view
        buf = torch.zeros(L, h * D + pad, dtype=x.dtype, device="cuda")
        view = buf[:, :h * D].view(L, h, D).transpose(0, 1)
        view.copy_(x)
        return view

    def run(q, k, v, g, do, outs):
        sh = ops.ZecoShard(h, L, D, D, 64, torch.bfloat16)
        sh.fwd_local(k, v, g)
        o = sh.fwd_output(q, k, v, g, out=outs[0])
        sh.bwd_local(q, g, do)
        grads = sh.bwd_output(q, k, v, g, do, grads=outs[1:])
        torch.cuda.synchronize()
        return [o] + list(grads)

    outs_d = [torch.empty(h, L, D, dtype=torch.bfloat16, device="cuda") for _ in range(4)] + \
             [torch.empty(h, L, D, device="cuda")]
    a = run(*dense, g, do, outs_d)
    strided_in = [token_major(x, pad=64) for x in dense] + [token_major(g, pad=32), token_major(do)]
    outs_s = [token_major(torch.empty(h, L, D, dtype=torch.bfloat16, device="cuda")) for _ in range(4)] + \
             [token_major(torch.empty(h, L, D, device="cuda"), pad=16)]
    b = run(*strided_in, outs_s)
    for name, x, y in zip(("o", "dq", "dk", "dv", "dg"), a, b):
        assert y.stride(2) == 1 and y.stride(0) != L * D  # really strided
        assert torch.equal(x, y), name


@pytest.mark.parametrize("P,L,h,long_memory", [(1, 1024, 2, False), (2, 512, 4, True), (4, 256, 3, True)])
def test_fast_d64_heads_against_oracle(P, L, h, long_memory):
    """d_k = d_v = 64 (the paper's GLA-1B heads, BASELINE config 1) on the fused path: the 128-channel
    kernels see the missing channels as TMA zero-fill; guarded stores write only the 64 real ones."""
    q, k, v, g, do = make_case(h, P, L, seed=200 + P + h, long_memory=long_memory, D=64)
    got = run_fast(q, k, v, g, do, P)
    want = oracle(q, k, v, g, do, P)
    check(got, want)
    assert rel(got["prev"], want["prev"]) <= TOL_BF16


def test_fast_domain_flag():
    """A tile whose summed log-decay is below -160 (per-token decay < ~0.08) is outside the fused path's
    exponent domain: check_domain() raises DomainError; gates inside the domain pass."""
    from paper_2507_01004_b200 import ops
    from paper_2507_01004_b200.errors import DomainError
    h, L, D = 2, 512, 128
    sh = ops.ZecoShard(h, L, D, D, 64, torch.bfloat16)
    k, v = ((torch.rand(h, L, D, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(2))
    g = torch.full((h, L, D), math.log(0.5), device="cuda")  # tile total 64 * -0.69 = -44: fine
    sh.fwd_local(k, v, g)
    sh.check_domain()
    g[1, 200, 7] = -200.0  # one strong gate makes its tile leave the domain
    sh.fwd_local(k, v, g)
    with pytest.raises(DomainError):
        sh.check_domain()
    g[1, 200, 7] = math.log(0.5)
    sh.fwd_local(k, v, g)  # the flag is per call
    sh.check_domain()


@pytest.mark.parametrize("long_memory", [False, True])
def test_fast_cfg1_full_size_seeds(long_memory):
    """BASELINE config 1 at its stated size on the fused path: H=4, d=64, P=2 ranks x 2,048 tokens, K=4,
    seeds 0..9, every output and gradient and the forward boundary states against the f64 oracle."""
    worst = {}
    for seed in range(10):
        q, k, v, g, do = make_case(4, 2, 2048, seed=seed, long_memory=long_memory, D=64)
        got = run_fast(q, k, v, g, do, 2, K=4)
        want = oracle(q, k, v, g, do, 2)
        errs = check(got, want)
        errs["prev"] = rel(got["prev"], want["prev"])
        assert errs["prev"] <= TOL_BF16
        for kk, e in errs.items():
            worst[kk] = max(worst.get(kk, 0.0), e)
    print("cfg1 worst rel errors", {kk: f"{e:.2e}" for kk, e in worst.items()})


@pytest.mark.parametrize("long_memory", [False, True])
def test_fast_cfg2_more_heads_both_gates(long_memory):
    """BASELINE config 2 (H=16, d=128, 16K tokens, 1 GPU): heads 0, 5, 10, 15 against the f64 oracle under
    both gate distributions (the default and the long-memory one)."""
    h, L = 16, 16384
    q, k, v, g, do = make_case(h, 1, L, seed=21 + long_memory, long_memory=long_memory)
    got = run_fast(q, k, v, g, do, 1)
    for hh in (0, 5, 10, 15):
        sl = slice(hh, hh + 1)
        want = oracle(q[sl], k[sl], v[sl], g[sl], do[sl], 1)
        check({kk: got[kk][sl] for kk in ("o", "dq", "dk", "dv", "dg")}, want)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_chunk_scalings_against_oracle(dtype):
    """glasp/gla.py:233-245 chunk_scalings on the device: the reference's hand values (tests/test_gla.py:89-94)
    and random chunks against the oracle; Lambda * Gamma = gamma."""
    from paper_2507_01004_b200 import chunk_scalings
    cs = chunk_scalings(np.log(np.array([[[0.5], [0.5]]], dtype=dtype)))
    np.testing.assert_allclose(cs.chunk_decay, [[0.25]], rtol=1e-7)
    np.testing.assert_allclose(cs.decay_from_start[0, :, 0], [0.5, 0.25], rtol=1e-7)
    np.testing.assert_allclose(cs.decay_to_end[0, :, 0], [0.5, 1.0], rtol=1e-7)
    rng = np.random.default_rng(4)
    gch = rng.uniform(orc.DECAY_LOW, orc.DECAY_HIGH, (3, 64, 128)).astype(dtype)
    cs = chunk_scalings(gch)
    want = orc.chunk_scalings(gch.astype(np.float64))
    tol = 1e-13 if dtype == np.float64 else 1e-6
    for got, w in zip((cs.chunk_decay, cs.decay_from_start, cs.decay_to_end), want):
        assert got.dtype == dtype and rel(got, w) <= tol
    np.testing.assert_allclose(cs.decay_from_start * cs.decay_to_end,
                               np.broadcast_to(cs.chunk_decay[:, None, :], gch.shape), rtol=1e-5 if dtype == np.float32 else 1e-14)


def _shard_step(q, k, v, g, do, dtype):
    """one P = 1 fwd + bwd through the per-rank entry points in `dtype` (bf16: fused tcgen05 kernels;
    fp32: the SIMT kernels with the exact token recurrence inside each chunk)"""
    from paper_2507_01004_b200 import ops
    h, L, D = q.shape
    sh = ops.ZecoShard(h, L, D, D, 64, dtype)
    assert sh.fast == (dtype == torch.bfloat16)
    Q, K_, V, DO = (x.to(dtype) for x in (q, k, v, do))
    sh.fwd_local(K_, V, g)
    o = sh.fwd_output(Q, K_, V, g, None)
    sh.bwd_local(Q, g, DO)
    grads = sh.bwd_output(Q, K_, V, g, DO, None, None)
    torch.cuda.synchronize()
    return [o.double().cpu().numpy()] + [x.double().cpu().numpy() for x in grads]


def test_fast_single_tile_shard():
    """L = 64: one tile, one segment per head (the smallest shard the fused path takes)"""
    q, k, v, g, do = make_case(3, 1, 64, seed=5, long_memory=True)
    got = run_fast(q, k, v, g, do, 1)
    check(got, oracle(q, k, v, g, do, 1))


def test_fast_long_shard_against_fp32_kernels():
    """BASELINE config 5's per-GPU length (131,072 tokens, 2,048 tiles per head, 228-tile segments): the fused
    bf16 path against the fp32 SIMT path on the same (bf16-rounded) inputs, both gate distributions"""
    h, L, D = 2, 131072, 128
    gen = torch.Generator(device="cuda").manual_seed(17)
    u = lambda lo, hi: torch.rand((h, L, D), device="cuda", generator=gen) * (hi - lo) + lo  # noqa: E731
    q, k, v, do = (u(-1, 1).to(torch.bfloat16).float() for _ in range(4))
    for lo, hi in ((orc.DECAY_LOW, orc.DECAY_HIGH), (orc.LONG_DECAY_LOW, orc.LONG_DECAY_HIGH)):
        g = u(lo, hi).float()
        a = _shard_step(q, k, v, g, do, torch.bfloat16)
        b = _shard_step(q, k, v, g, do, torch.float32)
        errs = {name: rel(x, y) for name, x, y in zip(("o", "dq", "dk", "dv", "dg"), a, b)}
        print("long shard rel errors", {n: f"{e:.2e}" for n, e in errs.items()})
        assert all(e <= TOL_BF16 for e in errs.values()), errs


@pytest.mark.parametrize("sms,h,D", [(1, 1, 128), (4, 1, 128), (1, 2, 64), (2, 3, 64)])
def test_fast_dg_long_segments_default_gates(sms, h, D):
    """dg = suffix sum of da: without re-seeding, the bf16 error of da accumulates along a segment (one
    256-tile segment: 2.7e-2 relative before the re-seed, over the 1e-2 bound).  The backward re-seeds the
    running sum every ZGLA_RHO_RESEED tiles from rowsum(S' (.) Dt), so the error no longer grows with the
    segment length (one head, 16K tokens, strongly decaying reference gates)"""
    q, k, v, g, do = make_case(h, 1, 16384, seed=5, D=D)  # d = 64: head pairs (h even) / zero-filled (h odd)
    got = run_fast(q, k, v, g, do, 1, sms=sms)
    errs = check(got, oracle(q, k, v, g, do, 1))
    assert errs["dg"] <= 7e-3, errs


def test_fast_forward_only_skips_saved_states():
    """fwd_output(save_states=False) (inference): the same outputs bit for bit, and a backward after it raises
    StateError instead of reading chunk states that were never written"""
    from paper_2507_01004_b200 import ops
    from paper_2507_01004_b200.errors import StateError
    q, k, v, g, do = make_case(4, 1, 2048, seed=9)
    dev = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)  # noqa: E731
    Q, K_, V, DO = (dev(x, torch.bfloat16) for x in (q, k, v, do))
    G = dev(g, torch.float32)
    sh = ops.ZecoShard(4, 2048, 128, 128, 64, torch.bfloat16)
    sh.fwd_local(K_, V, G)
    a = sh.fwd_output(Q, K_, V, G, None).clone()
    sh.fwd_local(K_, V, G)
    b = sh.fwd_output(Q, K_, V, G, None, save_states=False)
    assert torch.equal(a, b)
    sh.bwd_local(Q, G, DO)
    with pytest.raises(StateError):
        sh.bwd_output(Q, K_, V, G, DO, None, None)
