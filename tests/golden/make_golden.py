"""Freeze golden vectors from the reference `glasp` implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the UNMODIFIED reference from /root/reference/pkg/src, runs its own
public API (generate_sequence, run_forward/run_backward, all_scan, the gla
functions) and writes small .npz fixtures next to this script.  The fixtures
travel with the repo; nothing at test time reads /root/reference.

bf16 cases: q, k, v, dO are rounded to bfloat16 and g to float32 *before* the
reference runs (in float64 on the rounded values), so the CUDA path and the
reference consume bit-identical inputs.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np
import torch

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).to(torch.float64).numpy()


def _bf16_bits(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def strategy_case(glasp, P, L, C, h, dk, dv, seed, K, quant, decay=None):
    from glasp import ModelDims, generate_sequence
    from glasp.cluster import NetConfig, create_cluster
    from glasp.collectives import PipelineConfig
    from glasp.engine import GlobalSequence, StrategyKind, run_backward, run_forward

    kw = {}
    if decay is not None:
        kw = {"decay_low": decay[0], "decay_high": decay[1]}
    seq = generate_sequence(P, L, C, ModelDims(h, dk, dv), seed, **kw)
    do = np.random.default_rng(seed + 1).uniform(-1.0, 1.0, (h, P * L, dv))
    q, k, v, g = seq.q, seq.k, seq.v, seq.g
    if quant == "bf16":
        q, k, v, do = _bf16(q), _bf16(k), _bf16(v), _bf16(do)
        g = _f32(g)
    seq = GlobalSequence(q=q, k=k, v=v, g=g, num_ranks=P, layout=seq.layout, dims=seq.dims)
    cluster = create_cluster(P, NetConfig())
    pipe = PipelineConfig(K)
    fwd = run_forward(seq, StrategyKind.ZECO, cluster, pipe)
    bwd = run_backward(seq, do, StrategyKind.ZECO, cluster, pipe, fwd)
    out = {
        "P": P, "L": L, "C": C, "h": h, "dk": dk, "dv": dv, "seed": seed, "K": K,
        "o": fwd.outputs,
        "dq": bwd.grads.dq, "dk_": bwd.grads.dk, "dv_": bwd.grads.dv, "dg": bwd.grads.dg,
        "prev": np.stack([s.values for s in fwd.saved.prev_states]),
        "scanned": np.stack([s.values for s in fwd.saved.final_states]),
        "g_tot": np.stack(fwd.saved.total_log_decays),
        "bounds": np.stack([np.stack([s.values for s in b]) for b in fwd.boundary_states]),
        "sent_per_rank": np.array([bwd.ledger.sent(rank=r) for r in range(P)]),
    }
    if quant == "bf16":
        out.update(q_bits=_bf16_bits(q), k_bits=_bf16_bits(k), v_bits=_bf16_bits(v),
                   do_bits=_bf16_bits(do), g=g.astype(np.float32))
        # outputs stored as float32 to keep fixtures small (errors ~1e-7 << bf16 tolerance)
        for key in ("o", "dq", "dk_", "dv_", "dg", "bounds"):
            out[key] = out[key].astype(np.float32)
    else:
        out.update(q=q, k=k, v=v, g=g, do=do)
    return out


def gla_function_case(glasp, seed):
    """Single-shard function-level vectors: local scan, outputs, reverse scan, backward."""
    from glasp.gla import (ModelDims, SeqShard, ShardLayout, State, backward, forward_outputs,
                           global_correct, local_state_scan, recurrent_forward, reverse_boundary_scan,
                           revcum)
    rng = np.random.default_rng(seed)
    h, L, C, dk, dv = 2, 48, 16, 5, 3
    q = rng.uniform(-1, 1, (h, L, dk))
    k = rng.uniform(-1, 1, (h, L, dk))
    v = rng.uniform(-1, 1, (h, L, dv))
    g = rng.uniform(math.log(0.5), math.log(0.99), (h, L, dk))
    do = rng.uniform(-1, 1, (h, L, dv))
    prev = rng.uniform(-1, 1, (h, dk, dv))
    ds_next = rng.uniform(-1, 1, (h, dk, dv))
    shard = SeqShard(q=q, k=k, v=v, g=g, layout=ShardLayout(L, C), dims=ModelDims(h, dk, dv))
    states, cum = local_state_scan(shard)
    o = forward_outputs(shard, states, cum, State(prev))
    corr = global_correct(states, cum, State(prev))
    rev = reverse_boundary_scan(shard, do)
    grads, dsb = backward(shard, do, State(prev), State(ds_next))
    rec_o, rec_b, _ = recurrent_forward(shard, init=State(prev))
    return {
        "h": h, "L": L, "C": C, "dk": dk, "dv": dv,
        "q": q, "k": k, "v": v, "g": g, "do": do, "prev": prev, "ds_next": ds_next,
        "states": np.stack([s.values for s in states], axis=1),
        "cum": np.stack([c.log_values for c in cum], axis=1),
        "o": o, "corrected": np.stack([s.values for s in corr], axis=1),
        "rev": np.stack([s.values for s in rev], axis=1),
        "dq": grads.dq, "dk_": grads.dk, "dv_": grads.dv, "dg": grads.dg,
        "ds_boundary": dsb.values, "rec_o": rec_o,
        "rec_bounds": np.stack([s.values for s in rec_b], axis=1),
        "revcum_in": q[0], "revcum_out": revcum(q)[0],
    }


def allscan_case(glasp, P, h, dk, dv, seed, K, precision):
    from glasp.cluster import NetConfig, create_cluster
    from glasp.collectives import PipelineConfig, ScanDirection, all_scan
    from glasp.gla import CumDecay, State
    rng = np.random.default_rng(seed)
    dt = np.float64 if precision == "f64" else np.float32
    states = [State(rng.uniform(-1, 1, (h, dk, dv)).astype(dt)) for _ in range(P)]
    cds = [CumDecay(rng.uniform(-2.0, 0.0, (h, dk)).astype(dt)) for _ in range(P)]
    out = {"P": P, "K": K, "local": np.stack([s.values for s in states]),
           "logdecay": np.stack([c.log_values for c in cds])}
    for direction in (ScanDirection.FWD, ScanDirection.BWD):
        cl = create_cluster(P, NetConfig())
        recv, scanned = all_scan(cl, states, cds, PipelineConfig(K), direction)
        tag = direction.value
        out[f"recv_{tag}"] = np.stack([r.values for r in recv])
        out[f"scanned_{tag}"] = np.stack([s.values for s in scanned])
        out[f"sent_{tag}"] = np.array([cl.read_ledger().sent(rank=r) for r in range(P)])
    return out


def main():
    sys.path.insert(0, REF)
    import glasp  # noqa: F401  (the reference, unmodified)

    cases = {
        # small f64 strategy case (reference defaults for gates)
        "zeco_f64_p4": strategy_case(glasp, P=4, L=32, C=8, h=2, dk=4, dv=4, seed=10, K=2, quant=None),
        # bf16 cases at the fast-path head dims
        "zeco_bf16_d64_p2": strategy_case(glasp, P=2, L=128, C=64, h=2, dk=64, dv=64, seed=3, K=4,
                                          quant="bf16"),
        "zeco_bf16_d128_p2_long": strategy_case(glasp, P=2, L=256, C=64, h=1, dk=128, dv=128, seed=5,
                                                K=4, quant="bf16",
                                                decay=(math.log(0.9999), math.log(0.99999))),
        "gla_functions": gla_function_case(glasp, seed=7),
        "allscan_f64_p5": allscan_case(glasp, P=5, h=2, dk=8, dv=3, seed=1, K=2, precision="f64"),
        "allscan_f32_p8": allscan_case(glasp, P=8, h=2, dk=16, dv=8, seed=2, K=4, precision="f32"),
    }
    for name, data in cases.items():
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
