"""Cost-model check of the All-Scan / compute overlap: predicted exposed communication
vs the exposure measured with an injected chain latency (profiles/r02_overlap_probe.jsonl,
scripts/overlap_probe.py).

* serial schedule (G = 1): the reference's own two-stream model, ``overlap_schedule``
  (glasp/engine.py:436-460), fed with the measured phase times of the fused kernels (no separate intra
  precompute exists: the output kernels are fused, so t_intra_precompute = 0) -- one timeline per
  direction;
* head-group schedule (G > 1, ZecoRank(overlap_groups=G)): the same two-stream rule generalised to the
  order local(0) local(1) out(0) local(2) out(1) ... with group j's chain on the communication stream
  between local(j) and out(j) (an event simulation; per-group kernel times = phase / G scaled to the
  measured G-group step without latency).

Writes profiles/r02_overlap_model_check.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_01004_b200.engine import overlap_schedule  # noqa: E402

bench = json.load(open(os.path.join(ROOT, "profiles", "r02s3_bench_full.json")))
ph = bench["phase_ms"]
tl = {"fwd": ph["fwd_local"] * 1e3, "bwd": ph["bwd_local"] * 1e3}
to = {"fwd": ph["fwd_output"] * 1e3, "bwd": ph["bwd_output"] * 1e3}


def simulate(G, d, scale):
    """makespan (us) of one direction: compute stream local/out per group, chains serial on the comm stream"""
    loc = [scale * tlx / G for tlx in [tl_cur] * G]
    out = [scale * to_cur / G for _ in range(G)]
    order = [("L", 0)] + [x for j in range(1, G) for x in (("L", j), ("O", j - 1))] + [("O", G - 1)]
    t = 0.0
    comm_free = 0.0
    chain_end = {}
    for kind, j in order:
        if kind == "L":
            t += loc[j]
            start = max(t, comm_free)
            chain_end[j] = comm_free = start + d
        else:
            t = max(t, chain_end[j]) + out[j]
    return t


rows = [json.loads(x) for x in open(os.path.join(ROOT, "profiles", "r02_overlap_probe.jsonl"))]
base = {r["groups"]: r["ms_per_step"] * 1e3 for r in rows if r["chain_us_per_direction"] == 0}
out_rows = []
for r in rows:
    G, d = r["groups"], r["chain_us_per_direction"]
    pred = 0.0
    for direction in ("fwd", "bwd"):
        tl_cur, to_cur = tl[direction], to[direction]
        if G == 1:
            tlv = overlap_schedule(tl_cur, d, 0.0, to_cur)
            span = max(e.end for e in tlv.events)
            pred += span - (tl_cur + to_cur)
        else:
            # per-group kernels inherit the grouping overhead measured at d = 0
            scale = base[G] / base[1]
            globals().update(tl_cur=tl_cur, to_cur=to_cur)
            pred += simulate(G, d, scale) - simulate(G, 0.0, scale)
    out_rows.append({"groups": G, "chain_us_per_direction": d, "measured_exposed_us": r["exposed_us"],
                     "predicted_exposed_us": round(pred, 2)})
res = {"phase_us": {"fwd_local": tl["fwd"], "fwd_output": to["fwd"], "bwd_local": tl["bwd"], "bwd_output": to["bwd"]},
       "model": "serial: glasp overlap_schedule(t_local, t_chain, 0, t_out) per direction; groups: two-stream event "
                "simulation of ZecoRank(overlap_groups=G)",
       "rows": out_rows}
json.dump(res, open(os.path.join(ROOT, "profiles", "r02_overlap_model_check.json"), "w"), indent=1)
for x in out_rows:
    print(x)
