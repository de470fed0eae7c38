"""Freeze the reference's exported artifacts (glasp/reports.py:66-87 export_artifacts) for a small run of
every strategy, so a GPU run of the drop-in can be diffed against them file by file.

Run in the build container (where /root/reference exists):

    python tests/golden/make_export_golden.py

It imports the UNMODIFIED reference from /root/reference/pkg/src and writes
tests/golden/export/<strategy>/{fwd,bwd}/{outputs,dq,dk,dv,dg}.zgla, ledger.csv, timeline.json.
The configuration (ALL below) is shared with tests/test_gpu_artifacts.py.
"""

from __future__ import annotations

import os
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "export")

# P, tokens/rank, chunk, (h, dk, dv), seed, K, alpha, beta (elements/s), per_chunk, per_state
CONFIG = dict(P=4, L=16, C=4, dims=(2, 4, 4), seed=5, K=2, alpha=2e-6, beta=5e8, per_chunk=3e-6, per_state=1e-6)
STRATEGIES = ("zeco", "lasp1", "lasp2", "single")


def run(glasp, strategy, outdir):
    from glasp.cluster import NetConfig, create_cluster
    from glasp.collectives import PipelineConfig
    from glasp.engine import ComputeCosts, StrategyKind, run_backward, run_forward
    from glasp.gla import ModelDims
    from glasp.instances import generate_sequence
    from glasp.reports import export_artifacts

    c = CONFIG
    seq = generate_sequence(c["P"], c["L"], c["C"], ModelDims(*c["dims"]), c["seed"])
    do = np.random.default_rng(c["seed"] + 1).uniform(-1, 1, (c["dims"][0], c["P"] * c["L"], c["dims"][2]))
    st = StrategyKind(strategy)
    P = 1 if st is StrategyKind.SINGLE_DEVICE else c["P"]
    net = NetConfig(latency_alpha=c["alpha"], bandwidth_beta=c["beta"])
    costs = ComputeCosts(per_chunk=c["per_chunk"], per_state=c["per_state"])
    pipe = PipelineConfig(c["K"])
    fwd = run_forward(seq, st, create_cluster(P, net), pipe, costs)
    bwd = run_backward(seq, do, st, create_cluster(P, net), pipe, fwd, costs)
    export_artifacts(fwd, os.path.join(outdir, "fwd"))
    export_artifacts(bwd, os.path.join(outdir, "bwd"))


def main():
    sys.path.insert(0, REF)
    import glasp

    assert glasp.__file__.startswith(REF), glasp.__file__
    shutil.rmtree(OUT, ignore_errors=True)
    for s in STRATEGIES:
        run(glasp, s, os.path.join(OUT, s))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
