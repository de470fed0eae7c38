"""GPU runs of the drop-in exported with export_artifacts, diffed against the reference's own export for the
same configuration (tests/golden/export, frozen by tests/golden/make_export_golden.py from the unmodified
glasp): ledger.csv and timeline.json byte for byte (same virtual schedule), the .zgla tensors within the
float64 tolerance of the reference's own tests (1e-10)."""

import os
import sys

import numpy as np
import pytest

from tests.helpers import rel

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_export_golden import CONFIG, STRATEGIES  # noqa: E402

GOLDEN = os.path.join(HERE, "golden", "export")


@pytest.mark.parametrize("strategy", STRATEGIES)
def test_export_matches_reference(tmp_path, strategy):
    import paper_2507_01004_b200 as z

    c = CONFIG
    seq = z.generate_sequence(c["P"], c["L"], c["C"], z.ModelDims(*c["dims"]), c["seed"])
    do = np.random.default_rng(c["seed"] + 1).uniform(-1, 1, (c["dims"][0], c["P"] * c["L"], c["dims"][2]))
    st = z.StrategyKind(strategy)
    P = 1 if st is z.StrategyKind.SINGLE_DEVICE else c["P"]
    net = z.NetConfig(latency_alpha=c["alpha"], bandwidth_beta=c["beta"])
    costs = z.ComputeCosts(per_chunk=c["per_chunk"], per_state=c["per_state"])
    pipe = z.PipelineConfig(c["K"])
    fwd = z.run_forward(seq, st, z.create_cluster(P, net), pipe, costs)
    bwd = z.run_backward(seq, do, st, z.create_cluster(P, net), pipe, fwd, costs)
    for tag, art in (("fwd", fwd), ("bwd", bwd)):
        out = tmp_path / tag
        written = z.export_artifacts(art, out)
        want_dir = os.path.join(GOLDEN, strategy, tag)
        assert sorted(p.name for p in written) == sorted(os.listdir(want_dir))
        for name in ("ledger.csv", "timeline.json"):
            assert (out / name).read_bytes() == open(os.path.join(want_dir, name), "rb").read(), name
        for name in sorted(os.listdir(want_dir)):
            if name.endswith(".zgla"):
                got, want = z.read_tensor(out / name), z.read_tensor(os.path.join(want_dir, name))
                assert got.shape == want.shape and rel(got, want) <= 1e-10, name
    assert fwd.measured_timeline is not None and len(fwd.measured_timeline.events) > 0
