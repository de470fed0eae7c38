"""Cost model: closed forms equal the reference's; the (alpha, beta) fit recovers
known parameters and calibrates against the committed All-Scan measurements."""

import math
import os
import sys

import pytest

from paper_2507_01004_b200 import costmodel as cm
from paper_2507_01004_b200.cluster import NetConfig
from paper_2507_01004_b200.errors import ConfigError
from paper_2507_01004_b200.gla import ModelDims

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _p(P=8, K=16, net=NetConfig(1e-6, 1e9, 4)):
    return cm.CostParams(net=net, dims=ModelDims(16, 128, 128), num_ranks=P, pipeline_blocks=K,
                         chunks_per_rank=256, tokens_per_rank=16384)


def test_eq13_known_values():
    net = NetConfig(0.0, 1e9, 4)
    S = 16 * 128 * 128
    assert cm.t_allscan(_p(8, 16, net)) == pytest.approx((16 + 7) * S / 16 / 1e9)
    assert cm.t_allscan(_p(1, 16, net)) == 0.0
    with pytest.raises(ConfigError):
        cm.t_allscan(_p(8, 3, net))
    r = cm.t_strategies(_p(4, 1, net), t_ideal=1.0, t_overlap=0.25)
    ts = S / 1e9
    assert (r.t_zeco, r.t_lasp1, r.t_lasp2) == pytest.approx((0.75 + ts, 4 * (1 + ts), 1 + 4 * ts))
    with pytest.raises(ConfigError):
        cm.t_strategies(_p(), 1.0, 2.0)


def test_fit_recovers_alpha_beta():
    net = NetConfig(2.5e-6, 3e10, 4)
    samples = [cm.Sample(P, K, S, (K + P - 1) * net.tau(S / K))
               for P in (2, 4, 8) for K in (1, 4, 16) for S in (16384, 262144, 1048576)]
    fit = cm.fit_net(samples)
    assert fit.latency_alpha == pytest.approx(2.5e-6, rel=1e-9)
    assert fit.bandwidth_beta == pytest.approx(3e10, rel=1e-9)
    rep = cm.calibration_report(samples)
    assert rep["ratio_min"] == pytest.approx(1.0) and rep["ratio_max"] == pytest.approx(1.0)


def test_calibration_on_committed_measurements():
    path = os.path.join(ROOT, "profiles", "r01_allscan_virtual.jsonl")
    samples = cm.samples_from_bench(open(path))
    assert len(samples) >= 10
    rep = cm.calibration_report(samples)
    assert rep["alpha_us"] > 0 and rep["beta_GBps"] > 0
    assert 0.2 < rep["ratio_geomean"] < 5.0


@pytest.mark.reference
def test_closed_forms_match_reference():
    sys.path.insert(0, "/root/reference/pkg/src")
    from glasp import costmodel as ref
    from glasp.cluster import NetConfig as RefNet
    from glasp.gla import ModelDims
    for P, K in ((1, 1), (2, 4), (8, 16)):
        ours = _p(P, K, NetConfig(1.5e-6, 2e9, 4))
        theirs = ref.CostParams(net=RefNet(1.5e-6, 2e9, 4), dims=ModelDims(16, 128, 128), num_ranks=P,
                                pipeline_blocks=K, chunks_per_rank=256, tokens_per_rank=16384)
        assert cm.t_allscan(ours) == ref.t_allscan(theirs)
        a, b = cm.t_strategies(ours, 2.0, 0.5), ref.t_strategies(theirs, 2.0, 0.5)
        assert (a.t_zeco, a.t_lasp1, a.t_lasp2) == (b.t_zeco, b.t_lasp1, b.t_lasp2)
        for m in cm.METHODS:
            assert cm.volume_compute_table(m, ours) == ref.volume_compute_table(m, theirs)
        assert [{k: r[k] for k in cm.TABLE_COLUMNS} for r in cm.table_rows(ours)] == ref.table_rows(theirs)
        assert all(cm.table_note(m) == ref.table_note(m) for m in cm.METHODS)
    assert cm.SIMULATED_METHODS == ref.SIMULATED_METHODS and cm.TABLE_COLUMNS == ref.TABLE_COLUMNS
