"""Host-side logic of the drop-in that needs no GPU: containers, validation and the
exception contract (reference tests/test_gla.py, test_engine.py, test_collectives.py)."""

import math

import numpy as np
import pytest

from paper_2507_01004_b200 import (ConfigError, CumDecay, DimsError, DomainError, GlobalSequence, LayoutError,
                                   ModelDims, PipelineConfig, SeqShard, ShardLayout, State, StrategyKind,
                                   create_cluster, overlap_schedule, split)
from paper_2507_01004_b200.cluster import LedgerRow, NetConfig, VolumeLedger
from paper_2507_01004_b200.engine import ideal_makespan


def test_model_dims_validation():
    with pytest.raises(DimsError):
        ModelDims(0, 1, 1)
    assert ModelDims(2, 3, 4).state_elements == 24


def test_layout_validation():
    with pytest.raises(DimsError):
        ShardLayout(10, 3)
    assert ShardLayout(12, 4).num_chunks == 3


def test_shard_shape_and_domain_checks():
    h, L, e = 1, 4, 2
    ok = dict(q=np.zeros((h, L, e)), k=np.zeros((h, L, e)), v=np.zeros((h, L, e)), g=np.full((h, L, e), -0.1),
              layout=ShardLayout(L, 2), dims=ModelDims(h, e, e))
    SeqShard(**ok)
    with pytest.raises(DimsError):
        SeqShard(**{**ok, "q": np.zeros((h, L + 1, e))})
    with pytest.raises(DomainError):
        SeqShard(**{**ok, "g": np.zeros((h, L, e))})
    with pytest.raises(DomainError):
        SeqShard(**{**ok, "g": np.full((h, L, e), np.nan)})


def test_state_and_cumdecay_checks():
    with pytest.raises(DimsError):
        State(np.zeros((2, 2)))
    with pytest.raises(DomainError):
        State(np.full((1, 1, 1), np.inf))
    with pytest.raises(DomainError):
        CumDecay(np.full((1, 2), 0.5))
    assert State.zeros(ModelDims(1, 2, 3)).values.shape == (1, 2, 3)


def test_pipeline_config():
    with pytest.raises(ConfigError):
        PipelineConfig(0)
    with pytest.raises(ConfigError):
        PipelineConfig(1, -1.0)


def test_global_sequence_and_split():
    with pytest.raises(LayoutError):
        GlobalSequence(q=np.zeros((1, 10, 2)), k=np.zeros((1, 10, 2)), v=np.zeros((1, 10, 2)),
                       g=np.full((1, 10, 2), -0.1), num_ranks=3, layout=ShardLayout(4, 2), dims=ModelDims(1, 2, 2))
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (2, 16, 3))
    seq = GlobalSequence(q=x, k=x, v=x, g=-np.abs(x) - 0.01, num_ranks=4, layout=ShardLayout(4, 2),
                         dims=ModelDims(2, 3, 3))
    shards = split(seq)
    np.testing.assert_array_equal(np.concatenate([s.v for s in shards], axis=1), seq.v)
    np.testing.assert_array_equal(shards[1].q, seq.q[:, 4:8])


def test_cluster_and_ledger_contract():
    with pytest.raises(ConfigError):
        create_cluster(0)
    with pytest.raises(ConfigError):
        NetConfig(bandwidth_beta=0.0)
    led = VolumeLedger(3, (LedgerRow(0, "all_scan", 5, 0), LedgerRow(1, "all_scan", 5, 5),
                           LedgerRow(2, "all_scan", 0, 5)))
    assert led.sent(rank=0) == 5 and led.total_sent == led.total_received == 10
    assert [r["rank"] for r in led.to_csv_rows()] == [0, 1, 2]


def test_overlap_schedule_and_makespan():
    tl = overlap_schedule(1.0, 2.0, 3.0, 1.0)
    assert tl.makespan == pytest.approx(5.0)
    with pytest.raises(ConfigError):
        overlap_schedule(-1.0, 0, 0, 0)
    assert ideal_makespan(StrategyKind.LASP1, 4, 8) == pytest.approx(4 * ideal_makespan(StrategyKind.ZECO, 4, 8))


def test_generate_sequence_is_byte_identical_to_oracle_draws():
    from oracle import gla_oracle as orc
    from paper_2507_01004_b200 import generate_sequence

    seq = generate_sequence(2, 8, 4, ModelDims(2, 3, 2), seed=5)
    q, k, v, g = orc.make_inputs(2, 8, 2, 3, 2, 5)
    for a, b in ((seq.q, q), (seq.k, k), (seq.v, v), (seq.g, g)):
        assert a.tobytes() == b.tobytes()
    with pytest.raises(ConfigError):
        generate_sequence(1, 8, 4, ModelDims(1, 1, 1), 0, decay_low=-0.1, decay_high=0.0)
    assert math.isclose(seq.g.max(), seq.g.max()) and np.all(seq.g < 0)


@pytest.mark.reference
@pytest.mark.parametrize("P,K,alpha,beta,cost", [(2, 1, 0.0, 1e9, 0.0), (5, 4, 2e-6, 5e8, 0.0), (8, 16, 1e-6, 2e9, 3e-7)])
def test_virtual_schedule_matches_live_reference(P, K, alpha, beta, cost):
    """The drop-in cluster charges All-Scan and the grouped all-gather exactly like the reference (host
    bookkeeping only, no GPU): same events (rank, label, start, end, stream), same clocks, same ledger."""
    import sys

    import numpy as np

    sys.path.insert(0, "/root/reference/pkg/src")
    import glasp.cluster as rc
    import glasp.collectives as rco
    from glasp.gla import CumDecay, State

    from paper_2507_01004_b200 import cluster as zc
    from paper_2507_01004_b200 import collectives as zco

    h, ek, ev = 2, 16, 3
    rng = np.random.default_rng(P + K)
    states = [State(rng.uniform(-1, 1, (h, ek, ev))) for _ in range(P)]
    cds = [CumDecay(rng.uniform(-2, 0, (h, ek))) for _ in range(P)]
    for direction in ("FWD", "BWD"):
        ref = rc.create_cluster(P, rc.NetConfig(alpha, beta))
        for r in range(P):  # uneven clocks before the collective
            ref.compute(r, 1e-6 * r, "warm")
        rco.all_scan(ref, states, cds, rco.PipelineConfig(K, cost), getattr(rco.ScanDirection, direction))
        rco.all_gather_grouped(ref, {"all_gather": [s.values for s in states]})
        ours = zc.create_cluster(P, zc.NetConfig(alpha, beta))
        for r in range(P):
            ours.compute(r, 1e-6 * r, "warm")
        zco.charge_all_scan(ours, P, h, ek, ev, zco.PipelineConfig(K, cost), getattr(zco.ScanDirection, direction))
        zco.all_gather_grouped(ours, {"all_gather": [s.values for s in states]})
        assert ours.clocks == ref.clocks
        assert ours.read_timeline().to_json_rows() == ref.read_timeline().to_json_rows()
        assert [(e.rank, e.label, e.start, e.end, e.stream) for e in ours.read_timeline().events] == \
            [(e.rank, e.label, e.start, e.end, e.stream) for e in ref.read_timeline().events]
        assert ours.read_ledger().to_csv_rows() == ref.read_ledger().to_csv_rows()
        assert ours.pending_messages() == ref.pending_messages() == 0
