"""Closed-form strategy model, calibrated against MEASURED All-Scan times.

The reference predicts communication with the alpha-beta message model
tau(s) = alpha + s / beta (glasp/costmodel.py:1-22, 78-90):

    All-Scan (P ranks, K blocks)   (K + P - 1) * tau(S / K)      (Eq. 13; 0 at P = 1)
    ZeCO                           t_ideal - t_overlap + tau(S)
    LASP-1                         P * (t_ideal + tau(S))
    LASP-2                         t_ideal + P * tau(S)

and a per-method volume / compute table (glasp/costmodel.py:118-140).  Those
closed forms are restated here with the same argument meaning and
ConfigError cases.  What is new is ``fit_net``: a least-squares fit of
(alpha, beta) to measured All-Scan timings (``scripts/allscan_bench.py``
output: P, K, state bytes, microseconds), which makes Eq. 13 a calibrated
predictor whose residuals are reported (``calibration_report``).  On one GPU
the measurements come from the list-form kernel (virtual ranks, flags through
L2); under torchrun from the NVLink peer-memory chain -- the fitted numbers
say which.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .cluster import NetConfig
from .errors import ConfigError
from .gla import ModelDims

METHODS = ("ulysses", "megatron_cp", "lasp1", "lasp2", "zeco")
SIMULATED_METHODS = ("zeco", "lasp1", "lasp2")
TABLE_COLUMNS = ("method", "P", "L", "D", "e", "N", "volume_elements", "compute_ops", "t_model_seconds")


@dataclass(frozen=True)
class CostParams:
    """Inputs of the closed forms, same fields as glasp/costmodel.py:38-62 (dims: ModelDims)."""

    net: NetConfig
    dims: ModelDims
    num_ranks: int
    pipeline_blocks: int = 1
    per_chunk_compute: float = 0.0
    chunks_per_rank: int = 1
    tokens_per_rank: int = 1

    def __post_init__(self):
        if self.num_ranks < 1:
            raise ConfigError(f"num_ranks must be >= 1, got {self.num_ranks}")
        if self.pipeline_blocks < 1:
            raise ConfigError(f"pipeline_blocks must be >= 1, got {self.pipeline_blocks}")
        if self.chunks_per_rank < 1 or self.tokens_per_rank < 1:
            raise ConfigError("chunks_per_rank and tokens_per_rank must be positive")
        if self.per_chunk_compute < 0.0:
            raise ConfigError("per_chunk_compute must be >= 0")

    @property
    def state_elements(self) -> int:
        return self.dims.state_elements


@dataclass(frozen=True)
class CostReport:
    t_allscan: float
    t_zeco: float
    t_lasp1: float
    t_lasp2: float
    volumes: dict
    computes: dict


def tau(size: float, net: NetConfig) -> float:
    if size < 0:
        raise ConfigError(f"message size must be >= 0, got {size}")
    return net.tau(size)


def t_allscan(p: CostParams) -> float:
    """Eq. 13: (K + P - 1) tau(S / K); a single rank sends nothing."""
    if p.dims.key_dim % p.pipeline_blocks:
        raise ConfigError(f"pipeline_blocks {p.pipeline_blocks} does not divide key dim {p.dims.key_dim}")
    if p.num_ranks == 1:
        return 0.0
    hops = p.pipeline_blocks + p.num_ranks - 1
    return hops * tau(p.state_elements / p.pipeline_blocks, p.net)


def volume_compute_table(method: str, p: CostParams):
    """(communication elements, compute ops) per method, D = h * e (square per-head states)."""
    if p.dims.key_dim != p.dims.value_dim:
        raise ConfigError("the unified table assumes e_k == e_v")
    e, P, L, N = p.dims.key_dim, p.num_ranks, p.tokens_per_rank, p.chunks_per_rank
    D = p.dims.heads * e
    table = {
        "ulysses": (4 * L * D, L * L * D * P),
        "megatron_cp": (2 * P * L * D, L * L * D * P),
        "lasp1": (P * D * e, P * L * D * e),
        "lasp2": (P * D * e, L * D * e + math.log2(P) * D * e + N * D * e),
        "zeco": (D * e, L * D * e + N * D * e + N * D),
    }
    if method not in table:
        raise ConfigError(f"unknown method {method!r}; expected one of {METHODS}")
    return table[method]


def t_strategies(p: CostParams, t_ideal: float, t_overlap: float) -> CostReport:
    if t_ideal < 0.0 or t_overlap < 0.0:
        raise ConfigError("phase times must be >= 0")
    if t_overlap > t_ideal:
        raise ConfigError(f"t_overlap {t_overlap} exceeds t_ideal {t_ideal}")
    ts = tau(p.state_elements, p.net)
    P = p.num_ranks
    vc = {m: volume_compute_table(m, p) for m in METHODS}
    return CostReport(t_allscan=t_allscan(p), t_zeco=t_ideal - t_overlap + ts, t_lasp1=P * (t_ideal + ts),
                      t_lasp2=t_ideal + P * ts, volumes={m: v[0] for m, v in vc.items()},
                      computes={m: v[1] for m, v in vc.items()})


def table_note(method: str) -> str:
    """Caveat attached to a table row (glasp/costmodel.py:140-148)."""
    return {"lasp1": "volume counts serialized order; per-rank physical volume is D*e",
            "lasp2": "table volume P*D*e vs per-rank gather volume (P-1)*D*e",
            "zeco": "compute term N*d read with d = D"}.get(method, "")


def table_rows(p: CostParams, methods=METHODS, report: CostReport | None = None):
    times = {} if report is None else {"zeco": report.t_zeco, "lasp1": report.t_lasp1, "lasp2": report.t_lasp2}
    rows = []
    for m in methods:
        vol, comp = volume_compute_table(m, p)
        rows.append({"method": m, "P": p.num_ranks, "L": p.tokens_per_rank, "D": p.dims.heads * p.dims.key_dim,
                     "e": p.dims.key_dim, "N": p.chunks_per_rank, "volume_elements": vol, "compute_ops": comp,
                     "t_model_seconds": times.get(m, "")})
    return rows


# ---------------------------------------------------------------- calibration against measurements

@dataclass(frozen=True)
class Sample:
    """One measured All-Scan: P ranks, K blocks, state of ``elements`` (fp32), ``seconds`` (mean)."""

    P: int
    K: int
    elements: int
    seconds: float


def fit_net(samples, element_bytes: int = 4) -> NetConfig:
    """Least-squares (alpha, beta) of  t = (K+P-1) alpha + (K+P-1) (S/K) / beta  over the samples.

    Linear in (alpha, 1/beta); solved by the 2x2 normal equations.  beta in elements/s."""
    rows = [((s.K + s.P - 1), (s.K + s.P - 1) * s.elements / s.K, s.seconds) for s in samples if s.P > 1]
    if len(rows) < 2:
        raise ConfigError("need at least two multi-rank samples to fit alpha and beta")
    a11 = sum(x * x for x, _, _ in rows)
    a12 = sum(x * y for x, y, _ in rows)
    a22 = sum(y * y for _, y, _ in rows)
    b1 = sum(x * t for x, _, t in rows)
    b2 = sum(y * t for _, y, t in rows)
    det = a11 * a22 - a12 * a12
    if det <= 0:
        raise ConfigError("degenerate samples: vary K, P or the state size")
    alpha = (b1 * a22 - b2 * a12) / det
    inv_beta = (a11 * b2 - a12 * b1) / det
    if inv_beta <= 0:  # bandwidth term not resolvable from these samples: latency-only fit
        alpha = sum(x * t for x, _, t in rows) / a11
        inv_beta = 1e-18
    return NetConfig(latency_alpha=max(alpha, 0.0), bandwidth_beta=1.0 / inv_beta, element_bytes=element_bytes)


def calibration_report(samples, net: NetConfig | None = None) -> dict:
    """Fit (unless given) and compare Eq. 13 with every sample: per-sample ratio measured / model."""
    samples = list(samples)
    net = net or fit_net(samples)
    out = []
    for s in samples:
        model = (s.K + s.P - 1) * net.tau(s.elements / s.K) if s.P > 1 else 0.0
        out.append({"P": s.P, "K": s.K, "state_bytes": s.elements * net.element_bytes, "measured_us": s.seconds * 1e6,
                    "model_us": model * 1e6, "ratio": s.seconds / model if model > 0 else float("nan")})
    ratios = [r["ratio"] for r in out if r["ratio"] == r["ratio"]]
    return {"alpha_us": net.latency_alpha * 1e6, "beta_GBps": net.bandwidth_beta * net.element_bytes / 1e9,
            "ratio_min": min(ratios), "ratio_max": max(ratios),
            "ratio_geomean": math.exp(sum(math.log(r) for r in ratios) / len(ratios)), "samples": out}


def samples_from_bench(lines) -> list:
    """Parse ``scripts/allscan_bench.py`` JSON lines into Samples: virtual rows (``allscan_us_mean``,
    one GPU) and NVLink rows of the product chain (``impl`` = ``p2p_K<k>``, ``us_mean``)."""
    import json
    out = []
    for ln in lines:
        ln = ln.strip()
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        if "allscan_us_mean" in d:
            K, us = int(d["K"]), float(d["allscan_us_mean"])
        elif str(d.get("impl", "")).startswith("p2p_K"):
            K, us = int(d["impl"][5:]), float(d["us_mean"])
        else:
            continue
        out.append(Sample(P=int(d["P"]), K=K, elements=int(d["state_bytes"]) // 4, seconds=us * 1e-6))
    return out
