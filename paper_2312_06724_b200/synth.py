"""Seeded synthetic bipartite graphs for the BASELINE.json configurations.

The reference ships no Chung-Lu generator (its ``synth_bipartite``,
bigraph.py:424-510, is an index-power skew with a per-edge Python loop that
cannot reach 1e8 edges), and the paper's datasets are not available, so the
configurations are seeded Chung-Lu stand-ins:

* expected-degree weights ``w_i ~ (i+1)^(-1/(beta-1))`` per side, optionally
  water-filled under a maximum expected degree (config 4's V hubs);
* covering edges first (a permutation on each side, as bigraph.py:468-471), so
  every node has degree >= 1 and |U|, |V| stay exactly as configured;
* then endpoint pairs drawn independently in proportion to the weights, keeping
  first occurrences, until exactly E distinct pairs exist;
* weights are unit or integers uniform in [1, 10] ("click counts").

Everything is vectorised numpy and deterministic in (config, seed).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .bigraph import BipartiteGraph
from .rng import substream


@dataclass(frozen=True)
class GraphConfig:
    name: str
    u_count: int
    v_count: int
    edge_count: int
    beta_u: float
    beta_v: float
    weights: str  # "unit" | "int10"
    alpha: float
    epsilons: tuple
    n_sources: int | None  # None = every u
    k: int
    max_deg_v: int | None = None
    seed: int = 2312


# BASELINE.json "configs", in order.
CONFIGS = {
    "c1": GraphConfig("c1", 1_000, 1_500, 10_000, 2.5, 2.5, "unit", 0.15, (1e-6,), 1, 10),
    "c2": GraphConfig("c2", 100_000, 200_000, 2_000_000, 2.2, 2.2, "int10", 0.15, (1e-7,), 64, 50),
    "c3": GraphConfig("c3", 5_000_000, 2_000_000, 100_000_000, 2.1, 2.1, "int10", 0.15, (1e-7,), 1024, 50),
    "c4": GraphConfig("c4", 2_000_000, 10_000_000, 300_000_000, 2.3, 1.8, "unit", 0.2, (1e-6,), 4096, 20,
                      max_deg_v=1_000_000),
    "c5": GraphConfig("c5", 100_000, 200_000, 2_000_000, 2.2, 2.2, "int10", 0.15, (1e-4, 1e-6, 1e-8), None, 50),
}


def _expected_shares(n: int, beta: float, edge_count: int, max_deg: int | None) -> np.ndarray:
    p = (np.arange(n, dtype=np.float64) + 1.0) ** (-1.0 / (beta - 1.0))
    p /= p.sum()
    if max_deg is not None:
        cap = max_deg / float(edge_count)
        for _ in range(200):  # water-filling: clip, renormalise the rest
            over = p > cap
            if not over.any():
                break
            free = ~over
            p[over] = cap
            rest = 1.0 - cap * over.sum()
            p[free] *= rest / p[free].sum()
    return p


def _draw(rng: np.random.Generator, cdf: np.ndarray, size: int) -> np.ndarray:
    return np.searchsorted(cdf, rng.random(size), side="right").astype(np.int64)


def chung_lu_edges(u_count: int, v_count: int, edge_count: int, beta_u: float, beta_v: float,
                   weights: str, seed: int, max_deg_v: int | None = None, max_deg_u: int | None = None):
    """(eu, ev, ew) with exactly ``edge_count`` distinct pairs, every node covered."""
    if edge_count < max(u_count, v_count) or edge_count > u_count * v_count:
        raise ValueError("edge_count must lie in [max(|U|,|V|), |U||V|]")
    rng = substream(seed, "chung-lu", u_count, v_count, edge_count)
    pu = _expected_shares(u_count, beta_u, edge_count, max_deg_u)
    pv = _expected_shares(v_count, beta_v, edge_count, max_deg_v)
    cu = np.cumsum(pu)
    cu /= cu[-1]
    cv = np.cumsum(pv)
    cv /= cv[-1]
    m = max(u_count, v_count)
    us = np.concatenate([rng.permutation(u_count), _draw(rng, cu, m - u_count)])
    vs = np.concatenate([rng.permutation(v_count), _draw(rng, cv, m - v_count)])
    rng.shuffle(vs)
    keys = us * v_count + vs
    _, first = np.unique(keys, return_index=True)
    keys = keys[np.sort(first)]
    while keys.size < edge_count:
        need = edge_count - keys.size
        n = int(need * 1.25) + 1024
        cand = _draw(rng, cu, n) * v_count + _draw(rng, cv, n)
        allk = np.concatenate([keys, cand])
        _, first = np.unique(allk, return_index=True)
        keys = allk[np.sort(first)][:edge_count]
    eu = keys // v_count
    ev = keys % v_count
    if weights == "unit":
        ew = np.ones(edge_count, dtype=np.float64)
    elif weights == "int10":
        ew = rng.integers(1, 11, size=edge_count).astype(np.float64)
    else:
        raise ValueError(f"unknown weight model {weights!r}")
    return eu, ev, ew


def make_graph(cfg: GraphConfig | str, seed: int | None = None, device: int | None = None) -> BipartiteGraph:
    """The config's graph; ``device`` canonicalises the CSR on that GPU."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    eu, ev, ew = chung_lu_edges(cfg.u_count, cfg.v_count, cfg.edge_count, cfg.beta_u, cfg.beta_v,
                                cfg.weights, cfg.seed if seed is None else seed, cfg.max_deg_v)
    return BipartiteGraph.from_arrays(cfg.u_count, cfg.v_count, eu, ev, ew, device=device)


def scaled_config(cfg: GraphConfig | str, scale: float, name: str | None = None) -> GraphConfig:
    """Same shape parameters at 1/scale of the node and edge counts (parity sizes)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    d = dict(cfg.__dict__)
    d["name"] = name or f"{cfg.name}_s{scale:g}"
    d["u_count"] = max(2, int(cfg.u_count / scale))
    d["v_count"] = max(2, int(cfg.v_count / scale))
    d["edge_count"] = max(d["u_count"], d["v_count"], int(cfg.edge_count / scale))
    if cfg.max_deg_v is not None:
        d["max_deg_v"] = max(1, int(cfg.max_deg_v / scale))
    return GraphConfig(**d)


def bench_sources(u_count: int, n: int, seed: int = 0) -> np.ndarray:
    """Source nodes drawn exactly as the reference's bench (cli.py:415-417)."""
    if n >= u_count:
        return np.arange(u_count, dtype=np.int64)
    return substream(seed, "bench-queries").choice(u_count, n, replace=False).astype(np.int64)
