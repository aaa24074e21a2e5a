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


class _HostOps:
    """numpy: inverse-CDF draws and first-occurrence dedupe."""

    def draw(self, rng, cdf, size):
        return _draw(rng, cdf, size)

    def first_unique(self, keys):
        _, first = np.unique(keys, return_index=True)
        return keys[np.sort(first)]


class _TorchOps:
    """The same two operations on a torch device (the uniforms still come from
    the numpy generator, so the graph is bit-identical to the host path):
    ``searchsorted(cdf, x, right=True)`` is an exact comparison on the same
    doubles, and a stable sort keeps the first occurrence of every key first in
    its run.  Test/bench input generation only (c3/c4 in seconds, not minutes)."""

    def __init__(self, device):
        import torch

        self.torch = torch
        self.dev = torch.device(device)
        self._cdf = {}

    def draw(self, rng, cdf, size):
        t = self.torch
        key = id(cdf)
        if key not in self._cdf:
            self._cdf[key] = (cdf, t.from_numpy(cdf).to(self.dev))
        dc = self._cdf[key][1]
        out = np.empty(size, dtype=np.int64)
        step = 1 << 26
        for i in range(0, size, step):  # bounded device memory; same draws, same order
            x = t.from_numpy(rng.random(min(step, size - i))).to(self.dev)
            out[i:i + x.numel()] = t.searchsorted(dc, x, right=True).cpu().numpy()
        return out

    def first_unique(self, keys):
        t = self.torch
        k = t.from_numpy(keys).to(self.dev)
        sk, order = t.sort(k, stable=True)
        head = t.ones_like(sk, dtype=t.bool)
        head[1:] = sk[1:] != sk[:-1]
        keep = t.zeros_like(head)
        keep[order[head]] = True
        out = k[keep].cpu().numpy()
        del k, sk, order, head, keep
        return out


def _ops(device):
    if device is None:
        return _HostOps()
    return _TorchOps(device)


def chung_lu_edges(u_count: int, v_count: int, edge_count: int, beta_u: float, beta_v: float,
                   weights: str, seed: int, max_deg_v: int | None = None, max_deg_u: int | None = None,
                   device=None):
    """(eu, ev, ew) with exactly ``edge_count`` distinct pairs, every node covered.

    ``device`` (a torch device such as ``"cuda:0"``) runs the draws' inverse-CDF
    lookups and the dedupe there; the result is identical to the host path."""
    if edge_count < max(u_count, v_count) or edge_count > u_count * v_count:
        raise ValueError("edge_count must lie in [max(|U|,|V|), |U||V|]")
    ops = _ops(device)
    rng = substream(seed, "chung-lu", u_count, v_count, edge_count)
    pu = _expected_shares(u_count, beta_u, edge_count, max_deg_u)
    pv = _expected_shares(v_count, beta_v, edge_count, max_deg_v)
    cu = np.cumsum(pu)
    cu /= cu[-1]
    cv = np.cumsum(pv)
    cv /= cv[-1]
    m = max(u_count, v_count)
    us = np.concatenate([rng.permutation(u_count), ops.draw(rng, cu, m - u_count)])
    vs = np.concatenate([rng.permutation(v_count), ops.draw(rng, cv, m - v_count)])
    rng.shuffle(vs)
    keys = ops.first_unique(us * v_count + vs)
    while keys.size < edge_count:
        need = edge_count - keys.size
        n = int(need * 1.25) + 1024
        cand = ops.draw(rng, cu, n) * v_count
        cand += ops.draw(rng, cv, n)
        keys = ops.first_unique(np.concatenate([keys, cand]))[:edge_count]
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
    """The config's graph; ``device`` also generates the edges (draw lookups,
    dedupe; identical graph) and canonicalises the CSR on that GPU."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    eu, ev, ew = chung_lu_edges(cfg.u_count, cfg.v_count, cfg.edge_count, cfg.beta_u, cfg.beta_v,
                                cfg.weights, cfg.seed if seed is None else seed, cfg.max_deg_v,
                                device=None if device is None else f"cuda:{device}")
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
