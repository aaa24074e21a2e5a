"""Batched callers of the query path.

The reference drives the hot path from its CLI one source at a time:
``_run_query`` for ``bipush query|topk`` (cli.py:360-369) and the
``cmd_bench`` loop (cli.py:410-521: seeded sources, every method at every
epsilon, timing rows, pairwise agreement rows within 2 eps, optionally a
thread pool over the sources, cli.py:444-450).  These are the same callers
over this package's API, returning the rows as dicts; the CLI's argument
parsing and text formatting (``emit_rows``) stay out of scope (section 8).

The difference is in how "ssbipush" runs: the whole source set is one
device batch (``bhpp_query_batch``), so its timing row reports the batch
wall time divided by the source count (``mean_s``) with ``stddev_s`` = None
and ``batched`` = True -- a batch has no per-source wall times.  "pisp" and
"mcsp" run per source as in the reference (their kernels take one source).
"""

from __future__ import annotations

import time
from itertools import combinations

import numpy as np

from .baselines import DeadlineExceeded, build_alias, mcsp_query, pisp_query
from .bhpp_query import bhpp_query, bhpp_query_batch
from .rng import substream

METHODS = ("ssbipush", "mcsp", "pisp")


def run_query(g, meta, method: str, query, epsilon: float, p_f: float = 1e-6, seed: int = 0, alias=None):
    """One query by method name (cli.py:360-369); ValueError for an unknown method."""
    if method == "ssbipush":
        return bhpp_query(g, meta, query, epsilon)
    if method == "mcsp":
        return mcsp_query(g, alias if alias is not None else build_alias(g), query, meta.alpha, epsilon, p_f, seed)
    if method == "pisp":
        return pisp_query(g, query, meta.alpha, epsilon)
    raise ValueError(f"unknown method {method!r}; choose from {', '.join(METHODS)}")


def bench_queries(g, n: int, seed: int = 0) -> list[int]:
    """The bench's sources: the reference sampler (cli.py:415-417)."""
    n = min(int(n), g.u_count)
    return substream(seed, "bench-queries").choice(g.u_count, size=n, replace=False).tolist()


def bench_rows(g, meta, methods=("ssbipush",), epsilons=(1e-4,), queries: int = 10, seed: int = 0,
               p_f: float = 1e-6, timeout: float = 60.0, dtype: str = "fp64") -> tuple[list[dict], bool]:
    """cmd_bench's measurement (cli.py:410-521) as rows: one "timing" row per
    (epsilon, method) and one "agreement" row per method pair that finished.
    Returns (rows, excluded_any); a method whose total time exceeds
    ``timeout`` x sources is reported excluded, as in the reference."""
    for m in methods:
        if m not in METHODS:
            raise ValueError(f"unknown method {m!r}; choose from {', '.join(METHODS)}")
    qs = bench_queries(g, queries, seed)
    n = len(qs)
    alias = build_alias(g) if "mcsp" in methods else None
    rows: list[dict] = []
    excluded_any = False
    for eps in epsilons:
        kept: dict[str, list[np.ndarray]] = {}
        for method in methods:
            budget = timeout * n
            start = time.perf_counter()
            deadline = start + budget
            times: list[float] = []
            scores: list[np.ndarray] = []
            excluded = False
            batched = method == "ssbipush"
            try:
                if batched:
                    res = bhpp_query_batch(g, meta, qs, eps, k=None, dtype=dtype, return_scores=True)
                    total = time.perf_counter() - start
                    scores = list(res.scores)
                    times = [total / max(n, 1)] * n
                    excluded = total > budget
                else:
                    for qi, q in enumerate(qs):
                        if time.perf_counter() > deadline:
                            excluded = True
                            break
                        if method == "pisp":
                            r = pisp_query(g, q, meta.alpha, eps)
                        else:
                            walk_seed = int(substream(seed, "bench-mc", qi).integers(0, 2**63))
                            r = mcsp_query(g, alias, q, meta.alpha, eps, p_f, walk_seed, deadline=deadline)
                        times.append(r.timing["total"])
                        scores.append(r.scores)
            except DeadlineExceeded:
                excluded = True
            if excluded:
                excluded_any = True
                rows.append({"kind": "timing", "method": method, "epsilon": eps, "mean_s": None, "stddev_s": None,
                             "n": len(times), "excluded": True, "batched": batched})
            else:
                arr = np.asarray(times)
                rows.append({"kind": "timing", "method": method, "epsilon": eps, "mean_s": float(arr.mean()),
                             "stddev_s": None if batched else float(arr.std(ddof=0)), "n": n, "excluded": False,
                             "batched": batched})
                kept[method] = scores
        for a, b in combinations([m for m in methods if m in kept], 2):
            worst = max(float(np.abs(sa - sb).max()) for sa, sb in zip(kept[a], kept[b])) if n else 0.0
            bound = 2.0 * eps
            rows.append({"kind": "agreement", "method": f"{a}|{b}", "epsilon": eps, "max_abs_diff": worst,
                         "bound": bound, "within": worst <= bound})
    return rows, excluded_any
