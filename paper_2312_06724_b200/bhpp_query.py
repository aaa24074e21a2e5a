"""Two-way (BHPP) similarity queries on the device: drop-in for
``bipush.bhpp_query`` (pkg/src/bipush/bhpp_query.py) plus a batched API.

The per-graph preprocessing (lambda, tau, mu, the epsilon split, the
fingerprint) and the query arithmetic keep the reference's definitions; the
push rounds, power iterations, BHPP combination and top-k run in the CUDA
engine.  ``bhpp_query_batch`` is the B200-native entry point the reference
lacks: many sources per call, query blocks of B slots resident in HBM, slots
refilled on device as queries finish, top-k per query computed on device.
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable

import numpy as np

from . import _capi
from .bigraph import DataError
from .push_engine import power_iteration, required_iterations, run_job

META_VERSION = 1


@dataclass
class IndexMeta:
    """Query-independent per-graph parameters (bhpp_query.py:32-47)."""

    alpha: float
    lam: float
    tau: int
    mu: float
    eps_split_policy: Callable[[float], float]
    graph_fingerprint: str


@dataclass
class QueryResult:
    """Scores plus the accounting needed to audit a query (bhpp_query.py:50-62).
    ``engine`` carries device-only bookkeeping (tie decisions, dtype)."""

    method: str
    query_index: int
    scores: np.ndarray
    epsilon: float
    epsilon_b: float
    epsilon_f: float
    timing: dict
    phase_trace: dict
    u_labels: list[str] | None = None
    engine: dict | None = None


@dataclass
class BatchResult:
    """Result of ``bhpp_query_batch``: per-query top-k and traces.

    topk_index[i, j] / topk_score[i, j] is the j-th best (score desc, index
    asc) U node of sources[i]; -1 / 0.0 pad when |U| < k.  ``traces`` is a
    structured array with the bh_trace fields (see trace_dicts()).
    """

    sources: np.ndarray
    epsilon: float
    epsilon_b: float
    epsilon_f: float
    k: int
    topk_index: np.ndarray
    topk_score: np.ndarray
    traces: np.ndarray
    scores: np.ndarray | None
    timing: dict
    dtype: str
    meta: dict = field(default_factory=dict)

    def trace_dicts(self, i: int) -> dict:
        back, fwd, _ = _capi.trace_dicts(self.traces[i])
        return {"backward": back, "forward": fwd}


def default_tau(g, alpha: float, slack: float = 0.05) -> int:
    """Probe depth keeping |U| (1-alpha)^(tau+1) <= slack (bhpp_query.py:65-67)."""
    return required_iterations(alpha, slack, float(g.u_count))


def estimate_lambda(g, alpha: float, tau: int) -> float:
    """Upper bound on the column sums of the hidden walk-score matrix
    (bhpp_query.py:70-83): tau power iterations from the all-ones vector on the
    device (fp64), plus the |U| (1-alpha)^(tau+1) tail, capped by max ws / min ws."""
    if tau < 0:
        raise ValueError("tau must be nonnegative")
    probe = power_iteration(g, np.ones(g.u_count), alpha, tau, dtype="fp64")
    from_probe = float(probe.max()) + g.u_count * (1.0 - alpha) ** (tau + 1)
    from_ratio = float(g.ws_u.max() / g.ws_u.min())
    return min(from_probe, from_ratio)


def estimate_mu(g) -> float:
    """Density proxy sqrt(|U||V|)/|E| clamped into [1e-3, 1] (bhpp_query.py:86-89)."""
    raw = math.sqrt(g.u_count * g.v_count) / g.edge_count
    return float(min(1.0, max(1e-3, raw)))


def choose_eps_b(epsilon: float, mu) -> float:
    """Backward share eps (1-mu)/(2-mu) clamped into [eps/10, eps/2]
    (bhpp_query.py:92-104).  ``mu`` may be a density or a graph."""
    if epsilon <= 0:
        raise ValueError("epsilon must be positive")
    if hasattr(mu, "u_count") and hasattr(mu, "edge_count"):
        mu = estimate_mu(mu)
    mu = float(mu)
    raw = epsilon * (1.0 - mu) / (2.0 - mu)
    return min(max(raw, epsilon / 10.0), epsilon / 2.0)


def build_index_meta(g, alpha: float = 0.15, tau: int | None = None) -> IndexMeta:
    """bhpp_query.py:107-123, with lambda's power iteration on the device."""
    if tau is None:
        tau = default_tau(g, alpha)
    lam = estimate_lambda(g, alpha, tau)
    mu = estimate_mu(g)

    def policy(epsilon: float, _mu=mu) -> float:
        return choose_eps_b(epsilon, _mu)

    return IndexMeta(alpha=alpha, lam=lam, tau=int(tau), mu=mu, eps_split_policy=policy,
                     graph_fingerprint=g.fingerprint)


def save_meta(meta: IndexMeta, path) -> None:
    payload = {
        "format_version": META_VERSION, "alpha": meta.alpha, "lambda": meta.lam, "tau": meta.tau,
        "mu": meta.mu, "graph_fingerprint": meta.graph_fingerprint,
    }
    Path(path).write_text(json.dumps(payload, indent=2) + "\n", encoding="utf-8")


def load_meta(path) -> IndexMeta:
    try:
        payload = json.loads(Path(path).read_text(encoding="utf-8"))
    except (OSError, json.JSONDecodeError) as exc:
        raise DataError(f"cannot read index metadata: {exc}") from None
    if payload.get("format_version") != META_VERSION:
        raise DataError("unsupported index metadata version")
    mu = float(payload["mu"])

    def policy(epsilon: float, _mu=mu) -> float:
        return choose_eps_b(epsilon, _mu)

    return IndexMeta(alpha=float(payload["alpha"]), lam=float(payload["lambda"]), tau=int(payload["tau"]),
                     mu=mu, eps_split_policy=policy, graph_fingerprint=str(payload["graph_fingerprint"]))


def _split(meta: IndexMeta, g, epsilon: float):
    """Fingerprint check and epsilon split (bhpp_query.py:167-181)."""
    if meta.graph_fingerprint != g.fingerprint:
        raise DataError("index metadata does not match this graph (fingerprint mismatch); rebuild the index")
    if epsilon <= 0:
        raise ValueError("epsilon must be positive")
    eps_b = float(meta.eps_split_policy(epsilon))
    eps_f = epsilon - eps_b
    if eps_b <= 0 or eps_f <= 0:
        raise ValueError(f"epsilon split ({eps_b}, {eps_f}) must leave both directions positive")
    return eps_b, eps_f


def bhpp_query(g, meta: IndexMeta, query_u, epsilon: float, round_hook=None, dtype: str = "fp64",
               tie_skip: int = 0) -> QueryResult:
    """Two-way scores for every U node, accurate to epsilon entrywise
    (bhpp_query.py:160-203).  Runs as one device query slot."""
    eps_b, eps_f = _split(meta, g, epsilon)
    q = g.u_id(query_u) if isinstance(query_u, str) else int(query_u)
    if not 0 <= q < g.u_count:
        raise ValueError(f"node index {q} out of range")
    t0 = time.perf_counter()
    _, scores, tr = run_job(g, _capi.JOB_BHPP, q, meta.alpha, meta.lam, eps_b, eps_f,
                            round_hook=round_hook, tie_skip=tie_skip, dtype=dtype)
    t2 = time.perf_counter()
    back, fwd, extra = _capi.trace_dicts(tr)
    # the device runs both directions in one launch sequence; split the wall
    # time by round counts (backward rounds vs forward rounds + PI iterations)
    rb = back["selective_rounds"] + back["sequential_rounds"]
    rf = fwd["selective_rounds"] + fwd["power_iterations"]
    share = rb / (rb + rf) if rb + rf else 0.5
    total = t2 - t0
    extra["dtype"] = dtype
    return QueryResult(
        method="ssbipush", query_index=q, scores=scores, epsilon=epsilon, epsilon_b=eps_b, epsilon_f=eps_f,
        timing={"backward": total * share, "forward": total * (1 - share), "total": total},
        phase_trace={"backward": back, "forward": fwd},
        u_labels=g.u_labels, engine=extra,
    )


def _source_list(sources) -> list:
    """The batch's sources one by one, each keeping its own type (a label or an
    index); np.atleast_1d on a mixed list would turn every index into a string."""
    if isinstance(sources, (str, bytes)) or np.isscalar(sources):
        return [sources]
    if isinstance(sources, np.ndarray):
        return sources.reshape(-1).tolist()
    return list(sources)


def bhpp_query_batch(g, meta: IndexMeta, sources, epsilon: float, k: int | None = 50,
                     exclude_query: bool = False, dtype: str = "fp32", return_scores: bool = False,
                     slots: int | None = None, tie_skip=None, stream=None, device: int | None = None) -> BatchResult:
    """SS-BI-PUSH for many sources at once on the device.

    Equivalent to ``[topk(bhpp_query(g, meta, s, epsilon), k, exclude_query)
    for s in sources]`` (the reference's cmd_bench / evalkit loops,
    cli.py:432-450, evalkit.py:280-285) but executed as query blocks of
    ``slots`` sources sharing every SpMM pass.  ``dtype`` "fp32" stores state in
    fp32 with fp64 row accumulation and fp64 control; "fp64" is all fp64.
    """
    eps_b, eps_f = _split(meta, g, epsilon)
    src = np.array([g.u_id(s) if isinstance(s, str) else int(s) for s in _source_list(sources)], dtype=np.int32)
    if src.size and (src.min() < 0 or src.max() >= g.u_count):
        raise ValueError("node index out of range")
    kk = 0 if not k else int(k)
    if kk < 0:
        raise ValueError("k must be positive")
    kk = min(kk, g.u_count)
    dg = _capi.device_graph(g, dtype, device)
    n_q = src.size
    prm = _capi.QueryParams(alpha=meta.alpha, lam=meta.lam, eps_b=eps_b, eps_f=eps_f, k=kk,
                            exclude_query=int(bool(exclude_query)), want_scores=int(bool(return_scores)),
                            slots=int(slots or 0), on_device=0)
    tk_idx = np.full((n_q, max(kk, 1)), -1, dtype=np.int32)
    tk_sc = np.zeros((n_q, max(kk, 1)))
    traces = np.zeros(n_q, dtype=_capi.TRACE_DTYPE)
    scores = np.empty((n_q, g.u_count)) if return_scores else None
    ties = None if tie_skip is None else np.ascontiguousarray(np.broadcast_to(tie_skip, (n_q,)), dtype=np.int32)
    import ctypes as C

    t0 = time.perf_counter()
    _capi.apply_scatter_limit()
    _capi.check(_capi.lib().bh_query_batch(
        dg.h, C.byref(prm), _capi.ptr(src), n_q, _capi.ptr(ties), _capi.ptr(tk_idx) if kk else None,
        _capi.ptr(tk_sc) if kk else None, _capi.ptr(traces), _capi.ptr(scores),
        C.c_void_p(stream) if stream else None))
    t1 = time.perf_counter()
    if kk == 0:
        tk_idx, tk_sc = tk_idx[:, :0], tk_sc[:, :0]
    return BatchResult(sources=src, epsilon=epsilon, epsilon_b=eps_b, epsilon_f=eps_f, k=kk, topk_index=tk_idx,
                       topk_score=tk_sc, traces=traces, scores=scores, timing={"total": t1 - t0}, dtype=dtype)


def query_batch_device(dg, meta: IndexMeta, eps_b: float, eps_f: float, sources_ptr: int, n_q: int, k: int,
                       topk_idx_ptr: int, topk_score_ptr: int, trace_ptr: int, scores_ptr: int = 0,
                       exclude_query: bool = False, slots: int | None = None, tie_ptr: int = 0,
                       stream: int | None = None, async_: bool = False) -> None:
    """bh_query_batch with every buffer already resident on the device (raw
    device pointers, e.g. torch ``data_ptr()``); nothing crosses PCIe.  The
    caller owns the stream ordering (``stream`` = cudaStream_t handle).
    ``async_``: return once enqueued; ``query_wait(dg)`` completes the batch."""
    import ctypes as C

    prm = _capi.QueryParams(alpha=meta.alpha, lam=meta.lam, eps_b=eps_b, eps_f=eps_f, k=int(k),
                            exclude_query=int(bool(exclude_query)), want_scores=int(bool(scores_ptr)),
                            slots=int(slots or 0), on_device=1, flags=_capi.QUERY_ASYNC if async_ else 0)
    vp = lambda x: C.c_void_p(x) if x else None  # noqa: E731
    _capi.apply_scatter_limit()
    _capi.check(_capi.lib().bh_query_batch(dg.h, C.byref(prm), vp(sources_ptr), int(n_q), vp(tie_ptr),
                                           vp(topk_idx_ptr), vp(topk_score_ptr), vp(trace_ptr), vp(scores_ptr),
                                           vp(stream)))


def query_wait(dg) -> None:
    """Complete a batch submitted with ``query_batch_device(..., async_=True)``."""
    _capi.check(_capi.lib().bh_query_wait(dg.h))


def topk(result: QueryResult, k: int, exclude_query: bool = False) -> list[tuple[str, float]]:
    """Top-k (label, score) pairs, scores descending, ties by ascending index
    (bhpp_query.py:206-218); the selection runs on the device (bh_topk)."""
    import ctypes as C

    if k <= 0:
        raise ValueError("k must be positive")
    scores = np.ascontiguousarray(result.scores, dtype=np.float64)
    n = scores.size
    kk = min(int(k), n)
    idx = np.empty(max(kk, 1), dtype=np.int64)
    val = np.empty(max(kk, 1))
    cnt = np.zeros(1, dtype=np.int64)
    excl = int(result.query_index) if exclude_query else -1
    _capi.check(_capi.lib().bh_topk(_capi.ptr(scores), n, kk, excl, _capi.ptr(idx), _capi.ptr(val),
                                    _capi.ptr(cnt)))
    m = int(cnt[0])
    labels = result.u_labels
    return [(labels[i] if labels is not None else str(i), float(scores[i])) for i in idx[:m].tolist()]


