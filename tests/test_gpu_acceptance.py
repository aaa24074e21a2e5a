"""Acceptance criteria of the reference (pkg/tests/test_acceptance.py, SPEC
criteria 1, 5 and 10 -- SURVEY.md section 4) on the device engine, over a
seeded corpus of random bipartite graphs checked against the dense solve
Pi = alpha (I - (1 - alpha) P)^-1 with P = U V the two-hop U -> U walk.

- crit 1: BHPP scores are within epsilon of the truth from below, every eps;
- symmetry: the BHPP truth pi(s, t) + pi(t, s) is symmetric (the two-way form of crit 5's
  weight-scaled symmetry of pi), so the engine's beta(s, t) and beta(t, s) agree within eps;
- crit 10: gamma (forward residue mass at PI-Push entry) is monotone in eps_b.
The corpus is this repository's own (the reference's random_bigraph cannot be
imported on the GPU box): |U|, |V| in [10, 200], covering assignment + random
distinct edges, integer or real weights.
"""

import numpy as np
import pytest

import paper_2312_06724_b200 as bh
from oracle import cpu_oracle as O
from paper_2312_06724_b200.rng import substream

pytestmark = pytest.mark.gpu

ALPHA = 0.15


def random_bigraph(rng, nu, nv, avg_deg, weight_hi):
    """Every node covered once, then random distinct extra edges."""
    eu = list(rng.integers(0, nu, size=nv))                     # each v gets one u
    ev = list(range(nv))
    eu += list(range(nu))                                       # each u gets one v
    ev += list(rng.integers(0, nv, size=nu))
    extra = int(avg_deg * nu)
    eu += list(rng.integers(0, nu, size=extra))
    ev += list(rng.integers(0, nv, size=extra))
    key = np.unique(np.asarray(eu, np.int64) * nv + np.asarray(ev, np.int64))
    w = rng.uniform(0.1, weight_hi, size=key.size)
    if weight_hi >= 10:
        w = np.ceil(w)
    return bh.BipartiteGraph([f"u{i}" for i in range(nu)], [f"v{i}" for i in range(nv)],
                             key // nv, key % nv, w)


def dense_pi(g):
    U = np.zeros((g.u_count, g.v_count))
    V = np.zeros((g.v_count, g.u_count))
    eu = np.repeat(np.arange(g.u_count), g.deg_u)
    U[eu, g.u_indices] = g.u_weights / g.ws_u[eu]
    ev = np.repeat(np.arange(g.v_count), g.deg_v)
    V[ev, g.v_indices] = g.v_weights / g.ws_v[ev]
    return ALPHA * np.linalg.inv(np.eye(g.u_count) - (1.0 - ALPHA) * (U @ V))


def corpus(n):
    rng = substream(2026, "acceptance-corpus")
    for i in range(n):
        nu, nv = (int(x) for x in rng.integers(10, 201, size=2))
        yield i, random_bigraph(rng, nu, nv, float(rng.uniform(1.0, 4.0)), float(rng.choice([1.0, 10.0])))


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_crit1_one_sided_error_and_two_way_symmetry(dtype):
    tol = 1e-10 if dtype == "fp64" else 1e-5  # fp32 storage: relative 1e-5 of scores <= 1
    for i, g in corpus(200):
        Pi = dense_pi(g)
        meta = bh.build_index_meta(g, ALPHA)
        srcs = np.arange(min(g.u_count, 12))
        for eps in (1e-2, 1e-3, 1e-4, 1e-5, 1e-6):
            res = bh.bhpp_query_batch(g, meta, srcs, eps, k=5, dtype=dtype, return_scores=True)
            for j, q in enumerate(srcs):
                truth = Pi[q, :] + Pi[:, q]
                diff = truth - res.scores[j]
                assert diff.min() >= -tol and diff.max() <= eps + tol, (i, eps, int(q), diff.min(), diff.max())
            # beta(s, t) and beta(t, s) estimate the same symmetric quantity
            for a in range(len(srcs)):
                for b in range(a + 1, len(srcs)):
                    assert abs(res.scores[a][srcs[b]] - res.scores[b][srcs[a]]) <= eps + tol, (i, eps, a, b)


def test_crit10_gamma_monotone_in_eps_b():
    """A smaller backward threshold leaves less residue mass for the forward
    pass: gamma at PI-Push entry is non-increasing as eps_b shrinks."""
    for i, g in corpus(20):
        meta = bh.build_index_meta(g, ALPHA)
        srcs = np.arange(min(g.u_count, 6))
        gam = []
        for eps in (1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6):
            res = bh.bhpp_query_batch(g, meta, srcs, eps, k=0, dtype="fp64")
            gam.append(np.array([res.trace_dicts(j)["forward"]["gamma"] for j in range(len(srcs))]))
        for a, b in zip(gam, gam[1:]):
            assert np.all(b <= a * (1 + 1e-12) + 1e-15), (i, a, b)


def _graph(nu, nv, edges, weights=None):
    eu = [a for a, _ in edges]
    ev = [b for _, b in edges]
    w = weights if weights is not None else [1.0] * len(edges)
    return bh.BipartiteGraph([f"u{i}" for i in range(nu)], [f"v{i}" for i in range(nv)], eu, ev, w)


@pytest.mark.parametrize("name", ["single_u", "single_v", "star_u", "star_v", "extreme_weights", "path"])
def test_degenerate_graphs_one_sided(name):
    """Shapes at the edges of the domain: one U node, one V node, stars, weight
    ratios of 1e12, a long path; every eps from loose (0.5) to 1e-9."""
    if name == "single_u":
        g = _graph(1, 3, [(0, 0), (0, 1), (0, 2)], [1.0, 2.0, 3.0])
    elif name == "single_v":
        g = _graph(5, 1, [(i, 0) for i in range(5)], [1.0, 2.0, 3.0, 4.0, 5.0])
    elif name == "star_u":  # one U hub on every V, every V also on one leaf U
        g = _graph(9, 8, [(0, j) for j in range(8)] + [(1 + j, j) for j in range(8)])
    elif name == "star_v":
        g = _graph(8, 9, [(i, 0) for i in range(8)] + [(i, 1 + i) for i in range(8)])
    elif name == "extreme_weights":
        g = _graph(4, 3, [(0, 0), (1, 0), (1, 1), (2, 1), (2, 2), (3, 2)], [1e-6, 1e6, 1.0, 1e-6, 1e6, 1.0])
    else:  # a path u0 - v0 - u1 - v1 - ... - u7
        g = _graph(8, 7, [(i, i) for i in range(7)] + [(i + 1, i) for i in range(7)])
    Pi = dense_pi(g)
    meta = bh.build_index_meta(g, ALPHA)
    srcs = np.arange(g.u_count)
    for eps in (0.5, 1e-3, 1e-6, 1e-9):
        for dtype, tol in (("fp64", 1e-10), ("fp32", 1e-5)):
            res = bh.bhpp_query_batch(g, meta, srcs, eps, k=3, dtype=dtype, return_scores=True)
            for j, q in enumerate(srcs):
                diff = (Pi[q, :] + Pi[:, q]) - res.scores[j]
                assert diff.min() >= -tol and diff.max() <= eps + tol, (name, eps, dtype, int(q), diff)
        # the single-query path against the oracle (the reference restated bit for bit)
        eps_b = float(meta.eps_split_policy(eps))
        og = O.OracleGraph(g)
        for q in range(min(g.u_count, 3)):
            ref_scores, ref_tr = og.bhpp_query(q, ALPHA, meta.lam, eps_b, eps - eps_b)
            one = bh.bhpp_query(g, meta, q, eps, tie_skip=O.tie_skip_for(ref_tr["forward"]))
            np.testing.assert_allclose(one.scores, ref_scores, atol=1e-12, rtol=0, err_msg=f"{name} {eps} {q}")
            assert one.phase_trace["backward"] == ref_tr["backward"], (name, eps, q)


@pytest.mark.parametrize("slots", [32, 64, 128])
def test_wide_engine_on_tiny_graphs(slots, monkeypatch):
    """The wide slot engine (row-flag pulls, 32+ slots) on graphs smaller than one warp range
    or one 32-edge tile: a single U node, stars, a path, and a handful of random graphs, with
    the small-graph path switched off.  One-sided against the dense solve like criterion 1."""
    monkeypatch.setenv("BH_NO_SMALL", "1")
    graphs = [
        _graph(1, 3, [(0, 0), (0, 1), (0, 2)], [1.0, 2.0, 3.0]),
        _graph(9, 8, [(0, j) for j in range(8)] + [(1 + j, j) for j in range(8)]),
        _graph(8, 9, [(i, 0) for i in range(8)] + [(i, 1 + i) for i in range(8)]),
        _graph(8, 7, [(i, i) for i in range(7)] + [(i + 1, i) for i in range(7)]),
    ]
    rng = substream(2027, "wide-tiny")
    for _ in range(6):
        nu, nv = (int(x) for x in rng.integers(3, 80, size=2))
        graphs.append(random_bigraph(rng, nu, nv, float(rng.uniform(0.5, 3.0)), 10.0))
    for gi, g in enumerate(graphs):
        Pi = dense_pi(g)
        meta = bh.build_index_meta(g, ALPHA)
        srcs = np.arange(g.u_count)
        for eps in (1e-2, 1e-7):
            for dtype, tol in (("fp64", 1e-10), ("fp32", 1e-5)):
                res = bh.bhpp_query_batch(g, meta, srcs, eps, k=min(3, g.u_count), dtype=dtype, return_scores=True,
                                          slots=slots)
                for j, q in enumerate(srcs):
                    diff = (Pi[q, :] + Pi[:, q]) - res.scores[j]
                    assert diff.min() >= -tol and diff.max() <= eps + tol, (gi, slots, eps, dtype, int(q), diff)
