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
