"""Baselines on the device kernels (reference baselines.py): PISP against the
oracle composition, MCSP / monte_carlo against their error bounds."""

import time
from pathlib import Path

import numpy as np
import pytest

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import BipartiteGraph
from golden_io import config_graph, load
from oracle import cpu_oracle as O

pytestmark = pytest.mark.gpu


def test_pisp_query_matches_oracle_composition():
    g = config_graph("c1")
    og = O.OracleGraph(g)
    for q, eps in ((0, 1e-4), (17, 1e-6)):
        r = bh.pisp_query(g, q, 0.15, eps)
        depth = O.required_iterations(0.15, eps / 2, 1.0)
        start = np.zeros(g.u_count)
        start[q] = 1.0
        fwd = og.power_iteration(start, 0.15, depth)
        led, tr = og.ss_push(q, 0.15, eps / 2, budget=False)
        np.testing.assert_allclose(r.scores, fwd + led["estimate"], atol=1e-12)
        assert r.phase_trace["forward"]["power_iterations"] == depth
        assert r.phase_trace["backward"]["selective_rounds"] == tr["selective_rounds"]
        assert r.method == "pisp"


def test_monte_carlo_within_its_bound():
    """Walk frequencies vs the exact forward HPP row: |error| <= eps_f entrywise
    (holds with probability >= 1 - p_f), frequencies sum to one, reproducible."""
    g = config_graph("c1")
    og = O.OracleGraph(g)
    alias = bh.build_alias(g)
    start = np.zeros(g.u_count)
    start[5] = 1.0
    exact = og.power_iteration(start, 0.15, 400)  # converged forward scores
    eps_f = 5e-3
    est = bh.monte_carlo(g, alias, 5, 0.15, eps_f, 1e-6, seed=7)
    assert est.sum() == pytest.approx(1.0, abs=1e-12)
    assert np.abs(est - exact).max() <= eps_f
    again = bh.monte_carlo(g, alias, 5, 0.15, eps_f, 1e-6, seed=7, batch_size=100_000)
    np.testing.assert_array_equal(est, again)  # walk i uses stream (seed, i) whatever the batching
    other = bh.monte_carlo(g, alias, 5, 0.15, eps_f, 1e-6, seed=8)
    assert not np.array_equal(est, other)


def test_mcsp_query_two_sided_bound_and_deadline():
    d = load("c1")
    g = config_graph("c1")
    alias = bh.build_alias(g)
    truth = d["scores"][0]  # reference bhpp_query at eps 1e-6 for source u0: within 1e-6 of the true score
    eps = 0.02
    r = bh.mcsp_query(g, alias, 0, 0.15, eps, p_f=1e-6, seed=3)
    assert np.abs(r.scores - truth).max() <= eps + 1e-6
    assert r.method == "mcsp" and r.phase_trace["forward"]["n_walks"] == bh.mc_walk_count(eps / 2, 1e-6, g.u_count)
    with pytest.raises(bh.DeadlineExceeded):
        bh.mcsp_query(g, alias, 0, 0.15, 1e-3, deadline=time.perf_counter() - 1.0)


def test_similarity_rows_batched_prefetch_matches_single_queries():
    """evalkit's row factory (evalkit.py:270-308) on the batched engine: one
    prefetch call, rows equal to per-node bhpp_query scores; memoised."""
    g = config_graph("c1")
    meta = bh.build_index_meta(g, 0.15)
    row = bh.similarity_rows("ssbipush", g, meta, epsilon=1e-6)
    nodes = [0, 17, 5, 17, 999]
    row.prefetch(nodes)
    assert sorted(row.cache) == [0, 5, 17, 999]
    for ui in (0, 17, 999):
        np.testing.assert_allclose(row(ui), bh.bhpp_query(g, meta, ui, 1e-6).scores, atol=1e-12, rtol=0)
    first = row(5)
    assert row(5) is first  # memoised
    extra = row(3)          # uncached node: a batch of one
    np.testing.assert_allclose(extra, bh.bhpp_query(g, meta, 3, 1e-6).scores, atol=1e-12, rtol=0)


def test_build_alias_matches_reference_tables():
    """build_alias (baselines.py:41-77) on the device (bh_alias_build): identical tables on the config-1
    graph and on a non-integer-weight graph (Vose pairing order, roundoff leftovers)."""
    d = np.load(Path(__file__).resolve().parent / "golden" / "alias.npz")
    g1 = config_graph("c1")
    g2 = BipartiteGraph([f"a{i}" for i in range(60)], [f"b{i}" for i in range(int(d["w_ev"].max()) + 1)],
                        d["w_eu"], d["w_ev"], d["w_ew"])
    for name, g in (("c1", g1), ("w", g2)):
        t = bh.build_alias(g)
        for side in ("u", "v"):
            np.testing.assert_array_equal(getattr(t, f"{side}_prob"), d[f"{name}_{side}_prob"])
            np.testing.assert_array_equal(getattr(t, f"{side}_alias"), d[f"{name}_{side}_alias"])
