"""Batched callers (callers.py) after the reference CLI's _run_query / cmd_bench
(cli.py:360-369, 410-521): host logic on CPU, the rows on the GPU."""

import numpy as np
import pytest

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import callers
from paper_2312_06724_b200.synth import bench_sources, make_graph


def test_bench_queries_follow_the_reference_sampler():
    g = make_graph("c1")
    np.testing.assert_array_equal(callers.bench_queries(g, 17), bench_sources(g.u_count, 17))
    every = callers.bench_queries(g, 10**6)  # clipped to |U|: a permutation of U
    assert sorted(every) == list(range(g.u_count))


def test_unknown_method_is_rejected_like_the_cli():
    g = make_graph("c1")
    with pytest.raises(ValueError, match="unknown method"):
        callers.run_query(g, None, "nope", 0, 1e-4)
    with pytest.raises(ValueError, match="unknown method"):
        callers.bench_rows(g, None, methods=("ssbipush", "nope"))


@pytest.mark.gpu
def test_bench_rows_on_the_device():
    g = make_graph("c1")
    meta = bh.build_index_meta(g, 0.15)
    rows, excluded = callers.bench_rows(g, meta, methods=("ssbipush", "pisp"), epsilons=(1e-4, 1e-5), queries=6)
    assert not excluded
    timing = [r for r in rows if r["kind"] == "timing"]
    agree = [r for r in rows if r["kind"] == "agreement"]
    assert [(r["method"], r["epsilon"]) for r in timing] == [("ssbipush", 1e-4), ("pisp", 1e-4),
                                                              ("ssbipush", 1e-5), ("pisp", 1e-5)]
    assert all(r["n"] == 6 and r["mean_s"] > 0 for r in timing)
    assert timing[0]["batched"] and timing[0]["stddev_s"] is None and timing[1]["stddev_s"] is not None
    assert len(agree) == 2 and all(r["within"] for r in agree), agree
    # the batched ssbipush rows equal per-source bhpp_query (the reference's loop)
    q = callers.bench_queries(g, 6)
    one = bh.bhpp_query(g, meta, q[2], 1e-4)
    res = bh.bhpp_query_batch(g, meta, q, 1e-4, k=None, dtype="fp64", return_scores=True)
    np.testing.assert_allclose(res.scores[2], one.scores, atol=1e-12, rtol=0)
    r = callers.run_query(g, meta, "ssbipush", q[2], 1e-4)
    np.testing.assert_allclose(r.scores, one.scores, atol=1e-15, rtol=0)
