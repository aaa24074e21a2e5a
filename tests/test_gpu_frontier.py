"""GPU: frontier rounds (K-F, csrc/frontier.cuh) against the reference.

The reference runs a round's push / flush half as a scatter over the pushed
rows' edges when they touch at most ``_SCATTER_LIMIT * |E|`` edges, and as a
dense matvec otherwise (pkg/src/bipush/push_engine.py:44, 269-277, 294-324);
its own test forces either path by monkeypatching the constant and checks they
agree (pkg/tests/test_push_engine.py:187-202).  The engine mirrors the
constant (``push_engine._SCATTER_LIMIT``): -1 forces dense rounds, >= 1 forces
frontier rounds whenever no slot is in power iteration; the default (0.01)
applies to blocks of up to 16 slots (wider blocks run dense rounds, see
frontier.cuh).  Every mode must meet
the same bar against the reference fixtures: fp64 scores within 1e-9 and
identical integer traces, fp32 top-k within 1e-5 relative.
"""

import numpy as np
import pytest

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import _capi
from paper_2312_06724_b200 import push_engine as pe
from golden_io import config_graph, graph_from, load, split_traces, trace_dict
from test_gpu_parity import ATOL64, RTOL32, assert_traces, tie_skip_from, topk_equal_up_to_ties

pytestmark = pytest.mark.gpu

FORCE_DENSE, DEFAULT, FORCE_FRONTIER = -1.0, pe._SCATTER_LIMIT, 10.0


def _stats(g, dtype):
    return _capi.device_graph(g, dtype).last_run_stats()


@pytest.mark.parametrize("limit", [FORCE_DENSE, DEFAULT, FORCE_FRONTIER])
@pytest.mark.parametrize("slots", [1, 4, 64])
@pytest.mark.parametrize("eager", [False, True])
def test_scaled_c2_every_mode(limit, slots, eager, monkeypatch):
    """c2 at 1/10 scale: golden fp64 scores / traces and fp32 top-k in every
    mode, slot width and launch form; forced modes run the rounds they name."""
    monkeypatch.setattr(pe, "_SCATTER_LIMIT", limit)
    if eager:
        monkeypatch.setenv("BH_NO_GRAPH", "1")
    d = load("c2s")
    g = config_graph("c2s")
    meta = bh.build_index_meta(g, 0.15)
    n = min(len(d["sources"]), 6 if slots > 1 else 3)
    srcs = d["sources"][:n]
    ties = np.array([tie_skip_from(t) for t in d["ties"][:n]], dtype=np.int32)
    k = int(d["k"])
    eps = float(d["eps"])
    r64 = bh.bhpp_query_batch(g, meta, srcs, eps, k=k, dtype="fp64", return_scores=True, tie_skip=ties,
                              slots=slots)
    st = _stats(g, "fp64")
    if limit == FORCE_DENSE:
        assert st["frontier_rounds"] == 0
    elif limit == FORCE_FRONTIER:
        assert st["frontier_rounds"] > 0 and st["frontier_u_rounds"] > 0, st
    for i in range(n):
        np.testing.assert_allclose(r64.scores[i], d["scores"][i], atol=ATOL64, rtol=0)
        back, fwd, gamma = split_traces(d["traces"][i])
        assert_traces(r64.trace_dicts(i), back, fwd, gamma)
    r32 = bh.bhpp_query_batch(g, meta, srcs, eps, k=k, dtype="fp32", tie_skip=ties, slots=slots)
    for i in range(n):
        ref, exp = d["scores"][i], d["topk"][i]
        np.testing.assert_allclose(r32.topk_score[i], ref[exp], rtol=RTOL32, atol=eps)
        topk_equal_up_to_ties(r32.topk_index[i], r32.topk_score[i], exp, ref, RTOL32, eps)


@pytest.mark.parametrize("limit", [FORCE_DENSE, FORCE_FRONTIER])
def test_scaled_c4_hub_rows_split(limit, monkeypatch):
    """c4 at 1/100 scale has V hubs of ~1e4 edges: in frontier rounds they are
    split into FRONT_CHUNK-edge items whose partials the last item adds."""
    monkeypatch.setattr(pe, "_SCATTER_LIMIT", limit)
    d = load("c4s")
    g = config_graph("c4s")
    assert int(np.diff(g.v_indptr).max()) > 2048
    meta = bh.build_index_meta(g, 0.2)
    srcs = d["sources"]
    ties = np.array([tie_skip_from(t) for t in d["ties"]], dtype=np.int32)
    k = int(d["k"])
    for slots in (1, 32):
        res = bh.bhpp_query_batch(g, meta, srcs, float(d["eps"]), k=k, dtype="fp64", return_scores=True,
                                  tie_skip=ties, slots=slots)
        if limit > 0:
            assert _stats(g, "fp64")["frontier_rounds"] > 0
        for i in range(len(srcs)):
            np.testing.assert_allclose(res.scores[i], d["scores"][i], atol=ATOL64, rtol=0)
            back, fwd, gamma = split_traces(d["traces"][i])
            assert_traces(res.trace_dicts(i), back, fwd, gamma)


@pytest.mark.parametrize("limit", [FORCE_DENSE, FORCE_FRONTIER])
def test_small_graphs_single_kernels(limit, monkeypatch):
    """The 40 reference-generated small graphs: ss_push and selective_push
    (one-slot engine) in both modes against the golden ledgers and traces."""
    monkeypatch.setattr(pe, "_SCATTER_LIMIT", limit)
    d = load("small")
    for i in range(int(d["count"])):
        p = f"g{i}_"
        g = graph_from(d, p)
        alpha, eps, q, _limit, lam, tau, mu = d[p + "params"]
        q = int(q)
        eb = bh.choose_eps_b(eps, mu)
        ss = bh.ss_push(g, q, alpha, eb)
        np.testing.assert_allclose(ss.ledger.estimate, d[p + "ss_est"], atol=1e-12, rtol=0, err_msg=p)
        np.testing.assert_allclose(ss.ledger.residue_u, d[p + "ss_res"], atol=1e-12, rtol=0, err_msg=p)
        assert {**ss.phase_trace, "terminated_by": ss.terminated_by} == trace_dict(d[p + "ss_trace"], False)
        sel = bh.selective_push(g, q, alpha, max(eb, 1e-7))
        np.testing.assert_allclose(sel.ledger.estimate, d[p + "sel_est"], atol=1e-12, rtol=0, err_msg=p)
        assert {**sel.phase_trace, "terminated_by": sel.terminated_by} == trace_dict(d[p + "sel_trace"], False)


def test_scatter_and_matrix_paths_agree(monkeypatch):
    """pkg/tests/test_push_engine.py:187-202 on the engine: ss_push with every
    round in frontier form equals ss_push with every round dense (1e-13, equal
    n_p and traces), on the c1 graph from several sources."""
    g = config_graph("c1")
    out = {}
    for limit in (FORCE_DENSE, FORCE_FRONTIER):
        monkeypatch.setattr(pe, "_SCATTER_LIMIT", limit)
        out[limit] = [bh.ss_push(g, q, 0.15, 1e-6) for q in (0, 3, 17, 400)]
    for a, b in zip(out[FORCE_DENSE], out[FORCE_FRONTIER]):
        np.testing.assert_allclose(a.ledger.estimate, b.ledger.estimate, atol=1e-13, rtol=0)
        np.testing.assert_allclose(a.ledger.residue_u, b.ledger.residue_u, atol=1e-13, rtol=0)
        assert a.ledger.n_p == b.ledger.n_p
        assert a.phase_trace == b.phase_trace and a.terminated_by == b.terminated_by


def test_frontier_rounds_are_deterministic(monkeypatch):
    """Work items are appended in atomic order, but every row is summed by one
    warp (or its chunks added in order): repeated runs are bitwise equal."""
    monkeypatch.setattr(pe, "_SCATTER_LIMIT", FORCE_FRONTIER)
    g = config_graph("c2s")
    meta = bh.build_index_meta(g, 0.15)
    srcs = load("c2s")["sources"][:6]
    a = bh.bhpp_query_batch(g, meta, srcs, 1e-7, k=50, dtype="fp32", return_scores=True, slots=16)
    b = bh.bhpp_query_batch(g, meta, srcs, 1e-7, k=50, dtype="fp32", return_scores=True, slots=16)
    np.testing.assert_array_equal(a.scores, b.scores)
    assert a.traces.tobytes() == b.traces.tobytes()


@pytest.mark.parametrize("name", ["c2s", "c4s"])
def test_row_pointer_pull_fallback(name, monkeypatch):
    """The dense pull that walks row pointers (k_pull_sw) serves device stores
    without the flagged edge stream; BH_PULL=sw selects it when an engine is
    built.  A fresh graph object (so a fresh store and engines) must meet the
    same bar against the golden fixtures as the default row-flag pull, and the
    two pulls must agree on the fp64 scores to summation-order noise."""
    from golden_io import _CFG
    from paper_2312_06724_b200.synth import make_graph

    d = load(name)
    g_rf = config_graph(name)
    monkeypatch.setenv("BH_PULL", "sw")
    g = graph_from(d) if "eu" in d else make_graph(_CFG[name])  # not the cached object: new store, new engines
    assert g.fingerprint == str(d["fingerprint"])
    alpha = _CFG[name].alpha
    meta = bh.build_index_meta(g, alpha)
    n = min(len(d["sources"]), 6)
    srcs = d["sources"][:n]
    ties = np.array([tie_skip_from(t) for t in d["ties"][:n]], dtype=np.int32)
    k, eps = int(d["k"]), float(d["eps"])
    r_sw = bh.bhpp_query_batch(g, meta, srcs, eps, k=k, dtype="fp64", return_scores=True, tie_skip=ties, slots=64)
    monkeypatch.delenv("BH_PULL")
    meta_rf = bh.build_index_meta(g_rf, alpha)
    r_rf = bh.bhpp_query_batch(g_rf, meta_rf, srcs, eps, k=k, dtype="fp64", return_scores=True, tie_skip=ties,
                               slots=64)
    for i in range(n):
        np.testing.assert_allclose(r_sw.scores[i], d["scores"][i], atol=ATOL64, rtol=0)
        np.testing.assert_allclose(r_sw.scores[i], r_rf.scores[i], atol=1e-13, rtol=0)
        back, fwd, gamma = split_traces(d["traces"][i])
        assert_traces(r_sw.trace_dicts(i), back, fwd, gamma)


def test_value_underflow_falls_back_to_row_pointer_pull():
    """The row-flag pull reads a row's end from the sign of the edge value, so the store
    builds its flagged edge stream only when every prescaled value is positive in the store's
    type.  A weight that underflows to zero in fp32 (1e-60 against sums of order 10) must make
    the fp32 store fall back to the row-pointer pull; fp64 keeps the flagged stream.  Both must
    agree with each other like any fp32 / fp64 pair."""
    d = load("c2s")
    g0 = config_graph("c2s")
    eu = np.repeat(np.arange(g0.u_count), np.diff(g0.u_indptr))
    ew = np.array(g0.u_weights, dtype=np.float64)
    ew[::97] = 1e-60  # many rows end in, start with or contain an underflowing value
    g = bh.BipartiteGraph.from_arrays(g0.u_count, g0.v_count, eu, np.array(g0.u_indices), ew)
    meta = bh.build_index_meta(g, 0.15)
    srcs = d["sources"][:6]
    k, eps = int(d["k"]), float(d["eps"])
    r64 = bh.bhpp_query_batch(g, meta, srcs, eps, k=k, dtype="fp64", return_scores=True, slots=64)
    r32 = bh.bhpp_query_batch(g, meta, srcs, eps, k=k, dtype="fp32", slots=64)
    for i in range(len(srcs)):
        assert np.isfinite(r64.scores[i]).all()
        ref = r64.scores[i]
        np.testing.assert_allclose(r32.topk_score[i], ref[r32.topk_index[i]], rtol=RTOL32, atol=eps)
        topk_equal_up_to_ties(r32.topk_index[i], r32.topk_score[i], r64.topk_index[i], ref, RTOL32, eps)


@pytest.mark.parametrize("geo", ["0", "1", "2"])
def test_row_flag_pull_geometries(geo, monkeypatch):
    """Every compiled geometry of the row-flag pull (BH_RF_GEO: 8 rows in flight at 3 or 2 blocks of
    8 warps, or 4 blocks of 7 warps per SM; the defaults pick one per lane width) meets the golden
    bar on c4 at 1/100 scale (hub rows cut across warps) in fp64 and fp32."""
    from golden_io import _CFG
    from paper_2312_06724_b200.synth import make_graph

    monkeypatch.setenv("BH_RF_GEO", geo)
    d = load("c4s")
    g = graph_from(d) if "eu" in d else make_graph(_CFG["c4s"])  # fresh store and engines
    meta = bh.build_index_meta(g, _CFG["c4s"].alpha)
    srcs = d["sources"]
    ties = np.array([tie_skip_from(t) for t in d["ties"]], dtype=np.int32)
    k, eps = int(d["k"]), float(d["eps"])
    r64 = bh.bhpp_query_batch(g, meta, srcs, eps, k=k, dtype="fp64", return_scores=True, tie_skip=ties, slots=64)
    r32 = bh.bhpp_query_batch(g, meta, srcs, eps, k=k, dtype="fp32", tie_skip=ties, slots=64)
    for i in range(len(srcs)):
        np.testing.assert_allclose(r64.scores[i], d["scores"][i], atol=ATOL64, rtol=0)
        back, fwd, gamma = split_traces(d["traces"][i])
        assert_traces(r64.trace_dicts(i), back, fwd, gamma)
        ref, exp = d["scores"][i], d["topk"][i]
        np.testing.assert_allclose(r32.topk_score[i], ref[exp], rtol=RTOL32, atol=eps)
        topk_equal_up_to_ties(r32.topk_index[i], r32.topk_score[i], exp, ref, RTOL32, eps)
