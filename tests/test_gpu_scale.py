"""GPU parity at the BASELINE configuration sizes, against the live C oracle.

config 2 (|U|=1e5, |V|=2e5, |E|=2e6, eps=1e-7) at full size on a sample of the
bench sources; batch semantics (slot refill with more sources than slots,
exclusion, k clipping, duplicate sources); power iteration and lambda.
"""

import os

import numpy as np
import pytest

import paper_2312_06724_b200 as bh
from golden_io import config_graph, load
from oracle import cpu_oracle as O
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    g = make_graph("c2")
    meta = bh.build_index_meta(g, 0.15)
    og = O.OracleGraph(g)
    src = bench_sources(g.u_count, 64)[:8]
    eps = 1e-7
    eb = meta.eps_split_policy(eps)
    ref = og.bhpp_query_many(src, 0.15, meta.lam, eb, eps - eb, threads=os.cpu_count())
    return g, meta, og, src, eps, ref


def test_c2_lambda_matches_oracle(c2):
    g, meta, og, *_ = c2
    om = O.index_meta(g, 0.15)
    assert meta.tau == om["tau"] and meta.mu == om["mu"]
    assert meta.lam == pytest.approx(om["lam"], rel=1e-12)


def test_c2_full_size_fp64_parity(c2):
    g, meta, og, src, eps, ref = c2
    ties = np.array([O.tie_skip_for(tr["forward"]) for _, tr in ref], dtype=np.int32)
    res = bh.bhpp_query_batch(g, meta, src, eps, k=50, dtype="fp64", return_scores=True, tie_skip=ties)
    for i, (scores, tr) in enumerate(ref):
        assert np.abs(res.scores[i] - scores).max() <= 1e-9
        got = res.trace_dicts(i)
        assert got["backward"] == tr["backward"]
        fwd = {k: v for k, v in tr["forward"].items() if k not in ("tie_checks", "tie_break_at", "gamma")}
        assert {k: v for k, v in got["forward"].items() if k != "gamma"} == fwd
        assert got["forward"]["gamma"] == pytest.approx(tr["forward"]["gamma"], rel=1e-12)
        top = O.topk_indices(scores, 50)
        diff = res.topk_index[i] != top
        if diff.any():  # only exact score ties may reorder
            assert np.abs(scores[res.topk_index[i][diff]] - scores[top[diff]]).max() <= 1e-12


def test_c2_full_size_fp32_parity(c2):
    g, meta, og, src, eps, ref = c2
    res = bh.bhpp_query_batch(g, meta, src, eps, k=50, dtype="fp32")
    for i, (scores, tr) in enumerate(ref):
        top = O.topk_indices(scores, 50)
        np.testing.assert_allclose(res.topk_score[i], scores[top], rtol=1e-5, atol=eps)
        kth = scores[top[-1]]
        diff = res.topk_index[i] != top
        if diff.any():
            assert np.abs(scores[res.topk_index[i][diff]] - scores[top[diff]]).max() <= 1e-5 * kth + eps


def test_refill_many_sources_few_slots():
    """More sources than slots: finished slots are refilled on device; every
    query must match its own single-query run."""
    d = load("c2s")
    g = config_graph("c2s")
    meta = bh.build_index_meta(g, 0.15)
    src = np.random.default_rng(7).choice(g.u_count, 40, replace=False)
    src = np.concatenate([src, src[:3]])  # duplicates are independent queries
    many = bh.bhpp_query_batch(g, meta, src, 1e-7, k=20, dtype="fp64", return_scores=True, slots=16)
    for i in (0, 5, 17, 39, 40, 42):
        one = bh.bhpp_query(g, meta, int(src[i]), 1e-7)
        assert np.abs(many.scores[i] - one.scores).max() <= 1e-12
        assert many.trace_dicts(i)["backward"] == one.phase_trace["backward"]
    np.testing.assert_array_equal(many.topk_index[40], many.topk_index[0])
    assert d["n"][0] == g.u_count


def test_batch_exclude_and_clipping():
    d = load("c1")
    g = config_graph("c1")
    meta = bh.build_index_meta(g, 0.15)
    src = d["sources"][:6]
    ties = np.array([t[1] - 1 if t[1] else t[0] for t in d["ties"][:6]], dtype=np.int32)
    res = bh.bhpp_query_batch(g, meta, src, float(d["eps"]), k=10, exclude_query=True, dtype="fp64", tie_skip=ties)
    for i in range(6):
        assert int(src[i]) not in res.topk_index[i]
        np.testing.assert_array_equal(res.topk_index[i], d["topk_ex"][i])
    tiny = bh.BipartiteGraph(["a", "b", "c"], ["x", "y"], [0, 1, 2, 0], [0, 0, 1, 1], [1.0, 2.0, 1.0, 1.0])
    tm = bh.build_index_meta(tiny, 0.15)
    r = bh.bhpp_query_batch(tiny, tm, [0, 1, 2], 1e-6, k=50, dtype="fp64", return_scores=True)
    assert r.k == 3 and (r.topk_index >= 0).all()
    for i in range(3):
        order = np.argsort(-r.scores[i], kind="stable")
        np.testing.assert_array_equal(r.topk_index[i], order)
    r0 = bh.bhpp_query_batch(tiny, tm, [0, 1], 1e-6, k=0, dtype="fp64")
    assert r0.topk_index.shape == (2, 0)


def test_power_iteration_batch_and_lambda():
    g = config_graph("c1")
    og = O.OracleGraph(g)
    rng = np.random.default_rng(3)
    starts = rng.random((5, g.u_count))
    for t in (0, 1, 17):
        got = bh.power_iteration(g, starts, 0.2, t)
        for i in range(5):
            np.testing.assert_allclose(got[i], og.power_iteration(starts[i], 0.2, t), rtol=1e-12, atol=1e-15)
    ref = O.index_meta(g, 0.15)
    assert bh.estimate_lambda(g, 0.15, ref["tau"]) == pytest.approx(ref["lam"], rel=1e-12)


@pytest.mark.parametrize("cfg", ["c4s"])
def test_scaled_config_refill_fp32_consistent(cfg):
    """fp32 and fp64 engines agree on the scaled hub-skewed config (1e-5 rel on top-k)."""
    g = config_graph(cfg)
    c = CONFIGS["c4"]
    meta = bh.build_index_meta(g, c.alpha)
    src = bench_sources(g.u_count, 24)
    a = bh.bhpp_query_batch(g, meta, src, 1e-6, k=20, dtype="fp64", return_scores=True)
    b = bh.bhpp_query_batch(g, meta, src, 1e-6, k=20, dtype="fp32", slots=16)
    for i in range(len(src)):
        np.testing.assert_allclose(b.topk_score[i], a.scores[i][a.topk_index[i]], rtol=1e-5, atol=1e-6)


def test_async_submit_and_gate_match_sync():
    """BH_QUERY_ASYNC + bh_query_wait and the measurement gate give the sync results."""
    import ctypes as C

    import torch

    from paper_2312_06724_b200 import _capi
    from paper_2312_06724_b200.bhpp_query import query_batch_device, query_wait

    g = config_graph("c2s")
    meta = bh.build_index_meta(g, 0.15)
    src = load("c2s")["sources"][:8]
    ref = bh.bhpp_query_batch(g, meta, src, 1e-7, k=20, dtype="fp32")
    dg = _capi.device_graph(g, "fp32")
    eb = meta.eps_split_policy(1e-7)
    dev = torch.device("cuda:0")
    st = torch.cuda.Stream(device=dev)
    s_t = torch.from_numpy(np.asarray(src, dtype=np.int32)).to(dev)
    ti = torch.empty((len(src), 20), dtype=torch.int32, device=dev)
    ts = torch.empty((len(src), 20), dtype=torch.float64, device=dev)
    tr = torch.empty((len(src), _capi.TRACE_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    gate = torch.zeros(1, dtype=torch.int32).pin_memory()
    _capi.check(_capi.lib().bh_stream_gate(C.c_void_p(st.cuda_stream), C.c_void_p(gate.data_ptr())))
    query_batch_device(dg, meta, eb, 1e-7 - eb, s_t.data_ptr(), len(src), 20, ti.data_ptr(), ts.data_ptr(),
                       tr.data_ptr(), stream=st.cuda_stream, async_=True)
    gate[0] = 1
    query_wait(dg)
    np.testing.assert_array_equal(ti.cpu().numpy(), ref.topk_index)
    np.testing.assert_array_equal(ts.cpu().numpy(), ref.topk_score)
    assert tr.cpu().numpy().tobytes() == ref.traces.tobytes()
    # an async batch left unwaited is completed by the next call on the graph
    query_batch_device(dg, meta, eb, 1e-7 - eb, s_t.data_ptr(), len(src), 20, ti.data_ptr(), ts.data_ptr(),
                       tr.data_ptr(), stream=st.cuda_stream, async_=True)
    again = bh.bhpp_query_batch(g, meta, src, 1e-7, k=20, dtype="fp32")
    np.testing.assert_array_equal(again.topk_index, ref.topk_index)
    np.testing.assert_array_equal(ti.cpu().numpy(), ref.topk_index)


def test_single_process_multi_device_sharding_matches_one_call():
    """bhpp_query_multi merges interleaved shards back into source order; with
    the devices of this box (here one GPU listed three times) it must equal one call."""
    from paper_2312_06724_b200.distributed import bhpp_query_multi

    g = config_graph("c2s")
    meta = bh.build_index_meta(g, 0.15)
    src = np.random.default_rng(11).choice(g.u_count, 13, replace=False)
    # same slot width everywhere -> same engine plan -> bitwise-equal per-query results
    one = bh.bhpp_query_batch(g, meta, src, 1e-7, k=20, dtype="fp32", return_scores=True, slots=16)
    multi = bhpp_query_multi(g, meta, src, 1e-7, k=20, dtype="fp32", devices=[0, 0, 0], return_scores=True,
                             slots=16)
    np.testing.assert_array_equal(multi.topk_index, one.topk_index)
    np.testing.assert_array_equal(multi.topk_score, one.topk_score)
    np.testing.assert_array_equal(multi.scores, one.scores)
    assert multi.traces.tobytes() == one.traces.tobytes()


def test_batch_edge_cases_duplicates_empty_labels_and_limits():
    """Duplicate sources give identical rows; an empty batch returns empty
    arrays; labels and indices mix; k is clipped to |U|; bad sources and eps
    raise ValueError / DataError like the reference's argument checks."""
    g = config_graph("c1")
    meta = bh.build_index_meta(g, 0.15)
    src = [5, 17, 5, 5, 17]
    r = bh.bhpp_query_batch(g, meta, src, 1e-6, k=10, dtype="fp64", return_scores=True)
    np.testing.assert_array_equal(r.scores[0], r.scores[2])
    np.testing.assert_array_equal(r.scores[0], r.scores[3])
    np.testing.assert_array_equal(r.scores[1], r.scores[4])
    np.testing.assert_array_equal(r.topk_index[0], r.topk_index[3])
    assert r.traces.tobytes()[: r.traces.itemsize] == r.traces[2:3].tobytes()
    lab = bh.bhpp_query_batch(g, meta, [g.u_labels[5], 17], 1e-6, k=10, dtype="fp64", return_scores=True)
    np.testing.assert_allclose(lab.scores[0], r.scores[0], atol=1e-15, rtol=0)  # other slot width
    np.testing.assert_allclose(lab.scores[1], r.scores[1], atol=1e-15, rtol=0)
    e = bh.bhpp_query_batch(g, meta, np.array([], dtype=np.int64), 1e-6, k=10, dtype="fp32")
    assert e.topk_index.shape[0] == 0 and e.traces.shape[0] == 0
    big = bh.bhpp_query_batch(g, meta, [0], 1e-6, k=2000, dtype="fp32")  # k clipped to |U| like topk
    assert big.k == g.u_count and big.topk_index.shape == (1, g.u_count)
    with pytest.raises(ValueError):
        bh.bhpp_query_batch(g, meta, [g.u_count], 1e-6, k=10, dtype="fp32")
    with pytest.raises(ValueError):
        bh.bhpp_query_batch(g, meta, [0], -1.0, k=10, dtype="fp32")
    with pytest.raises(bh.DataError):
        bh.bhpp_query_batch(g, meta, ["no-such-label"], 1e-6, k=10, dtype="fp32")
