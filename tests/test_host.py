"""CPU tests: the C ABI boundary, the host-side graph mirror and parameter logic.

No compute runs here without a GPU: the library is only loaded and probed.
"""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2312_06724_b200 as bh
from golden_io import config_graph, graph_from, load
from paper_2312_06724_b200 import _capi
from paper_2312_06724_b200.bigraph import BipartiteGraph, DataError, IndexLabels
from paper_2312_06724_b200.rng import substream
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, chung_lu_edges, make_graph, scaled_config

HEADER = Path(__file__).resolve().parents[1] / "include" / "bhpp.h"


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(bh_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert {"bh_graph_create", "bh_query_batch", "bh_push_run", "bh_topk"} <= set(names)
    lib = _capi.lib()
    for name in names:
        assert hasattr(lib, name), f"libbhpp.so does not export {name}"
    assert set(_capi.EXPORTS) == set(names)
    assert lib.bh_version() == 3


def test_struct_layouts_match_header():
    import ctypes as C

    assert C.sizeof(_capi.Trace) == 96
    assert C.sizeof(_capi.QueryParams) == 56
    assert C.sizeof(_capi.GraphInfo) == 56
    assert C.sizeof(_capi.RunStats) == 80
    assert _capi.TRACE_DTYPE.itemsize == C.sizeof(_capi.Trace)


def test_calls_fail_loudly_without_gpu(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = make_graph("c1")
    with pytest.raises(RuntimeError):
        bh.build_index_meta(g)
    res = bh.QueryResult("x", 0, np.array([0.5, 0.25]), 1e-3, 5e-4, 5e-4, {}, {}, ["a", "b"])
    with pytest.raises(RuntimeError):
        bh.topk(res, 1)


def test_missing_library_raises(monkeypatch, tmp_path):
    monkeypatch.setattr(_capi, "_lib", None)
    monkeypatch.setattr(_capi, "LIB_PATH", tmp_path / "nope.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _capi.lib()


# -- graph mirror -----------------------------------------------------------------

def test_graph_matches_golden_fingerprints():
    for name in ("c1", "c2s", "c4s"):
        g = config_graph(name)  # asserts the fingerprint inside
        assert g.fingerprint == str(load(name)["fingerprint"])


def test_graph_csr_invariants_and_roundtrip():
    g = config_graph("c1")
    assert g.u_indptr[-1] == g.v_indptr[-1] == g.edge_count
    assert (np.diff(g.u_indptr) == g.deg_u).all() and (g.deg_u >= 1).all() and (g.deg_v >= 1).all()
    eu = np.repeat(np.arange(g.u_count), g.deg_u)
    assert np.allclose(np.bincount(eu, weights=g.u_weights), g.ws_u)
    # V-CSR is the transpose of U-CSR
    k_u = np.sort(eu * g.v_count + g.u_indices)
    ev = np.repeat(np.arange(g.v_count), g.deg_v)
    k_v = np.sort(g.v_indices.astype(np.int64) * g.v_count + ev)
    np.testing.assert_array_equal(k_u, k_v)
    g2 = BipartiteGraph.from_bytes(g.to_bytes())
    assert g2.fingerprint == g.fingerprint
    np.testing.assert_array_equal(g2.v_weights, g.v_weights)


def test_graph_constructor_errors():
    with pytest.raises(DataError, match="empty"):
        BipartiteGraph(["a"], ["b"], [], [], [])
    with pytest.raises(DataError, match="both sides"):
        BipartiteGraph(["a"], ["a"], [0], [0], [1.0])
    with pytest.raises(DataError, match="positive"):
        BipartiteGraph(["a"], ["b"], [0], [0], [0.0])
    with pytest.raises(DataError, match="duplicate edge"):
        BipartiteGraph(["a"], ["b"], [0, 0], [0, 0], [1.0, 2.0])
    with pytest.raises(DataError, match="isolated"):
        BipartiteGraph(["a", "c"], ["b"], [0], [0], [1.0])
    with pytest.raises(DataError, match="out of range"):
        BipartiteGraph(["a"], ["b"], [1], [0], [1.0])
    with pytest.raises(DataError):
        BipartiteGraph.from_bytes(b"XXXX" + bytes(40))


def test_labels_and_lookup():
    g = BipartiteGraph.from_arrays(3, 2, [0, 1, 2], [0, 1, 1], [1.0, 2.0, 3.0])
    assert g.u_id("u2") == 2 and list(g.u_labels) == ["u0", "u1", "u2"]
    with pytest.raises(DataError):
        g.u_id("u3")
    with pytest.raises(DataError):
        g.u_id("u01")
    lab = IndexLabels("v", 4)
    assert lab[-1] == "v3" and lab[1:3] == ["v1", "v2"]
    h = BipartiteGraph.from_edges(["a", "b"], ["x"], [(0, 0, 1.0), (1, 0, 1.0), (0, 0, 2.0)])
    assert h.edge_count == 2 and h.u_weights[0] == 3.0


# -- parameters, sampling, generator ---------------------------------------------

def test_parameter_pickers_match_reference_definitions():
    assert bh.required_iterations(0.15, 0.1, 1.0) == 14
    assert bh.required_iterations(0.15, 1e-4, 0.5) == 52
    assert bh.required_iterations(0.15, 1.0, 1.0) == 0
    with pytest.raises(ValueError):
        bh.required_iterations(1.0, 0.1, 1.0)
    d = load("c1")
    g = config_graph("c1")
    assert bh.estimate_mu(g) == float(d["mu"])
    assert bh.default_tau(g, 0.15) == int(d["tau"])
    eps = float(d["eps"])
    assert [bh.choose_eps_b(eps, float(d["mu"])), eps - bh.choose_eps_b(eps, float(d["mu"]))] == list(d["eps_split"][0])
    for eps in (1e-2, 1e-6):
        for mu in (0.0, 0.5, 1.0):
            assert eps / 10 <= bh.choose_eps_b(eps, mu) <= eps / 2
    with pytest.raises(ValueError):
        bh.choose_eps_b(0.0, 0.5)


def test_meta_save_load_roundtrip(tmp_path):
    g = config_graph("c1")
    meta = bh.IndexMeta(0.15, 21.5, 60, 0.1225, lambda e: bh.choose_eps_b(e, 0.1225), g.fingerprint)
    bh.save_meta(meta, tmp_path / "m.json")
    m2 = bh.load_meta(tmp_path / "m.json")
    assert (m2.alpha, m2.lam, m2.tau, m2.mu, m2.graph_fingerprint) == (0.15, 21.5, 60, 0.1225, g.fingerprint)
    (tmp_path / "bad.json").write_text('{"format_version": 9}')
    with pytest.raises(DataError):
        bh.load_meta(tmp_path / "bad.json")


def test_substream_and_bench_sources_are_the_reference_draws():
    # the reference's cmd_bench draw for seed 0 (cli.py:415-417), recorded in the golden fixture
    d = load("c2s")
    got = substream(0, "bench-queries").choice(int(d["n"][0]), 6, replace=False)
    np.testing.assert_array_equal(got, d["sources"])
    assert list(bench_sources(10, 20)) == list(range(10))
    a = substream(1, "x", 2).random(3)
    b = substream(1, "x", "2").random(3)
    np.testing.assert_array_equal(a, b)


def test_chung_lu_generator_contract():
    cfg = scaled_config("c4", 1000)
    eu, ev, ew = chung_lu_edges(cfg.u_count, cfg.v_count, cfg.edge_count, cfg.beta_u, cfg.beta_v, cfg.weights,
                                cfg.seed, cfg.max_deg_v)
    assert eu.size == cfg.edge_count
    assert np.unique(eu * cfg.v_count + ev).size == cfg.edge_count
    assert np.bincount(eu, minlength=cfg.u_count).min() >= 1
    assert np.bincount(ev, minlength=cfg.v_count).min() >= 1
    assert (ew == 1.0).all()
    eu2, ev2, _ = chung_lu_edges(cfg.u_count, cfg.v_count, cfg.edge_count, cfg.beta_u, cfg.beta_v, cfg.weights,
                                 cfg.seed, cfg.max_deg_v)
    np.testing.assert_array_equal(eu, eu2)
    np.testing.assert_array_equal(ev, ev2)
    c2 = CONFIGS["c2"]
    _, _, w = chung_lu_edges(2000, 4000, 40000, c2.beta_u, c2.beta_v, "int10", 5)
    assert set(np.unique(w)) <= set(range(1, 11))


def test_small_golden_graphs_load():
    d = load("small")
    for i in range(int(d["count"])):
        g = graph_from(d, f"g{i}_")
        assert g.edge_count == int(d[f"g{i}_n"][2])


def test_operator_views_match_reference_definitions():
    """u_step / v_step / transposes / recv_* (bigraph.py:148-188) on a golden graph."""
    g = config_graph("c1")
    u = g.u_step.toarray()
    v = g.v_step.toarray()
    np.testing.assert_allclose(u.sum(axis=1), 1.0, rtol=1e-12)
    np.testing.assert_allclose(v.sum(axis=1), 1.0, rtol=1e-12)
    np.testing.assert_array_equal(g.u_step_t.toarray(), u.T)
    np.testing.assert_array_equal(g.v_step_t.toarray(), v.T)
    eu = np.repeat(np.arange(g.u_count), np.diff(g.u_indptr))
    np.testing.assert_array_equal(g.recv_uv, g.u_weights / g.ws_v[g.u_indices])
    assert g.v_id(g.v_labels[7]) == 7 and g.u_id(g.u_labels[eu[3]]) == eu[3]
    with pytest.raises(bh.DataError, match="unknown V-side label"):
        g.v_id("nope")


def test_mc_walk_count():
    assert bh.mc_walk_count(0.1, 1e-6, 1000) == 4283  # ceil(2 (1 + 0.1/3) ln(1e9) / 0.01)
    assert bh.mc_walk_count(10.0, 0.5, 1) == 1
    for bad in ((0.0, 1e-6, 10), (0.1, 0.0, 10), (0.1, 1e-6, 0)):
        with pytest.raises(ValueError):
            bh.mc_walk_count(*bad)


def test_host_side_abi_error_paths():
    """Entry points that need no GPU report bad arguments with status codes and
    bh_last_error, never by crashing (status -> exception mapping of _capi.check)."""
    import ctypes as C

    lib = _capi.lib()
    h = C.c_void_p()
    err = C.c_int64(0)
    assert lib.bh_edge_list_parse(None, 5, None, 0, 0, 0.0, C.byref(h), C.byref(err)) == _capi.BH_EINVAL
    assert b"null" in lib.bh_last_error()
    assert lib.bh_edge_list_parse(b"a x 1\n", 6, b"", 0, 0, 0.0, C.byref(h), C.byref(err)) == _capi.BH_EINVAL
    assert lib.bh_edge_list_parse(b"a x 1\nb y\n", 10, None, 0, 0, 0.0, C.byref(h), C.byref(err)) == _capi.BH_EFALLBACK
    assert err.value == 2  # the two-column line without a default weight
    assert lib.bh_edge_list_parse(b"a x 1\n", 6, None, 0, 0, 0.0, C.byref(h), C.byref(err)) == _capi.BH_OK
    n = [C.c_int64() for _ in range(5)]
    assert lib.bh_edge_list_sizes(h, *[C.byref(x) for x in n]) == _capi.BH_OK
    assert [x.value for x in n] == [1, 1, 1, 1, 1]
    lib.bh_edge_list_free(h)
    assert lib.bh_monte_carlo(None, 0, 0.15, 0, 1, 0, None) == _capi.BH_EINVAL
    assert lib.bh_query_wait(None) == _capi.BH_EINVAL
    with pytest.raises(ValueError):
        _capi.check(_capi.BH_EINVAL)
    with pytest.raises(MemoryError):
        _capi.check(_capi.BH_ENOMEM)


def test_similarity_rows_rejects_methods_off_the_bhpp_path():
    g = bh.BipartiteGraph(["a", "b"], ["x"], [0, 1], [0, 0], [1.0, 2.0])
    for m in ("jaccard", "naive-ppr", "nope"):
        with pytest.raises(bh.DataError):
            bh.similarity_rows(m, g)


def test_batch_source_list_keeps_each_elements_type():
    from paper_2312_06724_b200.bhpp_query import _source_list

    assert _source_list(5) == [5]
    assert _source_list("u3") == ["u3"]
    assert _source_list(["u3", 17, np.int64(4)]) == ["u3", 17, np.int64(4)]
    assert _source_list(np.array([[1, 2], [3, 4]])) == [1, 2, 3, 4]
    assert _source_list(np.array(["a", "b"])) == ["a", "b"]
    assert _source_list((x for x in (1, 2))) == [1, 2]


def test_scatter_limit_switch_mirrors_reference_constant(monkeypatch):
    """push_engine._SCATTER_LIMIT (push_engine.py:44) is handed to the engine
    before every run; NaN is rejected by the C ABI (no GPU needed)."""
    from paper_2312_06724_b200 import push_engine as pe

    assert 0.0 < pe._SCATTER_LIMIT <= 0.25
    lib = _capi.lib()
    assert lib.bh_set_scatter_limit(float("nan")) != 0
    monkeypatch.setattr(pe, "_SCATTER_LIMIT", -1.0)
    _capi.apply_scatter_limit()
    assert _capi._applied_limit == -1.0
    monkeypatch.setattr(pe, "_SCATTER_LIMIT", 0.25)
    _capi.apply_scatter_limit()
    assert _capi._applied_limit == 0.25
    monkeypatch.undo()
    _capi.apply_scatter_limit()
