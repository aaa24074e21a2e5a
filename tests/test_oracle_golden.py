"""Pin the C oracle against the reference's own outputs (tests/golden/*.npz).

The fixtures were produced by running the unmodified reference package
(tests/golden/make_golden.py).  The oracle restates it operation for
operation, so the bar here is bit-identity of scores and identity of every
integer trace counter -- including the PI-Push exact-tie decisions the
reference resolves by rounding.
"""

import numpy as np
import pytest

from golden_io import config_alpha, config_graph, graph_from, load, split_traces, trace_dict
from oracle import cpu_oracle as O


def test_numpy_pairwise_sum_bitwise():
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 8, 9, 127, 128, 129, 1000, 4097, 100_003, 2_000_001):
        x = rng.random(n) * rng.random(n) ** 6
        assert O.numpy_sum(x) == float(x.sum())


def test_required_iterations_pins():
    d = load("known")
    got = [O.required_iterations(0.15, 0.1, 1.0), O.required_iterations(0.15, 1e-4, 0.5),
           O.required_iterations(0.15, 1.0, 1.0)]
    assert got == list(d["req_iter"]) == [14, 52, 0]
    assert O.required_iterations(0.15, 1e-6, 0.0) == 0
    assert O.required_iterations(0.15, 1e-6, -1.0) == 0


@pytest.mark.parametrize("name", ["g2", "g3"])
def test_closed_form_graphs(name):
    from paper_2312_06724_b200.bigraph import BipartiteGraph

    d = load("known")
    if name == "g2":
        g = BipartiteGraph(["u1", "u2"], ["v1"], [0, 1], [0, 0], [1.0, 1.0])
    else:
        g = BipartiteGraph(["u1", "u2"], ["v1", "v2"], [0, 0, 1], [0, 1, 1], [1.0, 1.0, 1.0])
    og = O.OracleGraph(g)
    meta = O.index_meta(g, 0.15)
    assert meta["lam"] == float(d[f"{name}_lam"])
    for eps in (1e-3, 1e-6, 1e-9):
        eb = O.choose_eps_b(eps, meta["mu"])
        sc, tr = og.bhpp_query(0, 0.15, meta["lam"], eb, eps - eb)
        np.testing.assert_array_equal(sc, d[f"{name}_bhpp_{eps:g}"])
        vec = d[f"{name}_bhpp_{eps:g}_trace"]
        assert tr["backward"] == trace_dict(vec[:5], False)
        fwd = {k: v for k, v in tr["forward"].items() if k in trace_dict(vec[5:], True)}
        assert fwd == trace_dict(vec[5:], True)
        # one-sided within eps of the dense truth (acceptance criterion 1)
        diff = d[f"{name}_exact_bhpp0"] - sc
        assert diff.min() >= -1e-10 and diff.max() <= eps + 1e-12
    if name == "g2":
        np.testing.assert_array_equal(og.power_iteration(np.array([1.0, 0.0]), 0.15, 150), d["g2_pi150"])
        np.testing.assert_allclose(d["g2_pi150"], [0.575, 0.425], atol=1e-9)


@pytest.mark.parametrize("name", ["c1", "c2s", "c4s"])
def test_config_queries_bitwise(name):
    d = load(name)
    g = config_graph(name)
    alpha = config_alpha(name)
    og = O.OracleGraph(g)
    meta = O.index_meta(g, alpha)
    assert meta["lam"] == float(d["lam"]) and meta["tau"] == int(d["tau"]) and meta["mu"] == float(d["mu"])
    eps = float(d["eps"])
    k = int(d["k"])
    srcs = d["sources"] if name == "c1" else d["sources"][:3]
    for i, q in enumerate(srcs):
        eb = O.choose_eps_b(eps, meta["mu"])
        assert [eb, eps - eb] == list(d["eps_split"][i])
        sc, tr = og.bhpp_query(int(q), alpha, meta["lam"], eb, eps - eb)
        np.testing.assert_array_equal(sc, d["scores"][i])
        back, fwd, gamma = split_traces(d["traces"][i])
        assert tr["backward"] == back
        assert {k2: tr["forward"][k2] for k2 in fwd} == fwd
        assert tr["forward"]["gamma"] == gamma
        assert [tr["forward"]["tie_checks"], tr["forward"]["tie_break_at"]] == list(d["ties"][i])
        np.testing.assert_array_equal(O.topk_indices(sc, k), d["topk"][i])
        np.testing.assert_array_equal(O.topk_indices(sc, k, int(q)), d["topk_ex"][i])


def test_small_graphs_every_kernel_bitwise():
    d = load("small")
    for i in range(int(d["count"])):
        p = f"g{i}_"
        g = graph_from(d, p)
        og = O.OracleGraph(g)
        alpha, eps, q, limit, lam, tau, mu = d[p + "params"]
        q, tau = int(q), int(tau)
        meta = O.index_meta(g, alpha)
        assert meta["lam"] == lam and meta["tau"] == tau and meta["mu"] == mu
        eb = O.choose_eps_b(eps, mu)
        sc, tr = og.bhpp_query(q, alpha, lam, eb, eps - eb, scatter_limit=limit)
        np.testing.assert_array_equal(sc, d[p + "bhpp"], err_msg=p)
        vec = d[p + "bhpp_trace"]
        assert tr["backward"] == trace_dict(vec[0:5], False)
        assert {k: tr["forward"][k] for k in trace_dict(vec[5:10], True)} == trace_dict(vec[5:10], True)
        assert tr["forward"]["gamma"] == vec[10]
        assert [tr["forward"]["tie_checks"], tr["forward"]["tie_break_at"]] == [int(vec[11]), int(vec[12])]

        led, ss_tr = og.ss_push(q, alpha, eb, scatter_limit=limit)
        np.testing.assert_array_equal(led["estimate"], d[p + "ss_est"])
        np.testing.assert_array_equal(led["residue_u"], d[p + "ss_res"])
        assert ss_tr == trace_dict(d[p + "ss_trace"], False)

        sled, sel_tr = og.ss_push(q, alpha, max(eb, 1e-7), budget=False, scatter_limit=limit)
        np.testing.assert_array_equal(sled["estimate"], d[p + "sel_est"])
        np.testing.assert_array_equal(sled["residue_u"], d[p + "sel_res"])
        assert sel_tr == trace_dict(d[p + "sel_trace"], False)

        lam_id, ef = d[p + "pi_id_params"]
        init = {"residue_u": np.eye(1, g.u_count, q)[0], "residue_v": np.zeros(g.v_count),
                "estimate": np.zeros(g.u_count), "n_p": 0}
        pis, pi_tr = og.pi_push(q, alpha, lam_id, ef, init, scatter_limit=limit)
        np.testing.assert_array_equal(pis, d[p + "pi_id"])
        pv = d[p + "pi_id_trace"]
        assert {k: pi_tr[k] for k in trace_dict(pv[:5], True)} == trace_dict(pv[:5], True)
        assert pi_tr["gamma"] == pv[5]
        np.testing.assert_array_equal(np.concatenate([init["residue_u"], init["estimate"], [init["n_p"]]]),
                                      d[p + "pi_id_led"])

        np.testing.assert_array_equal(og.power_iteration(d[p + "pow_start"], alpha, int(d[p + "pow_t"])), d[p + "pow"])


def test_hub_and_skew_budget_paths():
    d = load("hub")
    g = graph_from(d, "hub_")
    og = O.OracleGraph(g)
    lam = float(g.ws_u.max() / g.ws_u.min())
    init = {"residue_u": np.eye(1, g.u_count, 0)[0], "residue_v": np.zeros(g.v_count),
            "estimate": np.zeros(g.u_count), "n_p": 0}
    sc, tr = og.pi_push(0, 0.15, lam, 1e-7, init)
    np.testing.assert_array_equal(sc, d["hub_pi"])
    assert tr["terminated_by"] == "budget-switch" and tr["power_iterations"] > 0
    assert {k: tr[k] for k in trace_dict(d["hub_pi_trace"][:5], True)} == trace_dict(d["hub_pi_trace"][:5], True)

    s = graph_from(d, "skew_")
    os_ = O.OracleGraph(s)
    led, tr = os_.ss_push(0, 0.15, 1e-7)
    assert tr["terminated_by"] == "budget-switch" and tr["sequential_rounds"] > 0
    np.testing.assert_array_equal(led["estimate"], d["skew_ss_est"])
    assert tr == trace_dict(d["skew_ss_trace"], False)
    diff = d["skew_exact_col0"] - led["estimate"]
    assert diff.min() >= -1e-11 and diff.max() <= 1e-7 + 1e-12


def test_topk_tie_order():
    assert "".join("abcd"[i] for i in O.topk_indices(np.array([0.5, 0.25, 0.25, 0.25]), 4)) == str(load("known")["topk_ties"])


def test_round_hook_conservation():
    """Reference acceptance criterion 4 / test_push_engine.py:122-138 on the oracle."""
    d = load("known")  # noqa: F841  (fixture presence)
    from paper_2312_06724_b200.bigraph import BipartiteGraph

    rng = np.random.default_rng(5)
    for _ in range(5):
        n_u, n_v = int(rng.integers(3, 25)), int(rng.integers(3, 25))
        keys = set()
        eu, ev = [], []
        for i in range(max(n_u, n_v)):
            k = (i % n_u, i % n_v)
            keys.add(k)
        while len(keys) < min(n_u * n_v, int(2.5 * n_u) + max(n_u, n_v)):
            keys.add((int(rng.integers(n_u)), int(rng.integers(n_v))))
        for a, b in sorted(keys):
            eu.append(a)
            ev.append(b)
        g = BipartiteGraph.from_arrays(n_u, n_v, eu, ev, rng.random(len(eu)) + 0.1)
        og = O.OracleGraph(g)
        # dense truth via the closed form Pi = alpha (I - (1-alpha) P)^-1
        U = np.zeros((n_u, n_v))
        V = np.zeros((n_v, n_u))
        for u in range(n_u):
            for e in range(g.u_indptr[u], g.u_indptr[u + 1]):
                U[u, g.u_indices[e]] = g.u_weights[e] / g.ws_u[u]
        for v in range(n_v):
            for e in range(g.v_indptr[v], g.v_indptr[v + 1]):
                V[v, g.v_indices[e]] = g.v_weights[e] / g.ws_v[v]
        P = U @ V
        Pi = 0.15 * np.linalg.inv(np.eye(n_u) - 0.85 * P)
        t = int(rng.integers(0, n_u))

        def check(phase, rounds, led):
            assert np.abs(led["residue_v"]).max() == 0.0
            assert np.abs(led["estimate"] + Pi @ led["residue_u"] - Pi[:, t]).max() <= 1e-10

        og.ss_push(t, 0.15, 1e-5, budget=False, round_hook=check)
