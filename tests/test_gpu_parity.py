"""GPU parity: the CUDA engine (through the C ABI) against the reference.

The bar (BASELINE.json north_star): fp64 scores within 1e-9 absolute of the
reference and integer phase traces identical; fp32 top-k scores within 1e-5
relative and top-k index sets identical up to score ties inside that tolerance.

Golden fixtures were produced by the unmodified reference (tests/golden/);
larger cases compare against the bit-exact C oracle run live on the same
inputs.  PI-Push budget checks that are exact ties in real arithmetic (SURVEY.md
section 0 fact 11) are replayed with the reference's branch via ``tie_skip``
(the tie-aware protocol of SURVEY.md section 7, hard part 1).
"""

import numpy as np
import pytest

import paper_2312_06724_b200 as bh
from golden_io import config_alpha, config_graph, graph_from, load, split_traces, trace_dict
from oracle import cpu_oracle as O

pytestmark = pytest.mark.gpu

ATOL64 = 1e-9
RTOL32 = 1e-5


def meta_for(g, alpha):
    return bh.build_index_meta(g, alpha)


def tie_skip_from(ties_row):
    checks, broke_at = int(ties_row[0]), int(ties_row[1])
    return broke_at - 1 if broke_at else checks


def assert_traces(res_trace, back, fwd, gamma=None, rel_gamma=1e-12):
    assert res_trace["backward"] == back
    got_f = dict(res_trace["forward"])
    g = got_f.pop("gamma")
    exp_f = dict(fwd)
    exp_f.pop("gamma", None)
    assert got_f == exp_f
    if gamma is not None:
        assert g == pytest.approx(gamma, rel=rel_gamma, abs=1e-300)


def topk_equal_up_to_ties(got_idx, got_sc, exp_idx, scores_ref, rtol, atol=0.0):
    """Index lists equal, except positions whose reference scores tie within tolerance."""
    got_idx = list(got_idx)
    exp_idx = list(exp_idx)
    if got_idx == exp_idx:
        return
    kth = scores_ref[exp_idx[-1]]
    tol = max(abs(kth) * rtol, atol)
    # every differing entry must sit within tolerance of the cut
    for a, b in zip(got_idx, exp_idx):
        if a != b:
            assert abs(scores_ref[a] - scores_ref[b]) <= tol + abs(scores_ref[b]) * rtol, (a, b)


# -- closed forms --------------------------------------------------------------

@pytest.mark.parametrize("name", ["g2", "g3"])
def test_closed_form_graphs(name):
    d = load("known")
    if name == "g2":
        g = bh.BipartiteGraph(["u1", "u2"], ["v1"], [0, 1], [0, 0], [1.0, 1.0])
    else:
        g = bh.BipartiteGraph(["u1", "u2"], ["v1", "v2"], [0, 0, 1], [0, 1, 1], [1.0, 1.0, 1.0])
    meta = meta_for(g, 0.15)
    assert meta.lam == pytest.approx(float(d[f"{name}_lam"]), rel=1e-12)
    for eps in (1e-3, 1e-6, 1e-9):
        r = bh.bhpp_query(g, meta, 0, eps)
        np.testing.assert_allclose(r.scores, d[f"{name}_bhpp_{eps:g}"], atol=ATOL64, rtol=0)
        vec = d[f"{name}_bhpp_{eps:g}_trace"]
        assert_traces(r.phase_trace, trace_dict(vec[:5], False), trace_dict(vec[5:], True))
    if name == "g2":
        np.testing.assert_allclose(bh.power_iteration(g, np.array([1.0, 0.0]), 0.15, 150), [0.575, 0.425],
                                   atol=1e-9)


# -- config 1 (the reference's CPU-runnable case) ------------------------------

def test_c1_single_query_u0_fp64():
    d = load("c1")
    g = config_graph("c1")
    meta = meta_for(g, 0.15)
    assert meta.lam == pytest.approx(float(d["lam"]), rel=1e-12)
    assert meta.tau == int(d["tau"]) and meta.mu == float(d["mu"])
    assert int(d["sources"][0]) == 0
    r = bh.bhpp_query(g, meta, 0, float(d["eps"]), tie_skip=tie_skip_from(d["ties"][0]))
    np.testing.assert_allclose(r.scores, d["scores"][0], atol=ATOL64, rtol=0)
    back, fwd, gamma = split_traces(d["traces"][0])
    assert_traces(r.phase_trace, back, fwd, gamma)
    top = bh.topk(r, 10)
    assert [g.u_id(lab) for lab, _ in top] == list(d["topk"][0])


def test_c1_batch_fp64_all_golden_sources():
    d = load("c1")
    g = config_graph("c1")
    meta = meta_for(g, 0.15)
    srcs = d["sources"]
    ties = np.array([tie_skip_from(t) for t in d["ties"]], dtype=np.int32)
    res = bh.bhpp_query_batch(g, meta, srcs, float(d["eps"]), k=10, dtype="fp64", return_scores=True,
                              tie_skip=ties)
    for i in range(len(srcs)):
        np.testing.assert_allclose(res.scores[i], d["scores"][i], atol=ATOL64, rtol=0, err_msg=f"source {srcs[i]}")
        back, fwd, gamma = split_traces(d["traces"][i])
        assert_traces(res.trace_dicts(i), back, fwd, gamma)
        topk_equal_up_to_ties(res.topk_index[i], res.topk_score[i], d["topk"][i], d["scores"][i], 0, ATOL64)
        np.testing.assert_allclose(res.topk_score[i], d["scores"][i][res.topk_index[i]], atol=ATOL64)


def test_c1_unforced_ties_stay_one_sided():
    """Without replaying the reference's tie branch the engine takes the
    exact-arithmetic branch; its scores must still be within eps of the truth
    from below (acceptance criterion 1), checked against the dense solve."""
    d = load("c1")
    g = config_graph("c1")
    meta = meta_for(g, 0.15)
    P = np.zeros((g.u_count, g.u_count))
    U = np.zeros((g.u_count, g.v_count))
    V = np.zeros((g.v_count, g.u_count))
    eu = np.repeat(np.arange(g.u_count), g.deg_u)
    U[eu, g.u_indices] = g.u_weights / g.ws_u[eu]
    ev = np.repeat(np.arange(g.v_count), g.deg_v)
    V[ev, g.v_indices] = g.v_weights / g.ws_v[ev]
    P = U @ V
    Pi = 0.15 * np.linalg.inv(np.eye(g.u_count) - 0.85 * P)
    eps = float(d["eps"])
    res = bh.bhpp_query_batch(g, meta, d["sources"][:16], eps, k=10, dtype="fp64", return_scores=True)
    for i, q in enumerate(d["sources"][:16]):
        truth = Pi[q, :] + Pi[:, q]
        diff = truth - res.scores[i]
        assert diff.min() >= -1e-10 and diff.max() <= eps + 1e-12


@pytest.mark.parametrize("slots", [1, 4, 16, 32, 64, 128])
def test_c1_every_slot_width(slots):
    d = load("c1")
    g = config_graph("c1")
    meta = meta_for(g, 0.15)
    srcs = d["sources"][:20]
    ties = np.array([tie_skip_from(t) for t in d["ties"][:20]], dtype=np.int32)
    res = bh.bhpp_query_batch(g, meta, srcs, float(d["eps"]), k=10, dtype="fp64", return_scores=True,
                              tie_skip=ties, slots=slots)
    for i in range(len(srcs)):
        np.testing.assert_allclose(res.scores[i], d["scores"][i], atol=ATOL64, rtol=0)
        back, fwd, gamma = split_traces(d["traces"][i])
        assert_traces(res.trace_dicts(i), back, fwd, gamma)
    r32 = bh.bhpp_query_batch(g, meta, srcs, float(d["eps"]), k=10, dtype="fp32", tie_skip=ties, slots=slots)
    for i in range(len(srcs)):
        ref = d["scores"][i]
        exp = d["topk"][i]
        np.testing.assert_allclose(r32.topk_score[i], ref[exp], rtol=RTOL32, atol=float(d["eps"]))


# -- small random graphs: every kernel ------------------------------------------

def test_small_graphs_every_kernel_fp64():
    d = load("small")
    for i in range(int(d["count"])):
        p = f"g{i}_"
        g = graph_from(d, p)
        alpha, eps, q, limit, lam, tau, mu = d[p + "params"]
        q, tau = int(q), int(tau)
        og = O.OracleGraph(g)
        eb = O.choose_eps_b(eps, mu)
        vec = d[p + "bhpp_trace"]
        meta = bh.IndexMeta(alpha, lam, tau, mu, lambda e, _m=mu: bh.choose_eps_b(e, _m), g.fingerprint)
        r = bh.bhpp_query(g, meta, q, eps, tie_skip=tie_skip_from(vec[11:13]))
        np.testing.assert_allclose(r.scores, d[p + "bhpp"], atol=ATOL64, rtol=0, err_msg=p)
        assert_traces(r.phase_trace, trace_dict(vec[0:5], False), trace_dict(vec[5:10], True), vec[10])

        ss = bh.ss_push(g, q, alpha, eb)
        np.testing.assert_allclose(ss.ledger.estimate, d[p + "ss_est"], atol=1e-12, rtol=0)
        np.testing.assert_allclose(ss.ledger.residue_u, d[p + "ss_res"], atol=1e-12, rtol=0)
        assert {**ss.phase_trace, "terminated_by": ss.terminated_by} == trace_dict(d[p + "ss_trace"], False)

        sel = bh.selective_push(g, q, alpha, max(eb, 1e-7))
        np.testing.assert_allclose(sel.ledger.estimate, d[p + "sel_est"], atol=1e-12, rtol=0)
        assert {**sel.phase_trace, "terminated_by": sel.terminated_by} == trace_dict(d[p + "sel_trace"], False)

        lam_id, ef = d[p + "pi_id_params"]
        init = {"residue_u": np.eye(1, g.u_count, q)[0], "residue_v": np.zeros(g.v_count),
                "estimate": np.zeros(g.u_count), "n_p": 0}
        _, otr = og.pi_push(q, alpha, lam_id, ef, dict(init), scatter_limit=limit)
        led = bh.ResidueLedger.initial(g, q)
        pi = bh.pi_push(g, q, alpha, lam_id, ef, led, tie_skip=O.tie_skip_for(otr))
        np.testing.assert_allclose(pi.scores, d[p + "pi_id"], atol=ATOL64, rtol=0, err_msg=p)
        pv = d[p + "pi_id_trace"]
        assert {**pi.phase_trace, "terminated_by": pi.terminated_by} | {"gamma": 0} == \
            trace_dict(pv[:5], True) | {"gamma": 0}
        exp_led = d[p + "pi_id_led"]
        np.testing.assert_allclose(led.residue_u, exp_led[:g.u_count], atol=1e-12)
        np.testing.assert_allclose(led.estimate, exp_led[g.u_count:2 * g.u_count], atol=1e-12)
        assert led.n_p == int(exp_led[-1])

        np.testing.assert_allclose(bh.power_iteration(g, d[p + "pow_start"], alpha, int(d[p + "pow_t"])),
                                   d[p + "pow"], atol=1e-12, rtol=1e-12)


def test_hub_budget_paths():
    d = load("hub")
    g = graph_from(d, "hub_")
    lam = float(g.ws_u.max() / g.ws_u.min())
    led = bh.ResidueLedger.initial(g, 0)
    og = O.OracleGraph(g)
    _, otr = og.pi_push(0, 0.15, lam, 1e-7, {"residue_u": led.residue_u.copy(), "residue_v": led.residue_v.copy(),
                                             "estimate": led.estimate.copy(), "n_p": 0})
    out = bh.pi_push(g, 0, 0.15, lam, 1e-7, led, tie_skip=O.tie_skip_for(otr))
    assert out.terminated_by == "budget-switch" and out.phase_trace["power_iterations"] > 0
    np.testing.assert_allclose(out.scores, d["hub_pi"], atol=ATOL64)
    s = graph_from(d, "skew_")
    ss = bh.ss_push(s, 0, 0.15, 1e-7)
    assert ss.terminated_by == "budget-switch" and ss.phase_trace["sequential_rounds"] > 0
    np.testing.assert_allclose(ss.ledger.estimate, d["skew_ss_est"], atol=1e-12)
    diff = d["skew_exact_col0"] - ss.ledger.estimate
    assert diff.min() >= -1e-11 and diff.max() <= 1e-7 + 1e-12


# -- scaled configs 2 and 4 -----------------------------------------------------

@pytest.mark.parametrize("name", ["c2s", "c4s"])
def test_scaled_configs_fp64(name):
    d = load(name)
    g = config_graph(name)
    alpha = config_alpha(name)
    meta = meta_for(g, alpha)
    assert meta.lam == pytest.approx(float(d["lam"]), rel=1e-12)
    srcs = d["sources"]
    ties = np.array([tie_skip_from(t) for t in d["ties"]], dtype=np.int32)
    k = int(d["k"])
    res = bh.bhpp_query_batch(g, meta, srcs, float(d["eps"]), k=k, dtype="fp64", return_scores=True, tie_skip=ties)
    for i in range(len(srcs)):
        np.testing.assert_allclose(res.scores[i], d["scores"][i], atol=ATOL64, rtol=0)
        back, fwd, gamma = split_traces(d["traces"][i])
        assert_traces(res.trace_dicts(i), back, fwd, gamma)
        topk_equal_up_to_ties(res.topk_index[i], res.topk_score[i], d["topk"][i], d["scores"][i], 0, ATOL64)


@pytest.mark.parametrize("name", ["c2s", "c4s"])
def test_scaled_configs_fp32(name):
    d = load(name)
    g = config_graph(name)
    alpha = config_alpha(name)
    meta = meta_for(g, alpha)
    srcs = d["sources"]
    ties = np.array([tie_skip_from(t) for t in d["ties"]], dtype=np.int32)
    k = int(d["k"])
    res = bh.bhpp_query_batch(g, meta, srcs, float(d["eps"]), k=k, dtype="fp32", tie_skip=ties)
    for i in range(len(srcs)):
        ref = d["scores"][i]
        exp = d["topk"][i]
        np.testing.assert_allclose(res.topk_score[i], ref[exp], rtol=RTOL32, atol=float(d["eps"]))
        topk_equal_up_to_ties(res.topk_index[i], res.topk_score[i], exp, ref, RTOL32, float(d["eps"]))


@pytest.mark.parametrize("variant", [
    {},                      # default: one CUDA graph per batch (WHILE/IF conditional nodes)
    {"BH_NO_GRAPH": "1"},    # eager launches, host-polled round loop
])
def test_every_engine_variant(variant, monkeypatch):
    """Each engine variant (chosen when the engine is built) reproduces
    the golden fp64 scores / traces and the fp32 top-k on c2s."""
    for k, v in variant.items():
        monkeypatch.setenv(k, v)
    d = load("c2s")
    g = bh.BipartiteGraph.from_bytes(config_graph("c2s").to_bytes())  # fresh graph -> fresh engines
    meta = meta_for(g, 0.15)
    srcs = d["sources"][:6]
    ties = np.array([tie_skip_from(t) for t in d["ties"][:6]], dtype=np.int32)
    k = int(d["k"])
    r64 = bh.bhpp_query_batch(g, meta, srcs, float(d["eps"]), k=k, dtype="fp64", return_scores=True, tie_skip=ties)
    r32 = bh.bhpp_query_batch(g, meta, srcs, float(d["eps"]), k=k, dtype="fp32", tie_skip=ties)
    for i in range(len(srcs)):
        np.testing.assert_allclose(r64.scores[i], d["scores"][i], atol=ATOL64, rtol=0)
        back, fwd, gamma = split_traces(d["traces"][i])
        assert_traces(r64.trace_dicts(i), back, fwd, gamma)
        ref, exp = d["scores"][i], d["topk"][i]
        np.testing.assert_allclose(r32.topk_score[i], ref[exp], rtol=RTOL32, atol=float(d["eps"]))
        topk_equal_up_to_ties(r32.topk_index[i], r32.topk_score[i], exp, ref, RTOL32, float(d["eps"]))


# -- determinism, drop-in semantics, errors -------------------------------------

def test_runs_are_bitwise_deterministic():
    g = config_graph("c2s")
    meta = meta_for(g, 0.15)
    srcs = load("c2s")["sources"][:4]
    a = bh.bhpp_query_batch(g, meta, srcs, 1e-7, k=50, dtype="fp32", return_scores=True)
    b = bh.bhpp_query_batch(g, meta, srcs, 1e-7, k=50, dtype="fp32", return_scores=True)
    np.testing.assert_array_equal(a.scores, b.scores)
    np.testing.assert_array_equal(a.topk_index, b.topk_index)
    assert a.traces.tobytes() == b.traces.tobytes()


def test_topk_semantics():
    res = bh.QueryResult("x", 0, np.array([0.5, 0.25, 0.25, 0.25]), 1e-3, 5e-4, 5e-4, {}, {}, ["a", "b", "c", "d"])
    assert [lab for lab, _ in bh.topk(res, 4)] == list(str(load("known")["topk_ties"]))
    assert [lab for lab, _ in bh.topk(res, 50)] == ["a", "b", "c", "d"]
    assert [lab for lab, _ in bh.topk(res, 2, exclude_query=True)] == ["b", "c"]
    rng = np.random.default_rng(3)
    x = rng.integers(0, 50, 20000).astype(float) / 7.0
    res2 = bh.QueryResult("x", 5, x, 1e-3, 5e-4, 5e-4, {}, {}, None)
    for k in (1, 10, 1000, 1500):
        got = [int(lab) for lab, _ in bh.topk(res2, k, exclude_query=True)]
        assert got == list(O.topk_indices(x, k, 5))
    # radix-select edge cases: all equal, k-th inside a large tie block, negative and
    # zero values, sizes around the register-cached limit (16 x 256 per block)
    cases = [np.full(5000, 0.125), np.r_[np.full(3000, 2.0), np.full(3000, 1.0)],
             rng.normal(size=4096), np.r_[rng.random(4097), -rng.random(10), np.zeros(7)],
             rng.integers(0, 3, 100000).astype(float)]
    for x in cases:
        r = bh.QueryResult("x", 0, x, 1e-3, 5e-4, 5e-4, {}, {}, None)
        for k in (1, 50, 1023, 1024):
            got = [int(lab) for lab, _ in bh.topk(r, k)]
            assert got == list(O.topk_indices(x, k)), (x.size, k)


def test_errors_match_reference():
    g = config_graph("c1")
    meta = meta_for(g, 0.15)
    other = bh.BipartiteGraph.from_arrays(3, 2, [0, 1, 2], [0, 1, 1], [1.0, 1.0, 1.0])
    with pytest.raises(bh.DataError, match="rebuild"):
        bh.bhpp_query(other, meta, 0, 1e-3)
    broken = bh.IndexMeta(meta.alpha, meta.lam, meta.tau, meta.mu, lambda e: e, meta.graph_fingerprint)
    with pytest.raises(ValueError):
        bh.bhpp_query(g, broken, 0, 1e-3)
    led = bh.ResidueLedger.initial(g, 0)
    led.residue_v[0] = 0.5
    with pytest.raises(ValueError, match="unflushed"):
        bh.pi_push(g, 0, 0.15, 2.0, 1e-3, led)
    with pytest.raises(ValueError):
        bh.ss_push(g, 0, 1.0, 1e-3)
    with pytest.raises(ValueError):
        bh.bhpp_query_batch(g, meta, [g.u_count], 1e-3)


def test_round_hook_sees_phases_and_conserves():
    d = load("small")
    g = graph_from(d, "g3_")
    n_u = g.u_count
    U = np.zeros((n_u, g.v_count))
    V = np.zeros((g.v_count, n_u))
    eu = np.repeat(np.arange(n_u), g.deg_u)
    U[eu, g.u_indices] = g.u_weights / g.ws_u[eu]
    ev = np.repeat(np.arange(g.v_count), g.deg_v)
    V[ev, g.v_indices] = g.v_weights / g.ws_v[ev]
    Pi = 0.15 * np.linalg.inv(np.eye(n_u) - 0.85 * (U @ V))
    t = 1
    seen = []

    def check(phase, rounds, led):
        seen.append(phase)
        assert np.abs(led.residue_v).max() == 0.0
        if phase != "forward-selective":
            assert np.abs(led.estimate + Pi @ led.residue_u - Pi[:, t]).max() <= 1e-10

    bh.ss_push(g, t, 0.15, 1e-6, round_hook=check)
    meta = meta_for(g, 0.15)
    phases = set()
    bh.bhpp_query(g, meta, 0, 1e-5, round_hook=lambda ph, r, led: phases.add(ph))
    assert "selective" in phases or "sequential" in phases
    assert any(ph.startswith("forward") for ph in phases)
    snaps = []
    bh.selective_push(g, 0, 0.15, 1e-7, round_hook=lambda ph, r, led: snaps.append(led.estimate.copy()))
    for a, b in zip(snaps, snaps[1:]):
        assert (b - a).min() >= 0.0
