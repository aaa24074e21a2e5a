"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the dev container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures pin the C oracle (tests/test_oracle_golden.py) and the CUDA
engine (tests/test_gpu_parity.py).  /root/reference does not exist on the GPU
box, so nothing else may import it; the .npz files travel instead.

What is recorded, all from ``bipush`` (pkg/src/bipush) unmodified:
  known.npz     required_iterations pins, g2/g3 closed forms, topk tie order
  c1.npz        config-1 graph (edges), IndexMeta, bhpp_query for 48 sources
                (u=0 first) with scores, top-10, phase traces, and the PI-Push
                tie decisions read off round_hook (SURVEY.md section 7 hard part 1)
  small.npz     40 random small graphs: ss_push / selective_push / pi_push /
                power_iteration / bhpp_query outputs, both scatter and matrix
                paths forced on some (test_push_engine.py:188-202 idiom)
  hub.npz       the reference tests' hub graph (pi_push budget exit) and a
                skewed graph whose ss_push trips the budget switch
  c2s.npz       config-2 shape at 1/10 scale, 6 sources, eps=1e-7
  c4s.npz       config-4 shape at 1/100 scale, 3 sources, alpha=0.2, eps=1e-6
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import bipush  # noqa: E402
import bipush.push_engine as pe  # noqa: E402

from paper_2312_06724_b200.synth import CONFIGS, chung_lu_edges, scaled_config  # noqa: E402

TERM = {"threshold-met": 0, "budget-switch": 1, "mass-drained": 2}
TRACE_KEYS = ("selective_rounds", "sequential_rounds", "power_iterations", "n_p")


def ref_graph(n_u, n_v, eu, ev, ew):
    return bipush.BipartiteGraph([f"u{i}" for i in range(n_u)], [f"v{j}" for j in range(n_v)], eu, ev, ew)


def canon_edges(g):
    eu = np.repeat(np.arange(g.u_count, dtype=np.int64), g.deg_u)
    return eu, g.u_indices.astype(np.int64), np.asarray(g.u_weights)


def trace_vec(tr):
    return [tr[k] for k in TRACE_KEYS] + [TERM[tr["terminated_by"]]]


def query_with_ties(g, meta, q, eps):
    """bhpp_query plus the tie decisions observed through round_hook."""
    snaps = []
    res = bipush.bhpp_query(g, meta, q, eps, round_hook=lambda ph, r, led: snaps.append((ph, led.residue_u.copy())))
    ws = g.ws_u
    theta = (ws[q] / ws) * (res.epsilon_f / meta.lam)
    fwd_idx = [i for i, (ph, _) in enumerate(snaps) if ph == "forward-selective"]
    tie_checks = tie_break_at = 0
    all_full = True
    fwd = res.phase_trace["forward"]
    for j, i in enumerate(fwd_idx):
        pre = snaps[i - 1][1]
        post = snaps[i][1]
        if (pre > theta).sum() != g.u_count:
            all_full = False
        if not all_full:
            continue
        # the budget check after this round is reached only if the round did
        # not end the phase by threshold / mass
        if not (post > theta).any() or ((ws / ws[q]) * post).sum() <= 0.0:
            continue
        tie_checks += 1
        last = j == len(fwd_idx) - 1
        if last and fwd["terminated_by"] == "budget-switch":
            tie_break_at = tie_checks
    return res, tie_checks, tie_break_at


def random_graph(rng, n_u, n_v, avg_deg, weight_hi=10.0):
    """Covering assignment then distinct random edges; weights in (0, weight_hi]."""
    m = max(n_u, n_v)
    want = min(max(m, int(round(avg_deg * n_u))), n_u * n_v)
    vs = rng.permutation(n_v)
    keys = [(i % n_u) * n_v + int(vs[i % n_v]) for i in range(m)]
    seen = set(keys)
    while len(keys) < want:
        for a, b in zip(rng.integers(0, n_u, want).tolist(), rng.integers(0, n_v, want).tolist()):
            k = a * n_v + b
            if k not in seen:
                seen.add(k)
                keys.append(k)
                if len(keys) == want:
                    break
    keys = np.array(keys, dtype=np.int64)
    ew = weight_hi - rng.random(keys.size) * weight_hi * (1 - 1e-9)
    return keys // n_v, keys % n_v, ew


def known():
    out = {}
    out["req_iter"] = np.array([bipush.required_iterations(0.15, 0.1, 1.0),
                                bipush.required_iterations(0.15, 1e-4, 0.5),
                                bipush.required_iterations(0.15, 1.0, 1.0)])
    g2 = bipush.BipartiteGraph(["u1", "u2"], ["v1"], [0, 1], [0, 0], [1.0, 1.0])
    g3 = bipush.BipartiteGraph(["u1", "u2"], ["v1", "v2"], [0, 0, 1], [0, 1, 1], [1.0, 1.0, 1.0])
    out["g2_pi150"] = bipush.power_iteration(g2, np.array([1.0, 0.0]), 0.15, 150)
    for name, g in (("g2", g2), ("g3", g3)):
        meta = bipush.build_index_meta(g, 0.15)
        out[f"{name}_lam"] = np.array(meta.lam)
        for eps in (1e-3, 1e-6, 1e-9):
            r = bipush.bhpp_query(g, meta, 0, eps)
            out[f"{name}_bhpp_{eps:g}"] = r.scores
            out[f"{name}_bhpp_{eps:g}_trace"] = np.array(trace_vec(r.phase_trace["backward"]) + trace_vec(r.phase_trace["forward"]))
        dense = bipush.exact_hpp(g, 0.15, tol=1e-14)
        out[f"{name}_exact_bhpp0"] = bipush.exact_bhpp(dense, 0)
    res = bipush.QueryResult("x", 0, np.array([0.5, 0.25, 0.25, 0.25]), 1e-3, 5e-4, 5e-4, {}, {}, ["a", "b", "c", "d"])
    out["topk_ties"] = np.array("".join(lab for lab, _ in bipush.topk(res, 4)))
    np.savez_compressed(HERE / "known.npz", **out)


def config_fixture(name, cfg, sources, eps, with_full=True, k=None, store_edges=False):
    eu, ev, ew = chung_lu_edges(cfg.u_count, cfg.v_count, cfg.edge_count, cfg.beta_u, cfg.beta_v,
                                cfg.weights, cfg.seed, cfg.max_deg_v)
    g = ref_graph(cfg.u_count, cfg.v_count, eu, ev, ew)
    meta = bipush.build_index_meta(g, cfg.alpha)
    k = k or cfg.k
    out = {
        "n": np.array([g.u_count, g.v_count, g.edge_count]),
        "alpha": np.array(cfg.alpha), "eps": np.array(eps),
        "lam": np.array(meta.lam), "tau": np.array(meta.tau), "mu": np.array(meta.mu),
        "fingerprint": np.array(g.fingerprint),
        "sources": np.asarray(sources, dtype=np.int64),
        "k": np.array(k),
    }
    if store_edges:  # otherwise regenerate with synth.chung_lu_edges and check the fingerprint
        ceu, cev, cew = canon_edges(g)
        out["eu"], out["ev"], out["ew"] = ceu.astype(np.int32), cev.astype(np.int32), cew
    scores, topk, topk_ex, traces, ties, epsb = [], [], [], [], [], []
    for q in sources:
        res, tc, tb = query_with_ties(g, meta, int(q), eps)
        if with_full:
            scores.append(res.scores)
        order = np.argsort(-res.scores, kind="stable")
        topk.append(order[:k])
        topk_ex.append(order[order != q][:k])
        traces.append(trace_vec(res.phase_trace["backward"]) + trace_vec(res.phase_trace["forward"])
                      + [res.phase_trace["forward"]["gamma"]])
        ties.append([tc, tb])
        epsb.append([res.epsilon_b, res.epsilon_f])
        print(name, q, res.phase_trace["forward"]["terminated_by"], tc, tb, flush=True)
    out["topk_scores"] = np.array([np.asarray(s)[t] for s, t in zip(scores, topk)]) if with_full else np.zeros(0)
    if with_full:
        out["scores"] = np.array(scores)
    out["topk"] = np.array(topk)
    out["topk_ex"] = np.array(topk_ex)
    out["traces"] = np.array(traces, dtype=np.float64)
    out["ties"] = np.array(ties)
    out["eps_split"] = np.array(epsb)
    np.savez_compressed(HERE / f"{name}.npz", **out)


def small():
    rng = np.random.default_rng(20261019)
    out = {"count": np.array(40)}
    for i in range(40):
        n_u = int(rng.integers(5, 120))
        n_v = int(rng.integers(5, 120))
        eu, ev, ew = random_graph(rng, n_u, n_v, float(rng.uniform(1.5, 8.0)))
        if i % 4 == 0:
            ew = np.ones_like(ew)
        g = ref_graph(n_u, n_v, eu, ev, ew)
        ceu, cev, cew = canon_edges(g)
        p = f"g{i}_"
        out[p + "n"] = np.array([n_u, n_v, g.edge_count])
        out[p + "eu"], out[p + "ev"], out[p + "ew"] = ceu, cev, cew
        alpha = float(rng.choice([0.15, 0.2, 0.3]))
        eps = float(rng.choice([1e-2, 1e-4, 1e-6, 1e-8]))
        q = int(rng.integers(0, n_u))
        limit = [pe._SCATTER_LIMIT, 10.0, -1.0][i % 3]
        old = pe._SCATTER_LIMIT
        pe._SCATTER_LIMIT = limit
        try:
            meta = bipush.build_index_meta(g, alpha)
            out[p + "params"] = np.array([alpha, eps, q, limit, meta.lam, meta.tau, meta.mu])
            res, tc, tb = query_with_ties(g, meta, q, eps)
            out[p + "bhpp"] = res.scores
            out[p + "bhpp_trace"] = np.array(trace_vec(res.phase_trace["backward"]) + trace_vec(res.phase_trace["forward"])
                                            + [res.phase_trace["forward"]["gamma"], tc, tb], dtype=np.float64)
            eb = res.epsilon_b
            ss = bipush.ss_push(g, q, alpha, eb)
            out[p + "ss_est"], out[p + "ss_res"] = ss.ledger.estimate, ss.ledger.residue_u
            out[p + "ss_trace"] = np.array(trace_vec(ss.phase_trace | {"terminated_by": ss.terminated_by}))
            sel = bipush.selective_push(g, q, alpha, max(eb, 1e-7))
            out[p + "sel_est"], out[p + "sel_res"] = sel.ledger.estimate, sel.ledger.residue_u
            out[p + "sel_trace"] = np.array(trace_vec(sel.phase_trace | {"terminated_by": sel.terminated_by}))
            led = bipush.ResidueLedger.initial(g, q)
            lam = float(g.ws_u.max() / g.ws_u.min())
            ef = float(rng.choice([1e-3, 1e-5]))
            pi = bipush.pi_push(g, q, alpha, lam, ef, led)
            out[p + "pi_id"] = pi.scores
            out[p + "pi_id_params"] = np.array([lam, ef])
            out[p + "pi_id_trace"] = np.array(trace_vec(pi.phase_trace | {"terminated_by": pi.terminated_by})
                                              + [pi.phase_trace["gamma"]], dtype=np.float64)
            out[p + "pi_id_led"] = np.concatenate([led.residue_u, led.estimate, [led.n_p]])
            start = rng.random(n_u)
            t = int(rng.integers(0, 30))
            out[p + "pow_start"], out[p + "pow_t"] = start, np.array(t)
            out[p + "pow"] = bipush.power_iteration(g, start, alpha, t)
        finally:
            pe._SCATTER_LIMIT = old
    np.savez_compressed(HERE / "small.npz", **out)


def hub():
    out = {}
    n = 50
    eu = [0] * n + list(range(1, n + 1))
    ev = list(range(n)) + list(range(n))
    g = bipush.BipartiteGraph(["hub"] + [f"leaf{i}" for i in range(n)], [f"v{j}" for j in range(n)], eu, ev, [1.0] * (2 * n))
    ceu, cev, cew = canon_edges(g)
    out["hub_eu"], out["hub_ev"], out["hub_ew"] = ceu, cev, cew
    out["hub_n"] = np.array([g.u_count, g.v_count, g.edge_count])
    lam = float(g.ws_u.max() / g.ws_u.min())
    led = bipush.ResidueLedger.initial(g, 0)
    pi = bipush.pi_push(g, 0, 0.15, lam, 1e-7, led)
    out["hub_pi"] = pi.scores
    out["hub_pi_trace"] = np.array(trace_vec(pi.phase_trace | {"terminated_by": pi.terminated_by}) + [pi.phase_trace["gamma"]])
    s = bipush.synth_bipartite(60, 60, 400, degree_skew=2.5, seed=2)
    ceu, cev, cew = canon_edges(s)
    out["skew_eu"], out["skew_ev"], out["skew_ew"] = ceu, cev, cew
    out["skew_n"] = np.array([s.u_count, s.v_count, s.edge_count])
    ss = bipush.ss_push(s, 0, 0.15, 1e-7)
    out["skew_ss_est"] = ss.ledger.estimate
    out["skew_ss_trace"] = np.array(trace_vec(ss.phase_trace | {"terminated_by": ss.terminated_by}))
    dense = bipush.exact_hpp(s, 0.15, tol=1e-14)
    out["skew_exact_col0"] = dense.pi[:, 0]
    np.savez_compressed(HERE / "hub.npz", **out)


def main():
    known()
    print("known done", flush=True)
    small()
    print("small done", flush=True)
    hub()
    print("hub done", flush=True)
    c1 = CONFIGS["c1"]
    srcs = [0] + list(np.random.default_rng(1).choice(np.arange(1, c1.u_count), 47, replace=False))
    config_fixture("c1", c1, srcs, 1e-6, store_edges=True)
    c2s = scaled_config("c2", 10, "c2s")
    config_fixture("c2s", c2s, list(bipush.substream(0, "bench-queries").choice(c2s.u_count, 6, replace=False)), 1e-7)
    c4s = scaled_config("c4", 100, "c4s")
    config_fixture("c4s", c4s, list(bipush.substream(0, "bench-queries").choice(c4s.u_count, 3, replace=False)), 1e-6)


if __name__ == "__main__":
    main()
