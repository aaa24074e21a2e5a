"""Full-size parity on BASELINE configs c3, c4 and the c5 epsilon sweep,
against the live C oracle (bit-exact restatement of the reference, pinned by
tests/golden) on the same seeded graphs.

The graphs are the configs' seeded Chung-Lu stand-ins built with the device
generator (synth.make_graph(..., device=0): identical to the host generator,
seconds instead of minutes) and canonicalised on the device (bh_csr_build).
Both sides share one IndexMeta (device build_index_meta; lambda is checked
against the oracle's at c2 scale in test_gpu_scale.py).

Bars (BASELINE.json north_star): fp64 scores within 1e-9 absolute with
identical integer phase traces (PI-Push exact ties replayed from the oracle,
SURVEY.md section 7 hard part 1); fp32 top-k scores within 1e-5 relative (plus
an absolute floor of eps) with index sets equal up to ties inside that band.
Reference path: bhpp_query.py:160-203 (bhpp_query), push_engine.py:145-258.
"""

import os

import numpy as np
import pytest

import paper_2312_06724_b200 as bh
from oracle import cpu_oracle as O
from paper_2312_06724_b200.rng import substream
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

pytestmark = pytest.mark.gpu

RTOL32 = 1e-5   # north_star: fp32 scores within 1e-5 relative
ATOL64 = 1e-9   # north_star: fp64 scores within 1e-9 absolute


def _threads(n):
    return max(1, min(n, os.cpu_count() or 1))


def _setup(name, sources, eps):
    cfg = CONFIGS[name]
    g = make_graph(cfg, device=0)
    meta = bh.build_index_meta(g, cfg.alpha)
    og = O.OracleGraph(g)
    eb = meta.eps_split_policy(eps)
    ref = og.bhpp_query_many([int(s) for s in sources], cfg.alpha, meta.lam, eb, eps - eb,
                             threads=_threads(len(sources)))
    return cfg, g, meta, og, ref


def check_fp64(g, meta, src, eps, ref, k):
    ties = np.array([O.tie_skip_for(tr["forward"]) for _, tr in ref], dtype=np.int32)
    res = bh.bhpp_query_batch(g, meta, src, eps, k=k, dtype="fp64", return_scores=True, tie_skip=ties)
    for i, (scores, tr) in enumerate(ref):
        err = float(np.abs(res.scores[i] - scores).max())
        assert err <= ATOL64, (i, err)
        got = res.trace_dicts(i)
        assert got["backward"] == tr["backward"], (i, got, tr)
        fwd = {kk: v for kk, v in tr["forward"].items() if kk not in ("tie_checks", "tie_break_at", "gamma")}
        assert {kk: v for kk, v in got["forward"].items() if kk != "gamma"} == fwd, (i, got, tr)
        assert got["forward"]["gamma"] == pytest.approx(tr["forward"]["gamma"], rel=1e-12)
        top = O.topk_indices(scores, k)
        diff = res.topk_index[i] != top
        if diff.any():  # only exact score ties may reorder
            assert np.abs(scores[res.topk_index[i][diff]] - scores[top[diff]]).max() <= 1e-12
    return res


def check_fp32(g, meta, src, eps, ref, k):
    res = bh.bhpp_query_batch(g, meta, src, eps, k=k, dtype="fp32")
    worst = 0.0
    for i, (scores, _tr) in enumerate(ref):
        top = O.topk_indices(scores, k)
        np.testing.assert_allclose(res.topk_score[i], scores[top], rtol=RTOL32, atol=eps)
        worst = max(worst, float(np.max(np.abs(res.topk_score[i] - scores[top]) / np.abs(scores[top]))))
        kth = scores[top[-1]]
        diff = res.topk_index[i] != top
        if diff.any():  # index sets equal except for ties inside the tolerance band
            assert np.abs(scores[res.topk_index[i][diff]] - scores[top[diff]]).max() <= RTOL32 * kth + eps
    return res, worst


# -- c3: |U|=5e6, |V|=2e6, |E|=1e8, beta 2.1, int weights, eps 1e-7, top-50 ----------------------

@pytest.fixture(scope="module")
def c3():
    src = bench_sources(CONFIGS["c3"].u_count, 1024)[:2]
    cfg, g, meta, og, ref = _setup("c3", src, 1e-7)
    yield cfg, g, meta, src, ref
    del og


def test_c3_full_size_fp64_parity(c3):
    cfg, g, meta, src, ref = c3
    check_fp64(g, meta, src, 1e-7, ref, cfg.k)


def test_c3_full_size_fp32_parity(c3):
    cfg, g, meta, src, ref = c3
    _, worst = check_fp32(g, meta, src, 1e-7, ref, cfg.k)
    assert worst <= RTOL32


# -- c4: |U|=2e6, |V|=1e7, |E|=3e8, V hubs to 1e6, unit weights, alpha 0.2, eps 1e-6, top-20 ---

@pytest.fixture(scope="module")
def c4():
    src = bench_sources(CONFIGS["c4"].u_count, 4096)[:1]
    cfg, g, meta, og, ref = _setup("c4", src, 1e-6)
    yield cfg, g, meta, src, ref
    del og


def test_c4_full_size_fp64_parity(c4):
    cfg, g, meta, src, ref = c4
    assert int(g.deg_v.max()) >= 500_000  # the hub-skewed shape (max deg_V ~1e6)
    check_fp64(g, meta, src, 1e-6, ref, cfg.k)


def test_c4_full_size_fp32_parity(c4):
    cfg, g, meta, src, ref = c4
    check_fp32(g, meta, src, 1e-6, ref, cfg.k)


# -- c5: the c2 graph, every source once; epsilon sweep, 4 sampled sources per epsilon ---------

@pytest.fixture(scope="module")
def c5():
    cfg = CONFIGS["c5"]
    g = make_graph(cfg, device=0)
    meta = bh.build_index_meta(g, cfg.alpha)
    og = O.OracleGraph(g)
    return cfg, g, meta, og


@pytest.mark.parametrize("eps", [1e-4, 1e-6, 1e-8])
def test_c5_eps_sweep_parity(c5, eps):
    cfg, g, meta, og = c5
    src = substream(0, "c5-parity", int(round(-np.log10(eps)))).choice(g.u_count, 4, replace=False)
    eb = meta.eps_split_policy(eps)
    ref = og.bhpp_query_many([int(s) for s in src], cfg.alpha, meta.lam, eb, eps - eb, threads=_threads(4))
    check_fp64(g, meta, src, eps, ref, cfg.k)
    check_fp32(g, meta, src, eps, ref, cfg.k)
    # the c5 workload shape: many sources in one batch, slots refilled on the
    # device; at the same slot width a query's result does not depend on its
    # neighbours in the batch (bitwise)
    many = np.concatenate([src, bench_sources(g.u_count, g.u_count)[:252]])
    big = bh.bhpp_query_batch(g, meta, many, eps, k=cfg.k, dtype="fp32", slots=128)
    small = bh.bhpp_query_batch(g, meta, src, eps, k=cfg.k, dtype="fp32", slots=128)
    np.testing.assert_array_equal(big.topk_index[:4], small.topk_index)
    np.testing.assert_array_equal(big.topk_score[:4], small.topk_score)
