"""Run a BASELINE.json configuration end to end: throughput + sampled parity.

    python tools/run_configs.py --config c3 [--dtype fp32] [--n-sources 1024]
                                [--parity 2] [--eps 1e-7] [--slots 64] [--lambda-check]

Builds the seeded Chung-Lu graph, IndexMeta (device power iteration), runs the
batch through the public API (host sources in, top-k out, device-timed with CUDA
events), then checks the first ``--parity`` sources against the bit-exact C
oracle: fp64 scores within 1e-9 with identical phase traces (the PI-Push exact
ties replayed from the oracle), fp32 top-k scores within 1e-5 relative with
index sets equal up to ties.  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2312_06724_b200 as bh
from oracle import cpu_oracle as O
from paper_2312_06724_b200 import _capi
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--dtype", default="fp32")
    ap.add_argument("--n-sources", type=int, default=0)
    ap.add_argument("--parity", type=int, default=2)
    ap.add_argument("--eps", type=float, default=0.0)
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--lambda-check", action="store_true")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    out = {"config": a.config, "dtype": a.dtype}
    t0 = time.perf_counter()
    g = make_graph(cfg, device=0)  # CSR canonicalised on the GPU (bh_csr_build)
    out["graph_build_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    fp = g.fingerprint
    out["fingerprint_s"] = time.perf_counter() - t0
    out["graph"] = {"u": g.u_count, "v": g.v_count, "e": g.edge_count, "max_deg_u": int(g.deg_u.max()),
                    "max_deg_v": int(g.deg_v.max()), "fingerprint": fp[:16]}
    t0 = time.perf_counter()
    meta = bh.build_index_meta(g, cfg.alpha)
    out["meta_s"] = time.perf_counter() - t0
    out["meta"] = {"lam": meta.lam, "tau": meta.tau, "mu": meta.mu}
    og = O.OracleGraph(g) if a.parity > 0 or a.lambda_check else None
    if a.lambda_check:
        t0 = time.perf_counter()
        om = O.index_meta(og, cfg.alpha)
        out["meta"]["lam_oracle"] = om["lam"]
        out["meta"]["lam_rel_err"] = abs(meta.lam - om["lam"]) / om["lam"]
        out["meta"]["oracle_meta_s"] = time.perf_counter() - t0
    n = a.n_sources or (cfg.n_sources or cfg.u_count)
    src = bench_sources(g.u_count, n)
    epss = [a.eps] if a.eps else list(cfg.epsilons)
    out["runs"] = []
    for eps in epss:
        run = {"eps": eps, "n_sources": int(n)}
        stream = torch.cuda.Stream()
        bh.bhpp_query_batch(g, meta, src[: min(n, 64)], eps, k=cfg.k, dtype=a.dtype, slots=a.slots or None,
                            stream=stream.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = bh.bhpp_query_batch(g, meta, src, eps, k=cfg.k, dtype=a.dtype, slots=a.slots or None,
                                  stream=stream.cuda_stream)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        st = _capi.device_graph(g, a.dtype).last_run_stats()
        run.update(ms=ms, queries_per_s=n / (ms / 1e3), rounds=st["rounds"], slots=st["slots"])
        tr = res.traces
        run["trace_mean"] = {k: float(tr[k].mean()) for k in ("sel_b", "seq_b", "sel_f", "pi_iters")}
        run["n_p_f_mean"] = float(tr["n_p_f"].mean())
        # ---- parity on the first P sources
        if a.parity > 0:
            P = min(a.parity, n)
            eb = meta.eps_split_policy(eps)
            t0 = time.perf_counter()
            ref = og.bhpp_query_many(src[:P], cfg.alpha, meta.lam, eb, eps - eb, threads=min(P, os.cpu_count()))
            run["oracle_s"] = time.perf_counter() - t0
            ties = np.array([O.tie_skip_for(t["forward"]) for _, t in ref], dtype=np.int32)
            r64 = bh.bhpp_query_batch(g, meta, src[:P], eps, k=cfg.k, dtype="fp64", return_scores=True,
                                      tie_skip=ties)
            worst64, traces_ok, topk32_rel, sets32, topk32_abs = 0.0, True, 0.0, True, 0.0
            for i, (scores, t) in enumerate(ref):
                worst64 = max(worst64, float(np.abs(r64.scores[i] - scores).max()))
                got = r64.trace_dicts(i)
                fwd = {kk: v for kk, v in t["forward"].items() if kk not in ("tie_checks", "tie_break_at", "gamma")}
                traces_ok &= got["backward"] == t["backward"] and \
                    {kk: v for kk, v in got["forward"].items() if kk != "gamma"} == fwd
                top = O.topk_indices(scores, cfg.k)
                rel = np.abs(res.topk_score[i] - scores[top]) / np.maximum(np.abs(scores[top]), 1e-300)
                topk32_rel = max(topk32_rel, float(rel.max()))
                topk32_abs = max(topk32_abs, float(np.abs(res.topk_score[i] - scores[top]).max()))
                diff = res.topk_index[i] != top
                if diff.any():
                    gap = np.abs(scores[res.topk_index[i][diff]] - scores[top[diff]]).max()
                    sets32 &= bool(gap <= 1e-5 * scores[top[-1]] + eps)
            run["parity"] = {"sources": P, "fp64_max_abs_err": worst64, "fp64_traces_identical": bool(traces_ok),
                             f"{a.dtype}_topk_max_rel_err": topk32_rel, f"{a.dtype}_topk_sets_equal_up_to_ties": sets32,
                             f"{a.dtype}_topk_max_abs_err": topk32_abs, f"{a.dtype}_topk_abs_err_over_eps": topk32_abs / eps,
                             "pass": bool(worst64 <= 1e-9 and traces_ok and topk32_rel <= 1e-5 and sets32)}
        out["runs"].append(run)
        print(json.dumps(run), file=sys.stderr, flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
