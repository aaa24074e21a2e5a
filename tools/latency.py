"""Single-query latency (the reference's own API: bhpp_query one source at a
time) with frontier rounds on (default _SCATTER_LIMIT = 0.25) and off (-1).

    python tools/latency.py [--configs c1 c2 c3] [--n 8]
Prints one JSON line per (config, path, limit): median ms per query, rounds,
frontier rounds.  c1 also through the one-CTA small path.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import _capi
from paper_2312_06724_b200 import push_engine as pe
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="*", default=["c1", "c2", "c3"])
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--dtype", default="fp64")
ap.add_argument("--limits", nargs="*", type=float, default=[0.25, -1.0])
a = ap.parse_args()
for name in a.configs:
    cfg = CONFIGS[name]
    g = make_graph(cfg, device=0)
    meta = bh.build_index_meta(g, cfg.alpha)
    eps = cfg.epsilons[0]
    src = bench_sources(cfg.u_count, a.n)
    paths = [("engine", 1)] + ([("small", None)] if name == "c1" else [])
    for path, slots in paths:
        for lim in (a.limits if path == "engine" else a.limits[:1]):
            pe._SCATTER_LIMIT = lim
            bh.bhpp_query_batch(g, meta, src[:1], eps, k=cfg.k, dtype=a.dtype, slots=slots)  # warm
            ts, rounds, fr = [], [], []
            for s in src:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                bh.bhpp_query_batch(g, meta, [s], eps, k=cfg.k, dtype=a.dtype, slots=slots)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
                st = _capi.device_graph(g, a.dtype).last_run_stats()
                rounds.append(st["rounds"])
                fr.append(st["frontier_rounds"])
            print(json.dumps({"config": name, "path": path, "scatter_limit": lim, "dtype": a.dtype,
                              "ms_median": round(1e3 * float(np.median(ts)), 3),
                              "queries_per_s": round(1.0 / float(np.median(ts)), 1),
                              "rounds_mean": float(np.mean(rounds)), "frontier_rounds_mean": float(np.mean(fr))}),
                  flush=True)
