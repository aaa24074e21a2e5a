"""A/B of store-level switches (degree relabelling, L2 persisting window) on one
graph in one process: the device store is rebuilt per setting.

    python tools/ab_store.py --config c3 --n 256 [--settings "BH_RELABEL=0" "BH_RELABEL=1" ...]
Prints queries/s (graph mode, device-synchronised wall) and the per-kernel
breakdown of an event-profiled replay per setting.
"""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import _capi
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--dtype", default="fp32")
ap.add_argument("--slots", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--settings", nargs="*", default=["BH_RELABEL=1", "BH_RELABEL=0", "BH_RELABEL=1 BH_L2_PERSIST_MB=0"])
a = ap.parse_args()
cfg = CONFIGS[a.config]
t0 = time.perf_counter()
g = make_graph(cfg, device=0)
meta = bh.build_index_meta(g, cfg.alpha)
print(f"graph+meta {time.perf_counter() - t0:.1f} s", flush=True)
src = bench_sources(cfg.u_count, a.n)
eps = cfg.epsilons[0]
kw = dict(k=cfg.k, dtype=a.dtype, slots=a.slots or None)
keys = set()
for s in a.settings:
    for kv in s.split():
        keys.add(kv.split("=")[0])
ref = None
for s in a.settings:
    for k in keys:
        os.environ.pop(k, None)
    for kv in s.split():
        k, v = kv.split("=")
        os.environ[k] = v
    _capi._graph_cache.clear()
    torch.cuda.synchronize()
    r = bh.bhpp_query_batch(g, meta, src, eps, **kw)  # build store + engine + graph
    best = 1e30
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = bh.bhpp_query_batch(g, meta, src, eps, **kw)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    same = "" if ref is None else f" topk_same={np.array_equal(ref.topk_index, r.topk_index)}"
    ref = ref or r
    dg = _capi.device_graph(g, a.dtype)
    _capi.set_profiling(True)
    bh.bhpp_query_batch(g, meta, src, eps, **kw)
    _capi.set_profiling(False)
    st = dg.last_run_stats()
    print(f"[{s}] {a.n / best:.2f} q/s ({best * 1e3:.1f} ms) rounds={st['rounds']} slots={st['slots']} "
          f"prep={st['ms_prep']:.1f} v={st['ms_vpull']:.1f} u={st['ms_upull']:.1f} ctl={st['ms_control']:.1f} ms{same}", flush=True)
