"""Per-kernel breakdown of a c5-style run (all-sources sweep: slots refilled
every round) -- eager rounds with CUDA events per kernel, and graph-mode time.

    python tools/c5_profile.py [--n 4096] [--eps 1e-6]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import _capi
from paper_2312_06724_b200.synth import CONFIGS, make_graph

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--eps", type=float, default=1e-6)
ap.add_argument("--slots", type=int, default=0)
a = ap.parse_args()
cfg = CONFIGS["c5"]
g = make_graph(cfg)
meta = bh.build_index_meta(g, cfg.alpha)
src = np.arange(a.n, dtype=np.int64)
kw = dict(k=cfg.k, dtype="fp32", slots=a.slots or None)
bh.bhpp_query_batch(g, meta, src[:256], a.eps, **kw)
torch.cuda.synchronize()
t0 = time.perf_counter()
r = bh.bhpp_query_batch(g, meta, src, a.eps, **kw)
t1 = time.perf_counter()
dg = _capi.device_graph(g, "fp32")
st = dg.last_run_stats()
print(f"graph mode: {a.n / (t1 - t0):.1f} queries/s, {st['rounds']} rounds, slots {st['slots']}, "
      f"{(t1 - t0) / max(1, st['rounds']) * 1e6:.1f} us/round")
_capi.set_profiling(True)
t0 = time.perf_counter()
bh.bhpp_query_batch(g, meta, src, a.eps, **kw)
t1 = time.perf_counter()
_capi.set_profiling(False)
st = dg.last_run_stats()
rounds = max(1, st["rounds"])
print(f"eager+events: {a.n / (t1 - t0):.1f} q/s; per round us: prep {st['ms_prep'] / rounds * 1e3:.1f}, "
      f"V {st['ms_vpull'] / rounds * 1e3:.1f}, U {st['ms_upull'] / rounds * 1e3:.1f}, "
      f"control(K4+K5) {st['ms_control'] / rounds * 1e3:.1f}")
