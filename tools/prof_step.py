"""One bench step under a profiler range (for ncu --profile-from-start off).

    python tools/prof_step.py [--config c2] [--dtype fp32] [--slots 0]
Builds the config graph and IndexMeta, runs one warm-up batch, then one
batch inside cudaProfilerStart/Stop.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--dtype", default="fp32")
ap.add_argument("--slots", type=int, default=0)
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
cfg = CONFIGS[a.config]
g = make_graph(cfg, device=0)
meta = bh.build_index_meta(g, cfg.alpha)
src = bench_sources(cfg.u_count, a.n or cfg.n_sources or 64)
eps = cfg.epsilons[0]
bh.bhpp_query_batch(g, meta, src, eps, k=cfg.k, dtype=a.dtype, slots=a.slots or None)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = bh.bhpp_query_batch(g, meta, src, eps, k=cfg.k, dtype=a.dtype, slots=a.slots or None)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("rounds/query sample", r.trace_dicts(0), "time", r.timing)
