"""One single-source c2 query through the slot engine with frontier rounds forced
(for ncu captures of the K-F kernels): python tools/front_step.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import push_engine as pe
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

cfg = CONFIGS["c2"]
g = make_graph(cfg, device=0)
meta = bh.build_index_meta(g, cfg.alpha)
src = bench_sources(cfg.u_count, 2)
pe._SCATTER_LIMIT = 10.0
bh.bhpp_query_batch(g, meta, src[:1], 1e-7, k=50, dtype="fp32", slots=1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
bh.bhpp_query_batch(g, meta, src[1:2], 1e-7, k=50, dtype="fp32", slots=1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
