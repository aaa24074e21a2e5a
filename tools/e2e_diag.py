"""Per-step e2e timing at c2 (diagnostic): event interval vs host wall, to
separate device time from host scheduling stalls."""
import os
import sys
import time

import numpy as np
import torch

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

cfg = CONFIGS["c2"]
g = make_graph(cfg)
src = bench_sources(cfg.u_count, 64)
meta = bh.build_index_meta(g, cfg.alpha)
eps = cfg.epsilons[0]
st = torch.cuda.Stream()
if os.environ.get("PIN"):
    os.sched_setaffinity(0, {int(os.environ["PIN"])})
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ts = []
for i in range(n):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    t1 = time.perf_counter()
    r = bh.bhpp_query_batch(g, meta, src, eps, k=50, dtype="fp32", stream=st.cuda_stream)
    e1.record(st)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = np.array(ts)
print(os.environ.get("TAG", ""), "median", np.median(ts), "mean", ts.mean(), "max", ts.max(),
      "n>26ms", int((ts > 26).sum()), np.round(ts, 1).tolist(), flush=True)
