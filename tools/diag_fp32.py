"""Where does fp32 lose precision on a config?  fp64 vs fp32 batch on a few sources."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = make_graph(cfg)
meta = bh.build_index_meta(g, cfg.alpha)
src = bench_sources(g.u_count, 1024)[:n]
eps = cfg.epsilons[0]
r64 = bh.bhpp_query_batch(g, meta, src, eps, k=cfg.k, dtype="fp64", return_scores=True)
r32 = bh.bhpp_query_batch(g, meta, src, eps, k=cfg.k, dtype="fp32", return_scores=True)
for i in range(n):
    s64, s32 = r64.scores[i], r32.scores[i]
    top = r64.topk_index[i]
    rel = np.abs(s32[top] - s64[top]) / s64[top]
    j = int(np.argmax(rel))
    allrel = np.abs(s32 - s64) / np.maximum(s64, 1e-300)
    big = s64 > 1e-6
    print(f"src {src[i]} deg {g.deg_u[src[i]]} ws {g.ws_u[src[i]]:.0f}: topk max rel {rel.max():.2e} at rank {j} "
          f"(node {top[j]}, deg {g.deg_u[top[j]]}, score {s64[top[j]]:.3e}); median topk rel {np.median(rel):.2e}; "
          f"max rel over scores>1e-6: {allrel[big].max():.2e}")
    print("   traces64", r64.trace_dicts(i))
    print("   traces32", r32.trace_dicts(i))
    est_only = None
