"""c1 small path: per-phase cycles of CTA 0 (BH_SMALL_PROF), fp64 and fp32."""
import os, sys
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
os.environ["BH_SMALL_PROF"] = "1"
import paper_2312_06724_b200 as bh
from paper_2312_06724_b200.synth import CONFIGS, make_graph
g = make_graph("c1", device=0); meta = bh.build_index_meta(g, 0.15)
for dt in ("fp64", "fp32"):
    for _ in range(2):
        bh.bhpp_query_batch(g, meta, [0], 1e-6, k=10, dtype=dt)
