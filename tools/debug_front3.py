import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import _capi, push_engine as pe
from golden_io import config_graph, load
g = config_graph("c1")
meta = bh.build_index_meta(g, 0.15)
os.environ["BH_NO_GRAPH"] = "1"
os.environ["BH_FRONT_DEBUG"] = "1"
for lim in (10.0, -1.0):
    pe._SCATTER_LIMIT = lim
    print("LIMIT", lim, file=sys.stderr, flush=True)
    r = bh.bhpp_query_batch(g, meta, [0], 1e-6, k=10, dtype="fp64", return_scores=True, slots=1)
    print(lim, r.trace_dicts(0), r.scores[:4], file=sys.stderr, flush=True)
