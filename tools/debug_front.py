"""Frontier-mode debug: max |scores - golden| per (graph, slots, eager, limit)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import _capi, push_engine as pe
from golden_io import config_graph, load
from test_gpu_parity import tie_skip_from

for name, alpha in (("c1", 0.15), ("c2s", 0.15)):
    d = load(name)
    g = config_graph(name)
    print(name, "max deg u", int(np.diff(g.u_indptr).max()), "v", int(np.diff(g.v_indptr).max()), flush=True)
    meta = bh.build_index_meta(g, alpha)
    srcs = d["sources"][:4]
    ties = np.array([tie_skip_from(t) for t in d["ties"][:4]], dtype=np.int32)
    for eager in (False, True):
        if eager: os.environ["BH_NO_GRAPH"] = "1"
        else: os.environ.pop("BH_NO_GRAPH", None)
        for slots in (1, 4, 64):
            for lim in (-1.0, 10.0):
                pe._SCATTER_LIMIT = lim
                try:
                    r = bh.bhpp_query_batch(g, meta, srcs, float(d["eps"]), k=10, dtype="fp64", return_scores=True,
                                            tie_skip=ties, slots=slots)
                    err = max(float(np.abs(r.scores[i] - d["scores"][i]).max()) for i in range(len(srcs)))
                    st = _capi.device_graph(g, "fp64").last_run_stats()
                    print(f"  eager={eager} slots={slots} lim={lim}: err={err:.3e} rounds={st['rounds']} "
                          f"front={st['frontier_rounds']} ufront={st['frontier_u_rounds']}", flush=True)
                except Exception as e:
                    print(f"  eager={eager} slots={slots} lim={lim}: EXC {e}", flush=True)
