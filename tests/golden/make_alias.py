"""Golden alias tables (reference baselines.build_alias, baselines.py:42-83).

Run in the dev container (where /root/reference exists):
    python tests/golden/make_alias.py
Writes alias.npz: build_alias of the config-1 graph and of a small graph with
non-integer weights (the Vose pairing order and the roundoff leftovers matter).
"""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))

import bipush  # noqa: E402

from golden_io import graph_from, load  # noqa: E402  (tests/golden_io.py)

out = {}
g1 = graph_from(load("c1"))
rg = bipush.BipartiteGraph(list(g1.u_labels), list(g1.v_labels), np.repeat(np.arange(g1.u_count), np.diff(g1.u_indptr)),
                           g1.u_indices, g1.u_weights)
rng = np.random.default_rng(9)
eu = np.r_[np.arange(60), rng.integers(0, 60, 400)]
ev = np.r_[rng.permutation(np.arange(80))[:60], rng.integers(0, 80, 400)]
ev[:20] = np.arange(60, 80)
key = np.unique(eu * 80 + ev)
eu, ev = key // 80, key % 80
keep_v = np.unique(ev)
remap = {v: i for i, v in enumerate(keep_v.tolist())}
ev = np.array([remap[v] for v in ev.tolist()])
ew = rng.random(eu.size) * 3 + 0.05
g2 = bipush.BipartiteGraph([f"a{i}" for i in range(60)], [f"b{i}" for i in range(len(keep_v))], eu, ev, ew)
for name, g in (("c1", rg), ("w", g2)):
    t = bipush.build_alias(g)
    out[f"{name}_u_prob"], out[f"{name}_u_alias"] = t.u_prob, t.u_alias
    out[f"{name}_v_prob"], out[f"{name}_v_alias"] = t.v_prob, t.v_alias
out["w_eu"], out["w_ev"], out["w_ew"] = eu, ev, ew
np.savez_compressed(HERE / "alias.npz", **out)
print("alias.npz:", {k: v.shape for k, v in out.items()})
