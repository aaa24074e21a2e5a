"""Load the reference-generated golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2312_06724_b200.bigraph import BipartiteGraph
from paper_2312_06724_b200.synth import CONFIGS, make_graph, scaled_config

GOLDEN = Path(__file__).resolve().parent / "golden"
TERMS = ("threshold-met", "budget-switch", "mass-drained")


@lru_cache(maxsize=None)
def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def graph_from(d: dict, prefix: str = "") -> BipartiteGraph:
    n_u, n_v, _ = (int(x) for x in d[prefix + "n"])
    return BipartiteGraph.from_arrays(n_u, n_v, d[prefix + "eu"], d[prefix + "ev"], d[prefix + "ew"])


_CFG = {"c1": CONFIGS["c1"], "c2s": scaled_config("c2", 10, "c2s"), "c4s": scaled_config("c4", 100, "c4s")}


@lru_cache(maxsize=None)
def config_graph(name: str) -> BipartiteGraph:
    d = load(name)
    g = graph_from(d) if "eu" in d else make_graph(_CFG[name])
    assert g.fingerprint == str(d["fingerprint"]), f"{name}: generator drifted from the golden graph"
    return g


def config_alpha(name: str) -> float:
    return _CFG[name].alpha


def trace_dict(vec, forward: bool) -> dict:
    d = {
        "selective_rounds": int(vec[0]),
        "sequential_rounds": int(vec[1]),
        "power_iterations": int(vec[2]),
        "n_p": int(vec[3]),
        "terminated_by": TERMS[int(vec[4])],
    }
    return d


def split_traces(row):
    """c*.npz `traces` row -> (backward dict, forward dict, gamma)."""
    return trace_dict(row[0:5], False), trace_dict(row[5:10], True), float(row[10])
