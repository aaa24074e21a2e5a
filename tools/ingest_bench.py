"""Graph ingestion: host (numpy sorts) vs device (bh_csr_build) canonicalisation.

    python tools/ingest_bench.py [--configs c2,c3] [--no-host]

For each config: the seeded Chung-Lu edge list (not timed beyond its own
line), then BipartiteGraph.from_arrays on the host and on cuda:0 (host arrays
in, host arrays out: upload, two radix sorts, CSR, ws sums, download), the
bitwise comparison of the two, and the BPGR load (from_bytes) both ways.
Prints one JSON line per config.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np

from paper_2312_06724_b200 import BipartiteGraph
from paper_2312_06724_b200.synth import CONFIGS, chung_lu_edges

FIELDS = ("u_indptr", "u_indices", "u_weights", "v_indptr", "v_indices", "v_weights", "ws_u", "ws_v")

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c3")
ap.add_argument("--no-host", action="store_true")
a = ap.parse_args()
for name in a.configs.split(","):
    c = CONFIGS[name]
    out = {"config": name, "edges": c.edge_count}
    t = time.perf_counter()
    eu, ev, ew = chung_lu_edges(c.u_count, c.v_count, c.edge_count, c.beta_u, c.beta_v, c.weights, c.seed,
                                c.max_deg_v)
    out["generate_s"] = time.perf_counter() - t
    BipartiteGraph.from_arrays(1, 1, [0], [0], [1.0], device=0)  # context + module load
    t = time.perf_counter()
    d = BipartiteGraph.from_arrays(c.u_count, c.v_count, eu, ev, ew, device=0)
    out["device_build_s"] = time.perf_counter() - t
    out["device_edges_per_s"] = c.edge_count / out["device_build_s"]
    if not a.no_host:
        t = time.perf_counter()
        h = BipartiteGraph.from_arrays(c.u_count, c.v_count, eu, ev, ew)
        out["host_build_s"] = time.perf_counter() - t
        out["host_edges_per_s"] = c.edge_count / out["host_build_s"]
        out["speedup"] = out["host_build_s"] / out["device_build_s"]
        out["bitwise_equal"] = all(np.array_equal(getattr(h, f).view(np.uint8), getattr(d, f).view(np.uint8))
                                   for f in FIELDS)
    buf = d.to_bytes()
    t = time.perf_counter()
    BipartiteGraph.from_bytes(buf, device=0)
    out["bpgr_load_device_s"] = time.perf_counter() - t
    if not a.no_host:
        t = time.perf_counter()
        BipartiteGraph.from_bytes(buf)
        out["bpgr_load_host_s"] = time.perf_counter() - t
    print(json.dumps(out), flush=True)
