"""A/B of engine variants on one BASELINE config, one graph build per process.

    python tools/variants.py --config c3 --n 256 --variants "BH_RELABEL=0" "BH_L2_PERSIST_MB=0" "" \
        [--slots 64 128] [--eps 1e-7] [--dtype fp32]

Each variant (space-separated VAR=VALUE settings, "" = defaults) gets a fresh
device graph store and engine (the switches are read at creation), runs the
batch once untimed, then timed (CUDA events, device-resident sources and
outputs), then once more with per-kernel events.  Prints one JSON line per
(variant, slots) with queries/s, the per-round kernel breakdown and whether
the top-k matches the first variant's.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import _capi
from paper_2312_06724_b200.bhpp_query import query_batch_device
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--eps", type=float, default=0.0)
    ap.add_argument("--dtype", default="fp32")
    ap.add_argument("--slots", type=int, nargs="*", default=[0])
    ap.add_argument("--variants", nargs="*", default=[""])
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    t0 = time.perf_counter()
    g = make_graph(cfg, device=0)
    t_graph = time.perf_counter() - t0
    t0 = time.perf_counter()
    meta = bh.build_index_meta(g, cfg.alpha)
    t_meta = time.perf_counter() - t0
    print(json.dumps({"config": cfg.name, "graph_s": round(t_graph, 1), "meta_s": round(t_meta, 1),
                      "lam": meta.lam, "max_deg_u": int(g.deg_u.max()), "max_deg_v": int(g.deg_v.max())}), flush=True)
    eps = a.eps or cfg.epsilons[0]
    eps_b = float(meta.eps_split_policy(eps))
    eps_f = eps - eps_b
    n = a.n
    src = bench_sources(cfg.u_count, n)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream()
    src_t = torch.from_numpy(src.astype(np.int32)).to(dev)
    k = cfg.k
    first_top = None
    for var in a.variants:
        env = dict(kv.split("=", 1) for kv in var.split() if kv)
        old = {kk: os.environ.get(kk) for kk in env}
        os.environ.update(env)
        try:
            dg = _capi.DeviceGraph(g, a.dtype, 0)
            for slots in a.slots:
                tk_i = torch.empty((n, k), dtype=torch.int32, device=dev)
                tk_s = torch.empty((n, k), dtype=torch.float64, device=dev)
                tr = torch.empty((n, _capi.TRACE_DTYPE.itemsize), dtype=torch.uint8, device=dev)

                def run():
                    query_batch_device(dg, meta, eps_b, eps_f, src_t.data_ptr(), n, k, tk_i.data_ptr(),
                                       tk_s.data_ptr(), tr.data_ptr(), slots=slots or None, stream=st.cuda_stream)

                run()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                run()
                e1.record(st)
                e1.synchronize()
                ms = e0.elapsed_time(e1)
                stats = dg.last_run_stats()
                _capi.set_profiling(True)
                run()
                torch.cuda.synchronize()
                _capi.set_profiling(False)
                p = dg.last_run_stats()
                rounds = max(1, p["rounds"])
                top = tk_i.cpu().numpy()
                if first_top is None:
                    first_top = top
                out = {"variant": var or "default", "slots": int(stats["slots"]), "n": n, "eps": eps,
                       "qps": round(n / (ms / 1e3), 2), "ms": round(ms, 1), "rounds": int(stats["rounds"]),
                       "us_per_round": {"prep": round(p["ms_prep"] * 1e3 / rounds, 1),
                                        "vpull": round(p["ms_vpull"] * 1e3 / rounds, 1),
                                        "upull": round(p["ms_upull"] * 1e3 / rounds, 1),
                                        "control": round(p["ms_control"] * 1e3 / rounds, 1)},
                       "topk_same_as_first": bool(np.array_equal(top, first_top)),
                       "topk_overlap_first": float(np.mean([len(set(x) & set(y)) / k for x, y in zip(top, first_top)]))}
                print(json.dumps(out), flush=True)
            dg.close()
        finally:
            for kk, v in old.items():
                if v is None:
                    os.environ.pop(kk, None)
                else:
                    os.environ[kk] = v


if __name__ == "__main__":
    main()
