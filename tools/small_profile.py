"""c1 small path: host-call latency vs device time.

    python tools/small_profile.py
"""
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

cfg = CONFIGS["c1"]
g = make_graph(cfg, device=0)
meta = bh.build_index_meta(g, cfg.alpha)
src = bench_sources(cfg.u_count, 64)
eps = 1e-6
for dtype in ("fp64", "fp32"):
    bh.bhpp_query_batch(g, meta, src[:1], eps, k=10, dtype=dtype)
    ts = []
    for s in src[:32]:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bh.bhpp_query_batch(g, meta, [s], eps, k=10, dtype=dtype)
        ts.append(time.perf_counter() - t0)
    one = float(np.median(ts))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bh.bhpp_query_batch(g, meta, src, eps, k=10, dtype=dtype)
    torch.cuda.synchronize()
    batch = time.perf_counter() - t0
    # device time of one query through the device-pointer API, CUDA events
    dg = _capi.device_graph(g, dtype)
    eb = meta.eps_split_policy(eps)
    dev = torch.device("cuda")
    s_t = torch.tensor([int(src[0])], dtype=torch.int32, device=dev)
    ti = torch.empty((1, 10), dtype=torch.int32, device=dev)
    tsc = torch.empty((1, 10), dtype=torch.float64, device=dev)
    tr = torch.empty((1, 96), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dts, walls = [], []
    for _ in range(10):
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record(st)
        query_batch_device(dg, meta, eb, eps - eb, s_t.data_ptr(), 1, 10, ti.data_ptr(), tsc.data_ptr(), tr.data_ptr(),
                           stream=st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - w0)
        dts.append(e0.elapsed_time(e1))
    print(f"{dtype}: public call {one*1e3:.3f} ms/query; 64-query batch {batch*1e3:.3f} ms ({64/batch:.0f} q/s); "
          f"device-pointer call: device {np.median(dts):.3f} ms, wall {np.median(walls)*1e3:.3f} ms", flush=True)
