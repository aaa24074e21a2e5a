"""Step time of the bench workload with and without per-kernel profiling events."""
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

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dtype = sys.argv[2] if len(sys.argv) > 2 else "fp32"
slots = int(sys.argv[3]) if len(sys.argv) > 3 else 0
g = make_graph(cfg)
meta = bh.build_index_meta(g, cfg.alpha)
src = bench_sources(cfg.u_count, cfg.n_sources)
eps = cfg.epsilons[0]
eb = meta.eps_split_policy(eps)
dg = _capi.device_graph(g, dtype)
dev = torch.device("cuda")
n, k = len(src), cfg.k
src_t = torch.from_numpy(src.astype(np.int32)).to(dev)
tk_i = torch.empty((n, k), dtype=torch.int32, device=dev)
tk_s = torch.empty((n, k), dtype=torch.float64, device=dev)
tr = torch.empty((n, 80), dtype=torch.uint8, device=dev)
for stream_kind in ("torch", "engine"):
    st = torch.cuda.Stream() if stream_kind == "torch" else None
    for prof in (False, True, False):
        _capi.set_profiling(prof)
        for it in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            query_batch_device(dg, meta, eb, eps - eb, src_t.data_ptr(), n, k, tk_i.data_ptr(), tk_s.data_ptr(),
                               tr.data_ptr(), slots=slots or None, stream=st.cuda_stream if st else None)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        s = dg.last_run_stats()
        print(f"stream={stream_kind} prof={prof} wall_ms={dt*1e3:.1f} rounds={s['rounds']} "
              f"prep={s['ms_prep']:.2f} v={s['ms_vpull']:.2f} u={s['ms_upull']:.2f} ctl={s['ms_control']:.2f}", flush=True)
