"""Compare the SS-Push ledger (fp64 vs fp32 engine) against the forward thresholds."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import push_engine as pe, _capi
from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
g = make_graph(cfg)
meta = bh.build_index_meta(g, cfg.alpha)
q = int(bench_sources(g.u_count, 1024)[1])
eps = cfg.epsilons[0]
eb = meta.eps_split_policy(eps)
ef = eps - eb
theta = (g.ws_u[q] / g.ws_u) * (ef / meta.lam)
for dt in ("fp64", "fp32"):
    (r, est, n_p), _, tr = pe.run_job(g, _capi.JOB_SS_PUSH, q, cfg.alpha, 1.0, eb, 1.0, dtype=dt)
    act = r > theta
    print(dt, "n_p", n_p, "zeros", int((r == 0).sum()), "active", int(act.sum()), "of", g.u_count,
          "min r", r[r > 0].min() if (r > 0).any() else 0, "min r/theta", (r / theta).min(),
          "inactive nodes (idx, r, theta, deg):", [(int(i), r[i], theta[i], int(g.deg_u[i])) for i in np.flatnonzero(~act)[:5]])
