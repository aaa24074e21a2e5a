import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import _capi, push_engine as pe
from golden_io import config_graph, load
g = config_graph("c1")
pe._SCATTER_LIMIT = 10.0
os.environ["BH_NO_GRAPH"] = "1"
os.environ["BH_FRONT_DEBUG"] = "1"
ss = bh.ss_push(g, 0, 0.15, 1e-6)
print(ss.phase_trace, ss.terminated_by, ss.ledger.estimate[:5], flush=True)
pe._SCATTER_LIMIT = -1.0
ss2 = bh.ss_push(g, 0, 0.15, 1e-6)
print(ss2.phase_trace, ss2.terminated_by, ss2.ledger.estimate[:5], flush=True)
