"""Column sequences of the c2 store (both sides, degree-relabelled, CSR order) for tools/gather_bench2."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2312_06724_b200.synth import CONFIGS, make_graph

g = make_graph(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
out = Path(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out")
out.mkdir(exist_ok=True)


def order(indptr):
    deg = np.diff(indptr)
    perm = np.argsort(-deg, kind="stable")  # ties by caller index
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    return perm, inv


pu, iu = order(g.u_indptr)
pv, iv = order(g.v_indptr)


def side(indptr, idx, perm, inv_col):
    rows = [inv_col[idx[indptr[r]:indptr[r + 1]]] for r in perm]
    return np.concatenate(rows).astype(np.int32)


side(g.v_indptr, g.v_indices, pv, iu).tofile(out / "c2_v_cols.bin")
side(g.u_indptr, g.u_indices, pu, iv).tofile(out / "c2_u_cols.bin")
print("dumped", g.edge_count)
