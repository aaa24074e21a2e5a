"""Multi-rank query sharding on CPU (gloo, world_size 2).

The device batch is replaced by the oracle through ``local_fn`` so the host
logic of the multi-GPU path -- interleaved sharding, padding, the all-gather of
top-k indices / scores / traces and the restoration of source order -- runs
here without GPUs.  The GPU path uses the same code with NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_06724_b200 import _capi
from paper_2312_06724_b200.bhpp_query import BatchResult
from paper_2312_06724_b200.distributed import bhpp_query_sharded, shard

K = 10


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_batch(sources):
    """What the device batch returns, computed by the C oracle."""
    from golden_io import config_graph
    from oracle import cpu_oracle as O

    g = config_graph("c1")
    og = O.OracleGraph(g)
    m = O.index_meta(g, 0.15)
    eb = O.choose_eps_b(1e-6, m["mu"])
    idx = np.full((len(sources), K), -1, dtype=np.int32)
    sc = np.zeros((len(sources), K))
    tr = np.zeros(len(sources), dtype=_capi.TRACE_DTYPE)
    for i, q in enumerate(sources):
        scores, t = og.bhpp_query(int(q), 0.15, m["lam"], eb, 1e-6 - eb)
        top = O.topk_indices(scores, K)
        idx[i, : top.size] = top
        sc[i, : top.size] = scores[top]
        tr[i]["sel_b"] = t["backward"]["selective_rounds"]
        tr[i]["sel_f"] = t["forward"]["selective_rounds"]
        tr[i]["pi_iters"] = t["forward"]["power_iterations"]
        tr[i]["n_p_f"] = t["forward"]["n_p"]
        tr[i]["source"] = q
    return BatchResult(np.asarray(sources, dtype=np.int32), 1e-6, eb, 1e-6 - eb, K, idx, sc, tr, None, {}, "fp64")


def _worker(rank, world, port, sources, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = bhpp_query_sharded(None, None, sources, 1e-6, k=K, local_fn=oracle_batch)
        if rank == 0:
            np.savez(out_path, idx=res.topk_index, sc=res.topk_score, tr=res.traces.view(np.uint8))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_src", [7, 12])
def test_sharded_gather_restores_source_order(tmp_path, n_src):
    sources = list(np.random.default_rng(n_src).choice(1000, n_src, replace=False))
    out = tmp_path / "res.npz"
    mp.spawn(_worker, args=(2, _free_port(), sources, str(out)), nprocs=2, join=True)
    got = np.load(out)
    ref = oracle_batch(sources)
    np.testing.assert_array_equal(got["idx"], ref.topk_index)
    np.testing.assert_array_equal(got["sc"], ref.topk_score)
    tr = got["tr"].view(_capi.TRACE_DTYPE)
    np.testing.assert_array_equal(tr["source"], np.asarray(sources, dtype=np.int32))
    np.testing.assert_array_equal(tr["n_p_f"], ref.traces["n_p_f"])


def test_shard_interleaves():
    s = np.arange(10)
    assert list(shard(s, 0, 3)) == [0, 3, 6, 9]
    assert list(shard(s, 2, 3)) == [2, 5, 8]
    assert sum(len(shard(s, r, 4)) for r in range(4)) == 10
