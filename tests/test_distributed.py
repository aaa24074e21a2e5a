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


@pytest.mark.parametrize("n_src", [1, 7, 12])
def test_sharded_gather_restores_source_order(tmp_path, n_src):
    """Includes fewer sources than ranks (rank 1 has an empty shard)."""
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


def _packed_worker(rank, world, port, n_total, k, out_path):
    """The device path's driver (sharded_run + PackedShard) with a local_fn that
    writes each query's rows straight into the packed send buffer, as K5 does."""
    import torch

    from paper_2312_06724_b200.distributed import sharded_run

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def local(lo, count, packed):
            q = torch.arange(lo, n_total, world, dtype=torch.int64)[:count]
            packed.idx[:count] = (q[:, None] * 100 + torch.arange(k)[None, :]).to(torch.int32)
            packed.score[:count] = q[:, None].double() + torch.arange(k)[None, :].double() / 1000
            packed.trace[:count] = (q[:, None] % 251).to(torch.uint8)

        gi, gs, gt = sharded_run(n_total, k, rank, world, local)
        if rank == 0:
            np.savez(out_path, idx=gi.numpy(), sc=gs.numpy(), tr=gt.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [0, 1, 5, 8])
def test_packed_all_gather_restores_source_order(tmp_path, n_total):
    k = 3
    out = tmp_path / "packed.npz"
    mp.spawn(_packed_worker, args=(2, _free_port(), n_total, k, str(out)), nprocs=2, join=True)
    got = np.load(out)
    q = np.arange(n_total)
    np.testing.assert_array_equal(got["idx"], (q[:, None] * 100 + np.arange(k)[None, :]).astype(np.int32))
    np.testing.assert_array_equal(got["sc"], q[:, None] + np.arange(k)[None, :] / 1000)
    assert got["tr"].shape == (n_total, _capi.TRACE_DTYPE.itemsize)
    np.testing.assert_array_equal(got["tr"], np.broadcast_to((q % 251)[:, None], got["tr"].shape).astype(np.uint8))


def test_source_order_index():
    from paper_2312_06724_b200.distributed import per_rank, source_order_index

    assert per_rank(7, 2) == 4 and per_rank(0, 3) == 0
    # 7 queries over 2 ranks: rank 0 holds 0,2,4,6 (rows 0..3), rank 1 holds 1,3,5 (rows 4..6)
    assert list(source_order_index(7, 2)) == [0, 4, 1, 5, 2, 6, 3]


def test_shard_interleaves():
    s = np.arange(10)
    assert list(shard(s, 0, 3)) == [0, 3, 6, 9]
    assert list(shard(s, 2, 3)) == [2, 5, 8]
    assert sum(len(shard(s, r, 4)) for r in range(4)) == 10
