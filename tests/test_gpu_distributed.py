"""GPU: query-batch sharding with two ranks on this box's one GPU.

Both ranks run the CUDA engine on cuda:0 (each process its own device graph
store and engine) and exchange their packed shard results with one
all-gather.  NCCL refuses two ranks on one device, so the exchange here runs
over gloo; with one GPU per rank the same calls run over NCCL (bench.py
--gpus N).  The sharded result must equal one single-process call bitwise:
the interleaved shards, the packed all-gather and the reorder may not change
a single byte (cli.py:444-450 is the loop this replaces).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_src, out_path, device_path):
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(repo))
    sys.path.insert(0, str(repo / "tests"))
    import torch
    import torch.distributed as dist

    import paper_2312_06724_b200 as bh
    from golden_io import config_graph
    from paper_2312_06724_b200.distributed import bhpp_query_sharded, bhpp_query_sharded_device

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = config_graph("c2s")
        meta = bh.build_index_meta(g, 0.15)
        src = np.random.default_rng(5).choice(g.u_count, n_src, replace=False)
        res = bhpp_query_sharded(g, meta, src, 1e-7, k=20, dtype="fp32", slots=16, local_fn=None)
        if device_path:
            gi, gs, gt = bhpp_query_sharded_device(g, meta, src, 1e-7, k=20, dtype="fp32", slots=16,
                                                   device="cuda:0")
            dev = (gi.cpu().numpy(), gs.cpu().numpy(), gt.cpu().numpy())
        if rank == 0:
            one = bh.bhpp_query_batch(g, meta, src, 1e-7, k=20, dtype="fp32", slots=16)
            out = dict(idx=res.topk_index, sc=res.topk_score, tr=res.traces.view(np.uint8),
                       one_idx=one.topk_index, one_sc=one.topk_score, one_tr=one.traces.view(np.uint8))
            if device_path:
                out.update(d_idx=dev[0], d_sc=dev[1], d_tr=dev[2])
            np.savez(out_path, **out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_src", [1, 13])
def test_two_ranks_on_one_gpu_match_one_call(tmp_path, n_src):
    """Host-API sharding (bhpp_query_sharded: numpy in / out) with 2 ranks,
    including fewer sources than ranks; equal to one call byte for byte."""
    out = tmp_path / "res.npz"
    mp.spawn(_worker, args=(2, _free_port(), n_src, str(out), False), nprocs=2, join=True)
    r = np.load(out)
    np.testing.assert_array_equal(r["idx"], r["one_idx"])
    np.testing.assert_array_equal(r["sc"], r["one_sc"])
    assert r["tr"].tobytes() == r["one_tr"].tobytes()


def test_two_ranks_device_resident_path(tmp_path):
    """bhpp_query_sharded_device: the engine writes each shard into its
    region of the packed send buffer on the GPU, one all-gather, device
    reorder; equal to one call byte for byte."""
    out = tmp_path / "res.npz"
    mp.spawn(_worker, args=(2, _free_port(), 13, str(out), True), nprocs=2, join=True)
    r = np.load(out)
    np.testing.assert_array_equal(r["d_idx"], r["one_idx"])
    np.testing.assert_array_equal(r["d_sc"], r["one_sc"])
    assert r["d_tr"].tobytes() == r["one_tr"].tobytes()
