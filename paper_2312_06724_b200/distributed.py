"""Query-batch sharding over the GPUs of one node.

Two forms: ``bhpp_query_sharded`` for one process per GPU (torchrun, NCCL
all-gather), and ``bhpp_query_multi`` for one process driving several GPUs
(a host thread per device; the C ABI releases the GIL, results are merged on
the host).

Queries are independent (one ledger per query, a read-only graph), so the
only multi-GPU structure is: replicate the device graph store on every rank,
give rank r the interleaved shard ``sources[r::world]`` (interleaving spreads
hub and leaf sources evenly), run the batch locally, then gather the per-shard
top-k (int32 indices, fp64 scores) and phase traces with one all-gather.  No
collective runs inside the propagation loop.  One process per GPU; the
collective is torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np

from . import _capi
from .bhpp_query import BatchResult, bhpp_query_batch


def shard(sources, rank: int, world: int) -> np.ndarray:
    return np.asarray(sources)[rank::world]


def _pad_rows(a: np.ndarray, rows: int, fill):
    out = np.full((rows,) + a.shape[1:], fill, dtype=a.dtype)
    out[: a.shape[0]] = a
    return out


def gather_results(topk_index: np.ndarray, topk_score: np.ndarray, traces: np.ndarray, n_total: int,
                   rank: int, world: int, device=None, group=None):
    """All-gather the shard results and restore the caller's source order.

    Every rank passes its shard's arrays (rows = its queries); every rank gets
    the full [n_total, k] arrays back.  ``device`` is the torch device the
    collective runs on (a CUDA device for NCCL, None/cpu for gloo)."""
    import torch
    import torch.distributed as dist

    per = -(-n_total // world)
    k = topk_index.shape[1]
    tbytes = traces.view(np.uint8).reshape(traces.shape[0], -1)
    dev = torch.device(device) if device is not None else torch.device("cpu")
    loc_i = torch.from_numpy(_pad_rows(topk_index.astype(np.int32), per, -1)).to(dev)
    loc_s = torch.from_numpy(_pad_rows(topk_score.astype(np.float64), per, 0.0)).to(dev)
    loc_t = torch.from_numpy(_pad_rows(tbytes, per, 0)).to(dev)
    all_i = torch.empty((world * per, k), dtype=torch.int32, device=dev)
    all_s = torch.empty((world * per, k), dtype=torch.float64, device=dev)
    all_t = torch.empty((world * per, tbytes.shape[1]), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(all_i, loc_i, group=group)
    dist.all_gather_into_tensor(all_s, loc_s, group=group)
    dist.all_gather_into_tensor(all_t, loc_t, group=group)
    gi, gs, gt = all_i.cpu().numpy(), all_s.cpu().numpy(), all_t.cpu().numpy()
    idx = np.empty((n_total, k), dtype=np.int32)
    sc = np.empty((n_total, k))
    tr = np.empty(n_total, dtype=traces.dtype)
    for r in range(world):
        rows = np.arange(r, n_total, world)
        idx[rows] = gi[r * per: r * per + rows.size]
        sc[rows] = gs[r * per: r * per + rows.size]
        tr[rows] = gt[r * per: r * per + rows.size].copy().view(traces.dtype).reshape(-1)
    return idx, sc, tr


def bhpp_query_sharded(g, meta, sources, epsilon: float, k: int = 50, exclude_query: bool = False,
                       dtype: str = "fp32", slots: int | None = None, group=None, device=None,
                       local_fn=None) -> BatchResult:
    """bhpp_query_batch over all ranks of ``group``; every rank returns the
    full result in the order of ``sources``.  ``local_fn`` replaces the local
    device batch (tests drive the gather logic on CPU with it)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    src = np.asarray(sources, dtype=np.int64)
    mine = shard(src, rank, world)
    run = local_fn or (lambda s: bhpp_query_batch(g, meta, s, epsilon, k=k, exclude_query=exclude_query,
                                                  dtype=dtype, slots=slots))
    loc = run(mine)
    idx, sc, tr = gather_results(loc.topk_index, loc.topk_score, loc.traces, src.size, rank, world,
                                 device=device, group=group)
    return BatchResult(sources=src.astype(np.int32), epsilon=epsilon, epsilon_b=loc.epsilon_b,
                       epsilon_f=loc.epsilon_f, k=loc.k, topk_index=idx, topk_score=sc, traces=tr, scores=None,
                       timing=dict(loc.timing), dtype=dtype, meta={"world": world, "rank": rank})


def trace_dtype():
    return _capi.TRACE_DTYPE


def bhpp_query_multi(g, meta, sources, epsilon: float, k: int = 50, exclude_query: bool = False,
                     dtype: str = "fp32", slots: int | None = None, devices=None,
                     return_scores: bool = False) -> BatchResult:
    """bhpp_query_batch sharded over ``devices`` (default: every visible GPU)
    from one process: device d runs the interleaved shard sources[i::n] on its
    own replica of the graph store, concurrently; the result is in the order of
    ``sources``, identical to a single-device call."""
    from concurrent.futures import ThreadPoolExecutor

    if devices is None:
        import torch

        devices = list(range(max(1, torch.cuda.device_count())))
    devices = [int(d) for d in devices]
    src = np.asarray(sources, dtype=np.int64)
    n = len(devices)
    for d in set(devices):  # build each replica once, before the threads race for it
        _capi.device_graph(g, dtype, d)

    def run(i):
        mine = shard(src, i, n)
        if mine.size == 0:
            return None
        return bhpp_query_batch(g, meta, mine, epsilon, k=k, exclude_query=exclude_query, dtype=dtype,
                                return_scores=return_scores, slots=slots, device=devices[i])

    with ThreadPoolExecutor(max_workers=n) as pool:
        parts = list(pool.map(run, range(n)))
    first = next(p for p in parts if p is not None)
    kk = first.k
    idx = np.full((src.size, max(kk, 1)), -1, dtype=np.int32)[:, :kk]
    sc = np.zeros((src.size, max(kk, 1)))[:, :kk]
    tr = np.zeros(src.size, dtype=_capi.TRACE_DTYPE)
    scores = np.empty((src.size, g.u_count)) if return_scores else None
    for i, part in enumerate(parts):
        if part is None:
            continue
        rows = np.arange(i, src.size, n)
        idx[rows] = part.topk_index
        sc[rows] = part.topk_score
        tr[rows] = part.traces
        if return_scores:
            scores[rows] = part.scores
    return BatchResult(sources=src.astype(np.int32), epsilon=epsilon, epsilon_b=first.epsilon_b,
                       epsilon_f=first.epsilon_f, k=kk, topk_index=idx, topk_score=sc, traces=tr, scores=scores,
                       timing={"total": max(p.timing["total"] for p in parts if p is not None)}, dtype=dtype,
                       meta={"devices": devices})
