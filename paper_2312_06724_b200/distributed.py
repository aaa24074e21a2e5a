"""Query-batch sharding over the GPUs of one node.

Queries are independent (one ledger per query, a read-only graph), so the
only multi-GPU structure is: replicate the device graph store on every rank,
give rank r the interleaved shard ``sources[r::world]`` (interleaving spreads
hub and leaf sources evenly), run the batch locally, then gather the per-shard
top-k (int32 indices, fp64 scores) and phase traces.  No collective runs
inside the propagation loop; the reference's only concurrency is the host
thread pool over independent queries (cli.py:444-450), which this replaces.

Three forms:

* ``bhpp_query_sharded_device``: one process per GPU (torchrun, NCCL), every
  buffer device-resident.  The engine's finalize kernel (K5) writes each
  shard's top-k and traces straight into its rank's region of ONE packed send
  buffer, one ``all_gather_into_tensor`` moves them, and a device gather puts
  the rows back in source order.  Nothing crosses PCIe.
* ``bhpp_query_sharded``: the same with host numpy sources in and numpy
  results out (the public ``bhpp_query_batch`` contract on every rank).
* ``bhpp_query_multi``: one process driving several GPUs (a host thread per
  device; the C ABI releases the GIL), results merged on the host.

The packing and reordering logic is shared by the CPU tests (gloo, world
size 2, with the oracle standing in for the device batch through
``local_fn``).
"""

from __future__ import annotations

import numpy as np

from . import _capi
from .bhpp_query import BatchResult, _split, bhpp_query_batch, query_batch_device


def shard(sources, rank: int, world: int) -> np.ndarray:
    return np.asarray(sources)[rank::world]


def per_rank(n_total: int, world: int) -> int:
    """Rows each rank's region holds (the largest shard)."""
    return -(-n_total // world) if n_total else 0


def source_order_index(n_total: int, world: int):
    """Row of the gathered [world * per] layout that holds query i: query i is
    row i // world of rank i % world's shard."""
    per = per_rank(n_total, world)
    i = np.arange(n_total)
    return (i % world) * per + i // world


class PackedShard:
    """One rank's send buffer: [per, k] int32 indices | [per, k] fp64 scores |
    [per, trace] bytes, as one uint8 tensor (8-byte aligned regions), so the
    whole result moves in one all-gather.  ``idx`` / ``score`` / ``trace`` are
    views the engine writes into directly."""

    def __init__(self, per: int, k: int, device):
        import torch

        self.per, self.k = per, k
        tsz = _capi.TRACE_DTYPE.itemsize
        self.b_idx = (per * k * 4 + 7) // 8 * 8
        self.b_sc = per * k * 8
        self.b_tr = per * tsz
        self.nbytes = self.b_idx + self.b_sc + self.b_tr
        self.buf = torch.zeros(max(self.nbytes, 8), dtype=torch.uint8, device=device)
        self.idx = self.buf[: per * k * 4].view(torch.int32).view(per, k)
        self.score = self.buf[self.b_idx: self.b_idx + self.b_sc].view(torch.float64).view(per, k)
        self.trace = self.buf[self.b_idx + self.b_sc: self.nbytes].view(per, tsz)
        self.idx.fill_(-1)

    def unpack(self, gathered, world: int, n_total: int):
        """Split the gathered [world * nbytes] buffer and restore source order:
        (idx [n, k] int32, score [n, k] fp64, trace [n, tsize] uint8), same device."""
        import torch

        g = gathered[: world * max(self.nbytes, 8)].view(world, max(self.nbytes, 8))
        per, k = self.per, self.k
        tsz = _capi.TRACE_DTYPE.itemsize
        gi = g[:, : per * k * 4].contiguous().view(torch.int32).view(world * per, k)
        gs = g[:, self.b_idx: self.b_idx + self.b_sc].contiguous().view(torch.float64).view(world * per, k)
        gt = g[:, self.b_idx + self.b_sc: self.nbytes].contiguous().view(world * per, tsz)
        order = torch.from_numpy(source_order_index(n_total, world)).to(gathered.device)
        return gi.index_select(0, order), gs.index_select(0, order), gt.index_select(0, order)


def sharded_run(n_total: int, k: int, rank: int, world: int, local_fn, device=None, group=None, stream=None):
    """Shared driver: ``local_fn(lo, count, packed)`` computes this rank's
    shard (queries rank, rank + world, ...; ``count`` of them) into
    ``packed.idx/score/trace[:count]``; then one all-gather and the reorder.
    Returns device (or CPU) tensors in source order."""
    import torch
    import torch.distributed as dist

    dev = torch.device(device) if device is not None else torch.device("cpu")
    per = per_rank(n_total, world)
    count = len(range(rank, n_total, world))
    packed = PackedShard(per, k, dev)
    ctx = torch.cuda.stream(stream) if stream is not None else _null()
    with ctx:
        if count:
            local_fn(rank, count, packed)
        out = torch.empty(world * packed.buf.numel(), dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(out, packed.buf, group=group)
        return packed.unpack(out, world, n_total)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def bhpp_query_sharded_device(g, meta, sources, epsilon: float, k: int = 50, exclude_query: bool = False,
                              dtype: str = "fp32", slots: int | None = None, group=None, device=None,
                              stream=None):
    """Device-resident sharded batch over all ranks of ``group`` (NCCL).

    ``sources``: every rank passes the same full list (numpy, or a torch
    tensor on ``device``).  The local batch runs on ``stream`` (a
    torch.cuda.Stream) with its top-k and traces written by the engine into
    this rank's region of the packed send buffer; returns (idx, score, trace)
    CUDA tensors in source order on every rank."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    src = sources if isinstance(sources, torch.Tensor) else torch.as_tensor(np.asarray(sources, dtype=np.int32))
    src = src.to(device=dev, dtype=torch.int32)
    n_total = int(src.numel())
    kk = min(int(k), g.u_count)
    eps_b, eps_f = _split(meta, g, epsilon)
    dg = _capi.device_graph(g, dtype, dev.index)
    st = stream or torch.cuda.current_stream(dev)
    mine = src[rank::world].contiguous()

    def local(lo, count, packed):
        query_batch_device(dg, meta, eps_b, eps_f, mine.data_ptr(), count, kk, packed.idx.data_ptr(),
                           packed.score.data_ptr(), packed.trace.data_ptr(), exclude_query=exclude_query,
                           slots=slots, stream=st.cuda_stream)

    return sharded_run(n_total, kk, rank, world, local, device=dev, group=group, stream=st)


def gather_results(topk_index: np.ndarray, topk_score: np.ndarray, traces: np.ndarray, n_total: int,
                   rank: int, world: int, device=None, group=None):
    """All-gather host shard results and restore the caller's source order.

    Every rank passes its shard's arrays (rows = its queries, possibly none);
    every rank gets the full [n_total, k] arrays back as numpy."""
    k = topk_index.shape[1]

    def local(lo, count, packed):
        import torch

        packed.idx[:count].copy_(torch.from_numpy(np.ascontiguousarray(topk_index, dtype=np.int32)))
        packed.score[:count].copy_(torch.from_numpy(np.ascontiguousarray(topk_score, dtype=np.float64)))
        tb = np.ascontiguousarray(traces).view(np.uint8).reshape(traces.shape[0], traces.dtype.itemsize)
        packed.trace[:count].copy_(torch.from_numpy(tb))

    gi, gs, gt = sharded_run(n_total, k, rank, world, local, device=device, group=group)
    tr = gt.cpu().numpy().copy().view(_capi.TRACE_DTYPE).reshape(-1) if n_total else np.zeros(0, _capi.TRACE_DTYPE)
    return gi.cpu().numpy(), gs.cpu().numpy(), tr


def bhpp_query_sharded(g, meta, sources, epsilon: float, k: int = 50, exclude_query: bool = False,
                       dtype: str = "fp32", slots: int | None = None, group=None, device=None,
                       local_fn=None) -> BatchResult:
    """bhpp_query_batch over all ranks of ``group``; every rank returns the
    full result (numpy) in the order of ``sources``.  On CUDA devices the
    device-resident path runs; ``local_fn`` (tests, CPU) replaces the local
    device batch with a function of the shard's sources returning a
    BatchResult."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    src = np.asarray(sources, dtype=np.int64)
    if local_fn is None and device is not None and str(device).startswith("cuda"):
        if src.size and (src.min() < 0 or src.max() >= g.u_count):
            raise ValueError("node index out of range")
        eps_b, eps_f = _split(meta, g, epsilon)
        gi, gs, gt = bhpp_query_sharded_device(g, meta, src, epsilon, k=k, exclude_query=exclude_query,
                                               dtype=dtype, slots=slots, group=group, device=device)
        tr = gt.cpu().numpy().copy().view(_capi.TRACE_DTYPE).reshape(-1)
        kk = min(int(k), g.u_count)
        return BatchResult(sources=src.astype(np.int32), epsilon=epsilon, epsilon_b=eps_b, epsilon_f=eps_f, k=kk,
                           topk_index=gi.cpu().numpy(), topk_score=gs.cpu().numpy(), traces=tr, scores=None,
                           timing={}, dtype=dtype, meta={"world": world, "rank": rank, "path": "device"})
    mine = shard(src, rank, world)
    run = local_fn or (lambda s: bhpp_query_batch(g, meta, s, epsilon, k=k, exclude_query=exclude_query,
                                                  dtype=dtype, slots=slots))
    loc = run(mine)
    idx, sc, tr = gather_results(loc.topk_index, loc.topk_score, loc.traces, src.size, rank, world,
                                 device=device, group=group)
    return BatchResult(sources=src.astype(np.int32), epsilon=epsilon, epsilon_b=loc.epsilon_b,
                       epsilon_f=loc.epsilon_f, k=loc.k, topk_index=idx, topk_score=sc, traces=tr, scores=None,
                       timing=dict(loc.timing), dtype=dtype, meta={"world": world, "rank": rank, "path": "host"})


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
    if src.size == 0:  # nothing to shard: the single-device call's empty result
        return bhpp_query_batch(g, meta, src, epsilon, k=k, exclude_query=exclude_query, dtype=dtype,
                                return_scores=return_scores, slots=slots, device=devices[0])
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


def trace_dtype():
    return _capi.TRACE_DTYPE
