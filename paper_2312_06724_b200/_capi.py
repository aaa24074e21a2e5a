"""ctypes binding of libbhpp.so (include/bhpp.h).

This is the only way the package reaches the device.  There is no CPU
fallback: if the library is missing or no CUDA device is usable, every compute
call raises.  The library is built in-tree by ``python -m
paper_2312_06724_b200.build`` (also ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import threading
import weakref
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libbhpp.so"
if os.environ.get("BH_LIBBHPP"):  # A/B of two in-tree builds (tools/ab_pull.sh)
    LIB_PATH = Path(os.environ["BH_LIBBHPP"]).resolve()

BH_OK, BH_EINVAL, BH_EUNFLUSHED, BH_ECUDA, BH_ENOMEM, BH_EDUP, BH_EFALLBACK = 0, 1, 2, 3, 4, 5, 6
DTYPES = {"fp64": 0, "f64": 0, "float64": 0, "fp32": 1, "f32": 1, "float32": 1}
JOB_BHPP, JOB_SS_PUSH, JOB_SELECTIVE, JOB_PI_PUSH, JOB_POWER = 0, 1, 2, 3, 4
TERMINATIONS = ("threshold-met", "budget-switch", "mass-drained")
PHASES = ("selective", "sequential", "forward-selective")

EXPORTS = (
    "bh_graph_create", "bh_graph_destroy", "bh_graph_get_info", "bh_query_batch", "bh_push_run",
    "bh_power_iteration", "bh_topk", "bh_last_error", "bh_version", "bh_kernel_launches",
    "bh_set_profiling", "bh_last_run_stats", "bh_csr_build", "bh_query_wait", "bh_stream_gate",
    "bh_edge_list_parse", "bh_edge_list_sizes", "bh_edge_list_export", "bh_edge_list_free",
    "bh_alias_create", "bh_monte_carlo", "bh_alias_destroy", "bh_alias_build", "bh_set_scatter_limit",
)
QUERY_ASYNC = 1


class Trace(C.Structure):
    _fields_ = [
        ("sel_b", C.c_int64), ("seq_b", C.c_int64), ("n_p_b", C.c_int64),
        ("sel_f", C.c_int64), ("pi_iters", C.c_int64), ("n_p_f", C.c_int64),
        ("gamma", C.c_double),
        ("term_b", C.c_int32), ("term_f", C.c_int32),
        ("tie_checks", C.c_int32), ("tie_broke", C.c_int32),
        ("source", C.c_int32), ("status", C.c_int32),
        ("near_ties", C.c_int32), ("pad", C.c_int32), ("min_margin", C.c_double),
    ]


TRACE_DTYPE = np.dtype([
    ("sel_b", "<i8"), ("seq_b", "<i8"), ("n_p_b", "<i8"), ("sel_f", "<i8"), ("pi_iters", "<i8"),
    ("n_p_f", "<i8"), ("gamma", "<f8"), ("term_b", "<i4"), ("term_f", "<i4"), ("tie_checks", "<i4"),
    ("tie_broke", "<i4"), ("source", "<i4"), ("status", "<i4"), ("near_ties", "<i4"), ("pad", "<i4"),
    ("min_margin", "<f8"),
])
assert TRACE_DTYPE.itemsize == C.sizeof(Trace)


class QueryParams(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("lam", C.c_double), ("eps_b", C.c_double), ("eps_f", C.c_double),
        ("k", C.c_int32), ("exclude_query", C.c_int32), ("want_scores", C.c_int32),
        ("slots", C.c_int32), ("on_device", C.c_int32), ("flags", C.c_int32),
    ]


class GraphInfo(C.Structure):
    _fields_ = [
        ("n_u", C.c_int64), ("n_v", C.c_int64), ("n_e", C.c_int64),
        ("dtype", C.c_int32), ("device", C.c_int32), ("device_bytes", C.c_int64),
        ("max_deg_u", C.c_int64), ("max_deg_v", C.c_int64),
    ]


class RunStats(C.Structure):
    _fields_ = [
        ("rounds", C.c_int64), ("launches", C.c_int64), ("slots", C.c_int64), ("profiled", C.c_int64),
        ("ms_prep", C.c_double), ("ms_vpull", C.c_double), ("ms_upull", C.c_double), ("ms_control", C.c_double),
        ("frontier_rounds", C.c_int64), ("frontier_u_rounds", C.c_int64),
    ]


HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                   C.c_int64)

_lib = None
_lock = threading.Lock()


def lib():
    """Load libbhpp.so; raise loudly when it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"CUDA extension {LIB_PATH} is not built; run `python -m paper_2312_06724_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        P = C.c_void_p
        L.bh_graph_create.restype = C.c_int
        L.bh_graph_create.argtypes = [C.c_int64] * 3 + [P] * 8 + [C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
        L.bh_graph_destroy.restype = None
        L.bh_graph_destroy.argtypes = [P]
        L.bh_graph_get_info.restype = C.c_int
        L.bh_graph_get_info.argtypes = [P, C.POINTER(GraphInfo)]
        L.bh_query_batch.restype = C.c_int
        L.bh_query_batch.argtypes = [P, C.POINTER(QueryParams), P, C.c_int64, P, P, P, P, P, P]
        L.bh_push_run.restype = C.c_int
        L.bh_push_run.argtypes = [P, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_int32, P, P, P, P, P, HOOK, P]
        L.bh_power_iteration.restype = C.c_int
        L.bh_power_iteration.argtypes = [P, P, C.c_int64, C.c_double, C.c_int32, P]
        L.bh_topk.restype = C.c_int
        L.bh_topk.argtypes = [P, C.c_int64, C.c_int64, C.c_int64, P, P, P]
        L.bh_last_error.restype = C.c_char_p
        L.bh_last_error.argtypes = []
        L.bh_version.restype = C.c_int
        L.bh_kernel_launches.restype = C.c_int64
        L.bh_set_profiling.restype = C.c_int
        L.bh_set_profiling.argtypes = [C.c_int32]
        L.bh_set_scatter_limit.restype = C.c_int
        L.bh_set_scatter_limit.argtypes = [C.c_double]
        L.bh_last_run_stats.restype = C.c_int
        L.bh_last_run_stats.argtypes = [P, C.POINTER(RunStats)]
        L.bh_edge_list_parse.restype = C.c_int
        L.bh_edge_list_parse.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, C.c_int32, C.c_double,
                                         C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
        L.bh_edge_list_sizes.restype = C.c_int
        L.bh_edge_list_sizes.argtypes = [P] + [C.POINTER(C.c_int64)] * 5
        L.bh_edge_list_export.restype = C.c_int
        L.bh_edge_list_export.argtypes = [P, C.c_char_p, P, C.c_char_p, P, P, P, P]
        L.bh_edge_list_free.restype = None
        L.bh_edge_list_free.argtypes = [P]
        L.bh_alias_build.restype = C.c_int
        L.bh_alias_build.argtypes = [C.c_int64, C.c_int64, P, P, C.c_int32, P, P]
        L.bh_alias_create.restype = C.c_int
        L.bh_alias_create.argtypes = [P, P, P, P, P, C.POINTER(C.c_void_p)]
        L.bh_monte_carlo.restype = C.c_int
        L.bh_monte_carlo.argtypes = [P, C.c_int64, C.c_double, C.c_int64, C.c_int64, C.c_uint64, P]
        L.bh_alias_destroy.restype = None
        L.bh_alias_destroy.argtypes = [P]
        L.bh_query_wait.restype = C.c_int
        L.bh_query_wait.argtypes = [P]
        L.bh_stream_gate.restype = C.c_int
        L.bh_stream_gate.argtypes = [P, P]
        L.bh_csr_build.restype = C.c_int
        L.bh_csr_build.argtypes = [C.c_int64] * 3 + [P] * 11 + [C.c_int32]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == BH_OK:
        return
    msg = (lib().bh_last_error() or b"").decode("utf-8", "replace")
    if rc in (BH_EINVAL, BH_EUNFLUSHED, BH_EDUP):
        raise ValueError(msg)
    if rc == BH_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"bhpp CUDA engine error: {msg}")


def ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def csr_build(n_u: int, n_v: int, eu, ev, ew, device: int = 0) -> dict | None:
    """Both canonical CSR sides of an edge list, built on ``device``
    (bh_csr_build).  Returns None when a (u, v) pair repeats."""
    eu = np.ascontiguousarray(eu, dtype=np.int64)
    ev = np.ascontiguousarray(ev, dtype=np.int64)
    ew = np.ascontiguousarray(ew, dtype=np.float64)
    n_e = int(eu.size)
    out = {
        "u_indptr": np.empty(n_u + 1, np.int64), "u_indices": np.empty(n_e, np.int32),
        "u_weights": np.empty(n_e, np.float64), "v_indptr": np.empty(n_v + 1, np.int64),
        "v_indices": np.empty(n_e, np.int32), "v_weights": np.empty(n_e, np.float64),
        "ws_u": np.empty(n_u, np.float64), "ws_v": np.empty(n_v, np.float64),
    }
    rc = lib().bh_csr_build(n_u, n_v, n_e, ptr(eu), ptr(ev), ptr(ew), *[ptr(out[k]) for k in (
        "u_indptr", "u_indices", "u_weights", "v_indptr", "v_indices", "v_weights", "ws_u", "ws_v")], int(device))
    if rc == BH_EDUP:
        return None
    check(rc)
    return out


def kernel_launches() -> int:
    return int(lib().bh_kernel_launches())


class DeviceGraph:
    """Owning handle of a device graph store (bh_graph)."""

    def __init__(self, g, dtype: str = "fp64", device: int = 0):
        self.dtype = dtype
        self.device = int(device)
        self.n_u, self.n_v, self.n_e = int(g.u_count), int(g.v_count), int(g.edge_count)
        arrs = [
            np.ascontiguousarray(g.u_indptr, dtype=np.int64),
            np.ascontiguousarray(g.u_indices, dtype=np.int32),
            np.ascontiguousarray(g.u_weights, dtype=np.float64),
            np.ascontiguousarray(g.v_indptr, dtype=np.int64),
            np.ascontiguousarray(g.v_indices, dtype=np.int32),
            np.ascontiguousarray(g.v_weights, dtype=np.float64),
            np.ascontiguousarray(g.ws_u, dtype=np.float64),
            np.ascontiguousarray(g.ws_v, dtype=np.float64),
        ]
        h = C.c_void_p()
        check(lib().bh_graph_create(self.n_u, self.n_v, self.n_e, *[ptr(a) for a in arrs], self.device,
                                    DTYPES[dtype], C.byref(h)))
        self.h = h
        self._fin = weakref.finalize(self, lib().bh_graph_destroy, h)

    def info(self) -> dict:
        gi = GraphInfo()
        check(lib().bh_graph_get_info(self.h, C.byref(gi)))
        return {f: getattr(gi, f) for f, _ in GraphInfo._fields_}

    def close(self):
        self._fin()

    def last_run_stats(self) -> dict:
        st = RunStats()
        check(lib().bh_last_run_stats(self.h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in RunStats._fields_}


def set_profiling(on: bool) -> None:
    check(lib().bh_set_profiling(1 if on else 0))


_applied_limit = None


def apply_scatter_limit() -> None:
    """Hand ``push_engine._SCATTER_LIMIT`` (the reference's module constant,
    push_engine.py:44, which its tests monkeypatch) to the engine before a run:
    rounds whose pushed rows touch at most that fraction of |E| run in frontier
    form (include/bhpp.h bh_set_scatter_limit)."""
    global _applied_limit
    from . import push_engine

    lim = float(push_engine._SCATTER_LIMIT)
    if lim != _applied_limit:
        check(lib().bh_set_scatter_limit(lim))
        _applied_limit = lim


_graph_cache: dict = {}
_graph_lock = threading.Lock()


def current_device() -> int:
    """CUDA device for calls that do not name one: torch's current device when
    torch is loaded (one process per GPU calls torch.cuda.set_device), else 0."""
    t = sys.modules.get("torch")
    if t is not None:
        try:
            if t.cuda.is_available():
                return int(t.cuda.current_device())
        except Exception:  # noqa: BLE001 -- no usable torch CUDA context: default device
            pass
    return 0


def device_graph(g, dtype: str = "fp64", device: int | None = None) -> DeviceGraph:
    """The device store for graph object ``g`` (either package's BipartiteGraph),
    built once per (graph, dtype, device) and freed with the graph.  ``device``
    defaults to the current CUDA device (see current_device)."""
    if device is None:
        device = current_device()
    if dtype not in DTYPES:
        raise ValueError(f"dtype must be one of {sorted(set(DTYPES))}")
    key = (id(g), DTYPES[dtype], int(device))
    with _graph_lock:
        ent = _graph_cache.get(key)
        if ent is not None and ent[0]() is g:
            return ent[1]
        dg = DeviceGraph(g, dtype, device)
        try:
            ref = weakref.ref(g, lambda _r, k=key: _graph_cache.pop(k, None))
        except TypeError:  # not weak-referenceable: cache for the process lifetime
            ref = (lambda obj=g: obj)
        _graph_cache[key] = (ref, dg)
        return dg


def trace_dicts(tr) -> tuple[dict, dict, dict]:
    """(backward, forward, engine-extra) dicts in the reference's key layout
    (push_engine.py:185-191,251-258; bhpp_query.py:198-201)."""
    back = {
        "selective_rounds": int(tr["sel_b"]),
        "sequential_rounds": int(tr["seq_b"]),
        "power_iterations": 0,
        "n_p": int(tr["n_p_b"]),
        "terminated_by": TERMINATIONS[int(tr["term_b"])],
    }
    fwd = {
        "selective_rounds": int(tr["sel_f"]),
        "sequential_rounds": 0,
        "power_iterations": int(tr["pi_iters"]),
        "n_p": int(tr["n_p_f"]),
        "gamma": float(tr["gamma"]),
        "terminated_by": TERMINATIONS[int(tr["term_f"])],
    }
    extra = {"tie_checks": int(tr["tie_checks"]), "tie_broke": int(tr["tie_broke"]),
             "near_ties": int(tr["near_ties"]), "min_budget_margin": float(tr["min_margin"])}
    return back, fwd, extra
