"""ctypes wrapper of the C oracle (oracle/bhpp_oracle.c).

TEST INFRASTRUCTURE ONLY: the parity checker and the CPU baseline.  Only
tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module; the product package
``paper_2312_06724_b200`` never does.

Every function restates the reference ``bipush`` function of the same name
(pkg/src/bipush/push_engine.py, bhpp_query.py) and returns the same shapes:
traces are dicts with the reference's keys plus the oracle-only tie fields
``tie_checks`` / ``tie_break_at`` used by the tie-aware parity protocol.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libbhpp_oracle.so"

TERMINATIONS = ("threshold-met", "budget-switch", "mass-drained")
PHASES = ("selective", "sequential", "forward-selective")
SCATTER_LIMIT = 0.25  # push_engine.py:44


class _Trace(C.Structure):
    _fields_ = [
        ("selective_rounds", C.c_int64),
        ("sequential_rounds", C.c_int64),
        ("power_iterations", C.c_int64),
        ("n_p", C.c_int64),
        ("terminated_by", C.c_int32),
        ("tie_checks", C.c_int32),
        ("tie_break_at", C.c_int32),
        ("_pad", C.c_int32),
        ("gamma", C.c_double),
    ]

    def as_dict(self, forward: bool) -> dict:
        d = {
            "selective_rounds": int(self.selective_rounds),
            "sequential_rounds": int(self.sequential_rounds),
            "power_iterations": int(self.power_iterations),
            "n_p": int(self.n_p),
        }
        if forward:
            d["gamma"] = float(self.gamma)
            d["tie_checks"] = int(self.tie_checks)
            d["tie_break_at"] = int(self.tie_break_at)
        d["terminated_by"] = TERMINATIONS[self.terminated_by]
        return d


HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double),
                   C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = C.CDLL(str(_LIB_PATH))
        P = C.c_void_p
        L.og_graph_create.restype = P
        L.og_graph_create.argtypes = [C.c_int64] * 3 + [P] * 8
        L.og_graph_destroy.argtypes = [P]
        L.og_numpy_sum.restype = C.c_double
        L.og_numpy_sum.argtypes = [P, C.c_int64]
        L.og_required_iterations.restype = C.c_int64
        L.og_required_iterations.argtypes = [C.c_double] * 3
        L.og_power_iteration.restype = C.c_int
        L.og_power_iteration.argtypes = [P, P, C.c_double, C.c_int64, P]
        L.og_ss_push.restype = C.c_int
        L.og_ss_push.argtypes = [P, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_double,
                                 P, P, P, P, P, HOOK, P]
        L.og_pi_push.restype = C.c_int
        L.og_pi_push.argtypes = [P, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double,
                                 P, P, P, P, P, P, HOOK, P]
        L.og_bhpp_query.restype = C.c_int
        L.og_bhpp_query.argtypes = [P, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double,
                                    C.c_double, P, P, P, HOOK, P]
        L.og_topk.restype = C.c_int64
        L.og_topk.argtypes = [P, C.c_int64, C.c_int64, C.c_int64, P]
        L.og_estimate_lambda.restype = C.c_double
        L.og_estimate_lambda.argtypes = [P, C.c_double, C.c_int64]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def numpy_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().og_numpy_sum(_ptr(a), a.size))


def required_iterations(alpha: float, epsilon_f: float, mass: float) -> int:
    r = lib().og_required_iterations(alpha, epsilon_f, mass)
    if r < 0:
        raise ValueError("bad alpha / epsilon_f")
    return int(r)


class OracleGraph:
    """The C oracle's private copy of a graph's CSR arrays (duck-typed input:
    either package's BipartiteGraph)."""

    def __init__(self, g):
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
        self.ws_u = arrs[6]
        self.h = lib().og_graph_create(self.n_u, self.n_v, self.n_e, *[_ptr(a) for a in arrs])
        if not self.h:
            raise MemoryError("oracle graph allocation failed")

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.og_graph_destroy(h)
            self.h = None

    # -- helpers --------------------------------------------------------------
    def _hook(self, round_hook):
        if round_hook is None:
            return HOOK(), None
        n_u, n_v = self.n_u, self.n_v

        def cb(_user, phase, rounds, r_u, r_v, est, n_p):
            led = {
                "residue_u": np.ctypeslib.as_array(r_u, shape=(n_u,)).copy(),
                "residue_v": np.ctypeslib.as_array(r_v, shape=(n_v,)).copy(),
                "estimate": np.ctypeslib.as_array(est, shape=(n_u,)).copy(),
                "n_p": int(n_p),
            }
            round_hook(PHASES[phase], int(rounds), led)

        h = HOOK(cb)
        return h, h

    # -- reference functions ----------------------------------------------------
    def power_iteration(self, start, alpha: float, t: int) -> np.ndarray:
        start = np.ascontiguousarray(start, dtype=np.float64)
        out = np.empty(self.n_u)
        rc = lib().og_power_iteration(self.h, _ptr(start), alpha, int(t), _ptr(out))
        if rc:
            raise ValueError("bad power_iteration arguments")
        return out

    def ss_push(self, target: int, alpha: float, epsilon_b: float, budget: bool = True,
                scatter_limit: float = SCATTER_LIMIT, round_hook=None):
        r_u, r_v, est = np.empty(self.n_u), np.empty(self.n_v), np.empty(self.n_u)
        n_p = np.zeros(1, dtype=np.int64)
        tr = _Trace()
        hook, _keep = self._hook(round_hook)
        rc = lib().og_ss_push(self.h, int(target), alpha, epsilon_b, int(budget), scatter_limit,
                              _ptr(r_u), _ptr(r_v), _ptr(est), _ptr(n_p), C.byref(tr), hook, None)
        if rc:
            raise ValueError("bad ss_push arguments")
        return {"residue_u": r_u, "residue_v": r_v, "estimate": est, "n_p": int(n_p[0])}, tr.as_dict(False)

    def pi_push(self, source: int, alpha: float, lam: float, epsilon_f: float, ledger: dict,
                scatter_limit: float = SCATTER_LIMIT, round_hook=None):
        """Mutates ``ledger`` (dict of residue_u/residue_v/estimate/n_p) like the reference."""
        r_u = np.ascontiguousarray(ledger["residue_u"], dtype=np.float64).copy()
        r_v = np.ascontiguousarray(ledger["residue_v"], dtype=np.float64).copy()
        est = np.ascontiguousarray(ledger["estimate"], dtype=np.float64).copy()
        n_p = np.array([ledger["n_p"]], dtype=np.int64)
        scores = np.empty(self.n_u)
        tr = _Trace()
        hook, _keep = self._hook(round_hook)
        rc = lib().og_pi_push(self.h, int(source), alpha, lam, epsilon_f, scatter_limit, _ptr(r_u),
                              _ptr(r_v), _ptr(est), _ptr(n_p), _ptr(scores), C.byref(tr), hook, None)
        if rc == 17:
            raise ValueError("unflushed ledger: V-side residues must be zero at the forward handoff")
        if rc:
            raise ValueError("bad pi_push arguments")
        ledger.update(residue_u=r_u, residue_v=r_v, estimate=est, n_p=int(n_p[0]))
        return scores, tr.as_dict(True)

    def bhpp_query(self, q: int, alpha: float, lam: float, eps_b: float, eps_f: float,
                   scatter_limit: float = SCATTER_LIMIT, round_hook=None):
        """Returns (scores, {"backward": trace, "forward": trace})."""
        scores = np.empty(self.n_u)
        tb, tf = _Trace(), _Trace()
        hook, _keep = self._hook(round_hook)
        rc = lib().og_bhpp_query(self.h, int(q), alpha, lam, eps_b, eps_f, scatter_limit, _ptr(scores),
                                 C.byref(tb), C.byref(tf), hook, None)
        if rc:
            raise ValueError("bad bhpp_query arguments")
        return scores, {"backward": tb.as_dict(False), "forward": tf.as_dict(True)}

    def bhpp_query_many(self, sources, alpha, lam, eps_b, eps_f, threads: int | None = None,
                        scatter_limit: float = SCATTER_LIMIT):
        """The reference's thread-pool pattern (cli.py:444-450); ctypes drops the GIL."""
        threads = threads or os.cpu_count() or 1
        srcs = [int(s) for s in sources]
        if threads <= 1:
            return [self.bhpp_query(s, alpha, lam, eps_b, eps_f, scatter_limit) for s in srcs]
        with ThreadPoolExecutor(max_workers=threads) as ex:
            return list(ex.map(lambda s: self.bhpp_query(s, alpha, lam, eps_b, eps_f, scatter_limit), srcs))

    def estimate_lambda(self, alpha: float, tau: int) -> float:
        return float(lib().og_estimate_lambda(self.h, alpha, int(tau)))


def topk_indices(scores, k: int, exclude: int | None = None) -> np.ndarray:
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    out = np.empty(max(1, k), dtype=np.int64)
    m = lib().og_topk(_ptr(scores), scores.size, int(k), -1 if exclude is None else int(exclude), _ptr(out))
    return out[:m].copy()


def choose_eps_b(epsilon: float, mu: float) -> float:
    """bhpp_query.py:92-104."""
    raw = epsilon * (1.0 - mu) / (2.0 - mu)
    return min(max(raw, epsilon / 10.0), epsilon / 2.0)


def estimate_mu(u_count: int, v_count: int, edge_count: int) -> float:
    """bhpp_query.py:86-89."""
    raw = math.sqrt(u_count * v_count) / edge_count
    return float(min(1.0, max(1e-3, raw)))


def default_tau(u_count: int, alpha: float) -> int:
    """bhpp_query.py:65-67."""
    return required_iterations(alpha, 0.05, float(u_count))


def index_meta(g, alpha: float = 0.15, tau: int | None = None) -> dict:
    """build_index_meta arithmetic (bhpp_query.py:107-123) without the fingerprint."""
    og = g if isinstance(g, OracleGraph) else OracleGraph(g)
    if tau is None:
        tau = default_tau(og.n_u, alpha)
    return {
        "alpha": alpha,
        "tau": int(tau),
        "lam": og.estimate_lambda(alpha, tau),
        "mu": estimate_mu(og.n_u, og.n_v, og.n_e),
    }


def tie_skip_for(forward_trace: dict) -> int:
    """Engine knob reproducing the oracle's tie decisions (SURVEY.md section 7,
    hard part 1): continue through this many exact-tie budget checks."""
    if forward_trace["tie_break_at"]:
        return forward_trace["tie_break_at"] - 1
    return forward_trace["tie_checks"]
