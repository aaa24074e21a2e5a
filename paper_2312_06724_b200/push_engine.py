"""Residue-push kernels, device-backed drop-ins for ``bipush.push_engine``.

Same names, signatures, return types, trace keys and errors as the reference
(pkg/src/bipush/push_engine.py); the rounds run on the GPU through
``bh_push_run`` / ``bh_power_iteration`` (include/bhpp.h).  A round here is
the reference's batch-synchronous ``_round`` (push_engine.py:280-324): push
every U node over threshold, then flush every positive V residue; the device
executes it as two pull SpMVs over the pre-scaled CSR sides.

``round_hook(phase, rounds, ledger)`` is honoured by stepping the device one
round at a time and handing the hook a host copy of the ledger after every
round (the reference hands its live ledger; tests only read it).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _capi

# Frontier ("scatter") rounds when the pushed rows touch at most this fraction of
# |E| (the reference's constant of the same name, push_engine.py:44, is 0.25 --
# tuned for numpy scatter against scipy matvec on a CPU; on the GPU a frontier
# round pays below a few % of |E|: single c3 queries 729 ms dense, 731 at 0.25,
# 673 at 0.05, 646 at 0.01, profiles/r02_latency.md).  The engine reads it at
# every run (_capi.apply_scatter_limit).  Results do not depend on it; tests
# monkeypatch it like the reference's own (pkg/tests/test_push_engine.py:188-202):
# -1 forces dense rounds, >= 1 frontier rounds.
_SCATTER_LIMIT = 0.01


@dataclass
class ResidueLedger:
    """Push state: residues on both sides, settled estimates on U, and the
    monotone operation counter n_p (push_engine.py:47-72)."""

    residue_u: np.ndarray
    residue_v: np.ndarray
    estimate: np.ndarray
    n_p: int = 0

    @classmethod
    def initial(cls, g, target_u: int) -> "ResidueLedger":
        if not 0 <= target_u < g.u_count:
            raise ValueError(f"node index {target_u} out of range")
        r_u = np.zeros(g.u_count)
        r_u[target_u] = 1.0
        return cls(r_u, np.zeros(g.v_count), np.zeros(g.u_count), 0)

    def active_u(self, threshold) -> np.ndarray:
        return np.flatnonzero(self.residue_u > threshold)

    def active_v(self) -> np.ndarray:
        return np.flatnonzero(self.residue_v > 0.0)


@dataclass
class PushOutcome:
    """Result of one kernel run. ``scores`` is set by forward kernels only."""

    ledger: ResidueLedger
    phase_trace: dict
    terminated_by: str
    scores: np.ndarray | None = None


def _check_alpha(alpha):
    if not 0.0 < alpha < 1.0:
        raise ValueError("alpha must lie strictly between 0 and 1")


def required_iterations(alpha: float, epsilon_f: float, mass: float) -> int:
    """Power-iteration depth t with truncation deficit at most epsilon_f:
    t = max(0, ceil(log_{1/(1-alpha)}(mass / epsilon_f)) - 1)  (push_engine.py:85-98).
    Scalar control arithmetic; the device evaluates the same formula in K4."""
    _check_alpha(alpha)
    if epsilon_f <= 0:
        raise ValueError("epsilon_f must be positive")
    if mass <= 0:
        return 0
    return max(0, math.ceil(math.log(mass / epsilon_f) / math.log(1.0 / (1.0 - alpha))) - 1)


def _dtype_of(dtype):
    return dtype or "fp64"


def power_iteration(g, start, alpha: float, t: int, dtype: str | None = None) -> np.ndarray:
    """alpha * sum_{l<=t} (1-alpha)^l start P^l  (push_engine.py:101-117).

    ``start`` may be one vector [|U|] or a batch [n, |U|]; a batch runs as one
    query block on the device."""
    _check_alpha(alpha)
    if t < 0:
        raise ValueError("iteration count must be nonnegative")
    base = np.asarray(start, dtype=np.float64)
    single = base.ndim == 1
    base2 = np.ascontiguousarray(base.reshape(1, -1) if single else base)
    if base2.shape[1] != g.u_count:
        raise ValueError("start vector length must match the U side")
    dg = _capi.device_graph(g, _dtype_of(dtype))
    out = np.empty_like(base2)
    _capi.check(_capi.lib().bh_power_iteration(dg.h, _capi.ptr(base2), base2.shape[0], float(alpha), int(t),
                                               _capi.ptr(out)))
    return out[0] if single else out


def _hook_adapter(g, round_hook):
    if round_hook is None:
        return _capi.HOOK()
    n_u, n_v = g.u_count, g.v_count

    def cb(_user, phase, rounds, r_u, est, n_p):
        led = ResidueLedger(
            np.ctypeslib.as_array(r_u, shape=(n_u,)).copy(),
            np.zeros(n_v),
            np.ctypeslib.as_array(est, shape=(n_u,)).copy(),
            int(n_p),
        )
        round_hook(_capi.PHASES[phase], int(rounds), led)

    return _capi.HOOK(cb)


def run_job(g, job: int, source: int, alpha: float, lam: float, eps_b: float, eps_f: float,
            ledger: ResidueLedger | None = None, round_hook=None, tie_skip: int = 0, dtype: str | None = None):
    """One device ledger job (bh_push_run).  Returns (ledger, scores, trace)."""
    dg = _capi.device_graph(g, _dtype_of(dtype))
    n_u = g.u_count
    if ledger is None:
        r_u, est, n_p = np.zeros(n_u), np.zeros(n_u), np.zeros(1, dtype=np.int64)
    else:
        r_u = np.ascontiguousarray(ledger.residue_u, dtype=np.float64).copy()
        est = np.ascontiguousarray(ledger.estimate, dtype=np.float64).copy()
        n_p = np.array([int(ledger.n_p)], dtype=np.int64)
    scores = np.empty(n_u)
    tr = _capi.Trace()
    hook = _hook_adapter(g, round_hook)
    _capi.apply_scatter_limit()
    _capi.check(_capi.lib().bh_push_run(dg.h, job, int(source), float(alpha), float(lam), float(eps_b),
                                        float(eps_f), int(tie_skip), _capi.ptr(r_u), _capi.ptr(est),
                                        _capi.ptr(n_p), _capi.ptr(scores), C.byref(tr), hook, None))
    trace = np.frombuffer(bytearray(tr), dtype=_capi.TRACE_DTYPE)[0]
    return (r_u, est, int(n_p[0])), scores, trace


def selective_push(g, target_u: int, alpha: float, epsilon_b: float, round_hook=None) -> PushOutcome:
    """Backward pushing until every U residue is at most epsilon_b
    (push_engine.py:120-142)."""
    _check_alpha(alpha)
    if epsilon_b <= 0:
        raise ValueError("epsilon_b must be positive")
    if not 0 <= target_u < g.u_count:
        raise ValueError(f"node index {target_u} out of range")
    (r_u, est, n_p), _, tr = run_job(g, _capi.JOB_SELECTIVE, target_u, alpha, 1.0, epsilon_b, 1.0,
                                     round_hook=round_hook)
    led = ResidueLedger(r_u, np.zeros(g.v_count), est, n_p)
    back, _, _ = _capi.trace_dicts(tr)
    trace = {k: back[k] for k in ("selective_rounds", "sequential_rounds", "power_iterations", "n_p")}
    return PushOutcome(led, trace, "threshold-met")


def ss_push(g, target_u: int, alpha: float, epsilon_b: float, round_hook=None) -> PushOutcome:
    """Budgeted backward pushing: selective rounds, then sequential fallback
    (push_engine.py:145-191, Alg. 3 of the paper)."""
    _check_alpha(alpha)
    if epsilon_b <= 0:
        raise ValueError("epsilon_b must be positive")
    if not 0 <= target_u < g.u_count:
        raise ValueError(f"node index {target_u} out of range")
    (r_u, est, n_p), _, tr = run_job(g, _capi.JOB_SS_PUSH, target_u, alpha, 1.0, epsilon_b, 1.0,
                                     round_hook=round_hook)
    led = ResidueLedger(r_u, np.zeros(g.v_count), est, n_p)
    back, _, _ = _capi.trace_dicts(tr)
    term = back.pop("terminated_by")
    return PushOutcome(led, back, term)


def pi_push(g, source_u: int, alpha: float, lam: float, epsilon_f: float, seed_ledger: ResidueLedger,
            round_hook=None, tie_skip: int = 0) -> PushOutcome:
    """Forward scores for source_u from a flushed backward ledger
    (push_engine.py:194-258, Alg. 4).  Mutates ``seed_ledger`` like the
    reference.  ``tie_skip`` replays reference runs that continued through
    exact budget ties; 0 = exact-arithmetic outcome."""
    _check_alpha(alpha)
    if epsilon_f <= 0:
        raise ValueError("epsilon_f must be positive")
    if lam <= 0:
        raise ValueError("lam must be positive")
    if not 0 <= source_u < g.u_count:
        raise ValueError(f"node index {source_u} out of range")
    led = seed_ledger
    if (np.asarray(led.residue_v) != 0.0).any():
        raise ValueError("unflushed ledger: V-side residues must be zero at the forward handoff")
    (r_u, est, n_p), scores, tr = run_job(g, _capi.JOB_PI_PUSH, source_u, alpha, lam, 1.0, epsilon_f,
                                          ledger=led, round_hook=round_hook, tie_skip=tie_skip)
    led.residue_u[...] = r_u
    led.estimate[...] = est
    led.n_p = n_p
    _, fwd, extra = _capi.trace_dicts(tr)
    term = fwd.pop("terminated_by")
    out = PushOutcome(led, fwd, term, scores=scores)
    out.engine = extra
    return out
