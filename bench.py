#!/usr/bin/env python
"""bench.py -- BHPP source queries/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling weak|strong] [--config c2] [--no-c3] [--no-fp64] [--no-cpu]

``--gpus N`` with N > 1 and no torchrun environment re-launches itself under
``torch.distributed.run`` (one rank per GPU, NCCL, 127.0.0.1); under torchrun
the ranks come from RANK / WORLD_SIZE / LOCAL_RANK.

Workload (N=1): BASELINE.json configs[1] ("c2"): seeded Chung-Lu bipartite
graph |U|=1e5, |V|=2e5, |E|=2e6, exponent 2.2, integer weights U{1..10},
alpha=0.15, eps=1e-7, 64 sources drawn like the reference's bench
(cli.py:415-417), top-50 per query.  A step = one SS-BI-PUSH pass (backward
push, forward push, power iteration, combine, top-k) over the batch.
Scaling (N>1): "weak" (default): every rank runs its own 64 sources on a
replica of the graph; "strong": one fixed batch (--batch, default the
config's source count) sharded interleaved over the ranks.  Either way each
rank's finalize kernel writes its top-k and traces into its region of one
packed buffer and ONE NCCL all-gather per step returns the full result, in
source order, to every rank (distributed.py).

value   : queries/s, inputs resident in HBM, device-timed (CUDA events on the
          engine stream, L2 flushed with a 256 MiB write between steps,
          outside the timed interval), max over ranks.
e2e     : same metric through the public host API (bhpp_query_batch; N>1
          bhpp_query_sharded): numpy sources in, numpy top-k/traces out, H2D
          and D2H inside the timing.  fp32 headline; fp64 beside it.
roofline: the dominant kernel (K2 V pull): SURVEY.md 8(d) algorithmic bytes
          per launch / its CUDA-event time in a replay of the timed steps;
          traffic from the committed ncu capture.
hbm_regime: the same measurement at config c3 (|E|=1e8, operands far larger
          than L2), N=1 only (--no-c3 skips it).
latency_c1: config c1 (configs[0]) single-query latency through the public
          API (the cluster small path) beside the C port on one host core.
cpu_baseline / --impl reference: the bit-exact C port of the reference
          (oracle/) on all host cores, the reference's thread-pool pattern.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "BHPP source queries/sec at fixed alpha,eps (achieved HBM GB/s vs B200 peak in roofline)"
UNIT = "queries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--batch", type=int, default=0, help="strong scaling: total sources (default: the config's)")
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 side measurement")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-c3", action="store_true", help="skip the config-c3 (HBM regime) leg")
    ap.add_argument("--c3-sources", type=int, default=1024)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def relaunch_under_torchrun(args) -> int:
    """bench.py --gpus N outside torchrun: start N ranks (one per GPU) and pass
    their output through; rank 0 prints the JSON line."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def workload(cfg_name: str, rank: int, world: int, scaling: str, batch: int):
    """(cfg, graph, this rank's sources, total sources in the job)."""
    from paper_2312_06724_b200.rng import substream
    from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

    cfg = CONFIGS[cfg_name]
    dev = 0 if not os.environ.get("BH_BENCH_HOST_GEN") else None
    try:
        import torch

        dev = torch.cuda.current_device() if dev is not None and torch.cuda.is_available() else None
    except Exception:  # noqa: BLE001 -- no torch CUDA: host generator
        dev = None
    g = make_graph(cfg, device=dev)
    n = cfg.n_sources or cfg.u_count
    if scaling == "strong":
        total = batch or n
        src = bench_sources(cfg.u_count, total)
        return cfg, g, src, total  # every rank holds the whole batch; the shard is taken per step
    if rank == 0:
        src = bench_sources(cfg.u_count, n)
    else:
        src = substream(0, "bench-queries", rank).choice(cfg.u_count, n, replace=False).astype(np.int64)
    return cfg, g, src, n * world


def config_json(cfg, n_local, world, slots, k, scaling, total):
    return {
        "workload": f"{cfg.name}: |U|={cfg.u_count}, |V|={cfg.v_count}, |E|={cfg.edge_count} Chung-Lu "
                    f"beta_u={cfg.beta_u} beta_v={cfg.beta_v} weights={cfg.weights}, alpha={cfg.alpha}, "
                    f"eps={cfg.epsilons[0]}, top-{k}, "
                    + (f"{n_local} sources/GPU" if scaling == "weak" else f"{total} sources sharded over {world} GPU(s)"),
        "queries_per_gpu": int(n_local),
        "global_batch": int(total),
        "top_k": int(k),
        "slots": int(slots),
        "parallelism": f"query-shard x{world} (graph replicated; one packed NCCL all-gather per step)",
        "l2": "256 MiB write between timed steps (outside the timed interval)",
    }


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line).

    The sampler is started and allowed to produce its first row before the
    timed steps begin (``start()`` returns once it is live); only rows whose
    timestamp falls inside [start(), stop()] are summarised."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.t0 = self.t1 = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
            return
        deadline = time.time() + 10.0
        while time.time() < deadline and not Path(self.f.name).read_text().strip():
            time.sleep(0.02)

    def start(self):
        import datetime
        self.t0 = datetime.datetime.now()

    def stop(self) -> dict:
        import datetime
        self.t1 = datetime.datetime.now()
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)  # let the sampler flush the row covering the end of the region
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [[c.strip() for c in r.split(",")] for r in Path(self.f.name).read_text().strip().splitlines()
                if r.strip()]
        os.unlink(self.f.name)

        def ts(r):
            try:
                return datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f")
            except (ValueError, IndexError):
                return None

        inside = [r for r in rows if len(r) >= 10 and ts(r) is not None and self.t0 <= ts(r) <= self.t1]
        num = lambda x: x.replace(".", "", 1).isdigit()  # noqa: E731
        sm = [float(r[2]) for r in inside if num(r[2])]
        mx = [float(r[3]) for r in rows if len(r) >= 10 and num(r[3])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in inside for j in range(4) if r[6 + j] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "sm_min_mhz": min(sm) if sm else None, "reasons": reasons, "samples": len(inside),
                "region_s": (self.t1 - self.t0).total_seconds()}


def _ncu_capture(name: str):
    """Latest committed ncu summary profiles/rNN_<name>.json (kernels dict), or (None, None)."""
    for p in sorted((REPO / "profiles").glob(f"r*_{name}.json"), reverse=True):
        try:
            return json.loads(p.read_text())["kernels"], p.name
        except Exception:  # noqa: BLE001
            continue
    return None, None


def ncu_traffic(name: str):
    """(V-pull DRAM bytes per launch, round K1+K2+K3+K1a DRAM bytes, source file) from
    the committed ncu --set full capture, or Nones."""
    ks, src = _ncu_capture(name)
    if not ks:
        return None, None, None
    vp = rnd = None
    for k, v in ks.items():  # k_pull*<B, T, SIDE, ...>: SIDE 0 is the V pull
        b = 1e6 * (v.get("dram_read_MB", 0) + v.get("dram_write_MB", 0))
        if k.startswith(("k_push", "k_pull", "k_combine")):
            rnd = (rnd or 0) + b
        if k.startswith("k_pull") and k.split("<", 1)[1].split(",")[2].strip().rstrip(">") == "0":
            vp = b
    return vp, rnd, f"profiles/{src}"


def peak_hbm():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:  # noqa: BLE001
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def algorithmic_bytes(g, traces, rounds: int, s: int) -> float:
    """per round 2E(i+s) + (|U|+|V|+2) o; per query
    push round s (4|U| + 2|V|), per power iteration s (3|U| + 2|V|); i = o = 4."""
    i = o = 4
    E, U, V = g.edge_count, g.u_count, g.v_count
    push_rounds = int(traces["sel_b"].sum() + traces["seq_b"].sum() + traces["sel_f"].sum())
    pi = int(traces["pi_iters"].sum())
    return rounds * (2 * E * (i + s) + (U + V + 2) * o) + push_rounds * s * (4 * U + 2 * V) + pi * s * (3 * U + 2 * V)


def vpull_bytes(g, slots: int, s: int) -> int:
    """SURVEY.md 8(d), one SpMM half (the V pull): E(i+s) + (|V|+1) o + B s (|U| + |V|)."""
    return g.edge_count * (4 + s) + (g.v_count + 1) * 4 + slots * s * (g.u_count + g.v_count)


# -----------------------------------------------------------------------------
def cpu_leg(g, src, alpha, eps_b, eps_f, lam, seconds: float, threads: int | None = None):
    """The reference path (bit-exact C port, oracle/) on host cores: a bounded
    sample of the same sources, all threads, the cmd_bench thread-pool pattern."""
    from oracle import cpu_oracle as O

    og = O.OracleGraph(g)
    threads = threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    og.bhpp_query(int(src[0]), alpha, lam, eps_b, eps_f)
    t1 = time.perf_counter() - t0
    n = int(max(threads, min(len(src) * 4, round(seconds / max(t1, 1e-3) * threads))))
    sample = [int(src[j % len(src)]) for j in range(n)]
    t0 = time.perf_counter()
    og.bhpp_query_many(sample, alpha, lam, eps_b, eps_f, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n} queries of the bench sources (cycled), {threads} threads, fp64 C port of the "
                      f"reference (oracle/bhpp_oracle.c), {dt:.1f} s; 1-thread single query {t1 * 1e3:.0f} ms"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import cpu_oracle as O

    cfg, g, src, total = workload(args.config, 0, 1, "weak", 0)
    om = O.index_meta(g, cfg.alpha)
    eps = cfg.epsilons[0]
    eps_b = O.choose_eps_b(eps, om["mu"])
    eps_f = eps - eps_b
    og = O.OracleGraph(g)
    threads = os.cpu_count() or 1
    per_step = threads
    cursor = 0

    def step():
        nonlocal cursor
        sample = [int(src[(cursor + j) % len(src)]) for j in range(per_step)]
        cursor += per_step
        og.bhpp_query_many(sample, cfg.alpha, om["lam"], eps_b, eps_f, threads=threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    v = per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Chung-Lu, configs[1])",
        "config": config_json(cfg, len(src), 1, 0, cfg.k, "weak", len(src)),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{per_step} queries per step ({threads} threads) of the bench sources, "
                                   "bit-exact C port of the reference (oracle/), host wall clock"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference is pure Python (numpy/scipy); its path is timed through its bit-exact C port",
    }
    print(json.dumps(line), flush=True)


# -----------------------------------------------------------------------------
class Runner:
    """One rank's device-resident batch loop (timed steps, profiled replay)."""

    def __init__(self, g, meta, src, eps, k, dtype, slots, rank, world, scaling, total, dev, stream, flush_buf):
        import torch

        from paper_2312_06724_b200 import _capi
        from paper_2312_06724_b200.distributed import PackedShard, per_rank

        self.g, self.meta, self.k, self.dtype, self.slots = g, meta, k, dtype, slots
        self.rank, self.world, self.scaling, self.total = rank, world, scaling, total
        self.dev, self.stream, self.flush_buf = dev, stream, flush_buf
        self.eps_b = float(meta.eps_split_policy(eps))
        self.eps_f = eps - self.eps_b
        self.dg = _capi.device_graph(g, dtype, device=dev.index)
        mine = src[rank::world] if scaling == "strong" else src
        self.n = len(mine)
        self.src_t = torch.from_numpy(np.asarray(mine, dtype=np.int32)).to(dev)
        per = per_rank(total, world) if world > 1 else self.n
        self.packed = PackedShard(per, k, dev)
        self.out = torch.empty(world * self.packed.buf.numel(), dtype=torch.uint8, device=dev) if world > 1 else None
        self.gate = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.gated = not os.environ.get("BH_NO_GRAPH") and not os.environ.get("BH_BENCH_NO_GATE")

    def step(self, async_=False):
        import torch
        import torch.distributed as dist

        from paper_2312_06724_b200.bhpp_query import query_batch_device

        if self.n:
            query_batch_device(self.dg, self.meta, self.eps_b, self.eps_f, self.src_t.data_ptr(), self.n, self.k,
                               self.packed.idx.data_ptr(), self.packed.score.data_ptr(),
                               self.packed.trace.data_ptr(), slots=self.slots or None,
                               stream=self.stream.cuda_stream, async_=async_)
        if self.world > 1:  # the shards' top-k + traces: one packed all-gather on the same stream
            with torch.cuda.stream(self.stream):
                dist.all_gather_into_tensor(self.out, self.packed.buf)

    def run_steps(self, nsteps, profiled, use_gate=False):
        import torch

        from paper_2312_06724_b200 import _capi
        from paper_2312_06724_b200.bhpp_query import query_wait

        _capi.set_profiling(profiled)
        ms, per_step, traces = 0.0, [], []
        prof = {"ms_prep": 0.0, "ms_vpull": 0.0, "ms_upull": 0.0, "ms_control": 0.0, "rounds": 0, "slots": 0,
                "step_rounds": []}
        for _ in range(nsteps):
            with torch.cuda.stream(self.stream):
                self.flush_buf.fill_(1.0)  # evict L2 (256 MiB > 126 MB) outside the timed interval
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            if use_gate and self.gated and not profiled and self.n:
                # the whole step is enqueued behind a gate before the device
                # starts it: e0..e1 is device time only, no host submission gaps
                self.gate[0] = 0
                _capi.check(_capi.lib().bh_stream_gate(self.stream.cuda_stream, self.gate.data_ptr()))
                e0.record(self.stream)
                self.step(async_=True)
                e1.record(self.stream)
                self.gate[0] = 1
                query_wait(self.dg)
            else:
                e0.record(self.stream)
                self.step()
                e1.record(self.stream)
            e1.synchronize()
            ms += e0.elapsed_time(e1)
            per_step.append(e0.elapsed_time(e1))
            st = self.dg.last_run_stats()
            prof["step_rounds"].append(int(st["rounds"]))
            for key in ("ms_prep", "ms_vpull", "ms_upull", "ms_control", "rounds"):
                prof[key] += st[key]
            prof["slots"] = st["slots"]
            traces.append(self.packed.trace[: self.n].cpu().numpy().copy().view(_capi.TRACE_DTYPE).reshape(-1))
        _capi.set_profiling(False)
        prof["step_ms"] = per_step
        return ms, prof, traces

    def measure(self, steps, warmup, clocks_index=None):
        """Timed steps (max over ranks), launches, clocks; then a profiled replay."""
        import torch
        import torch.distributed as dist

        from paper_2312_06724_b200 import _capi

        self.run_steps(max(1, warmup - 1), False)  # graph instantiation, first NCCL use
        if warmup > 1:
            self.run_steps(1, False, use_gate=True)
        torch.cuda.synchronize(self.dev)
        if self.world > 1:
            dist.barrier()
        clocks = Clocks(clocks_index) if clocks_index is not None and not os.environ.get("BH_BENCH_NO_CLOCKS") else None
        if clocks:
            clocks.start()
        launches0 = _capi.kernel_launches()
        ms, tprof, _ = self.run_steps(steps, False, use_gate=True)
        launches = _capi.kernel_launches() - launches0
        clk = clocks.stop() if clocks else {"sm_mhz": None, "reasons": ["not sampled"]}
        torch.cuda.synchronize(self.dev)
        if self.world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=self.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        pms, prof, ptraces = self.run_steps(steps, True)
        prof["timed_step_ms"] = tprof["step_ms"]
        prof["timed_step_rounds"] = tprof["step_rounds"]
        return ms, launches, prof, clk, ptraces, pms


def e2e_leg(g, meta, src, eps, k, dtype, slots, rank, world, scaling, dev, stream, flush_buf, steps):
    """The public host API per step (numpy in, numpy out): bhpp_query_batch at
    N=1 / weak scaling, bhpp_query_sharded (device-resident shard + packed
    all-gather, numpy in and out) for strong scaling.  Max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2312_06724_b200 as bh
    from paper_2312_06724_b200.distributed import bhpp_query_sharded, gather_results

    def one():
        if scaling == "strong" and world > 1:
            return bhpp_query_sharded(g, meta, src, eps, k=k, dtype=dtype, slots=slots or None, device=dev)
        res = bh.bhpp_query_batch(g, meta, src, eps, k=k, dtype=dtype, slots=slots or None,
                                  stream=stream.cuda_stream)
        if world > 1:
            gather_results(res.topk_index, res.topk_score, res.traces, world * len(src), rank, world, device=dev)
        return res

    for _ in range(2):
        one()
    tot, per = 0.0, []
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
        per.append(round(e0.elapsed_time(e1), 3))
    if world > 1:
        t = torch.tensor([tot], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    return tot, per


def roofline_block(g, prof, pms, steps, s_bytes, alg, peak, peak_src, traffic_name):
    B = prof.get("slots", 0)
    rounds = max(1, prof["rounds"])
    v_bytes = vpull_bytes(g, B, s_bytes)
    v_us = prof["ms_vpull"] * 1e3 / rounds
    v_ach = v_bytes / (v_us / 1e6) / 1e9 if v_us > 0 else None
    kern_ms = prof["ms_prep"] + prof["ms_vpull"] + prof["ms_upull"]
    ach = alg / (kern_ms / 1e3) / 1e9 if kern_ms > 0 else None
    vp_t, rnd_t, t_src = ncu_traffic(traffic_name)
    return {
        "bound": "hbm", "achieved": v_ach, "peak": peak, "unit": "GB/s",
        "frac": v_ach / peak if v_ach else None, "traffic": vp_t,
        "kernel": "K2 V pull (k_pull_rf / k_pull_small, SIDE_V), the dominant kernel",
        "algorithmic_bytes_per_launch": v_bytes,
        "algorithmic_model": "E(i+s) + (|V|+1) o + B s (|U| + |V|), i = o = 4 (SURVEY 8(d), one SpMM half)",
        "launch_us": v_us, "launches": int(prof["rounds"]),
        "share_of_step": prof["ms_vpull"] / pms if pms else None,
        "traffic_source": t_src,
        "round": {
            "unit": "push/PI round = K1 push + K2 V-pull + K3 U-pull + K1a combine (SURVEY 8(d) unit)",
            "achieved_gbs": ach, "frac": ach / peak if ach else None,
            "algorithmic_bytes_per_round": alg / rounds, "traffic_per_round": rnd_t,
            "share_of_step": kern_ms / pms if pms else None,
        },
        "gather": {"bytes_per_round": 2 * g.edge_count * B * s_bytes,
                   "achieved_tbs": (2 * g.edge_count * B * s_bytes * prof["rounds"]
                                    / ((prof["ms_vpull"] + prof["ms_upull"]) / 1e3) / 1e12)
                   if prof["ms_vpull"] + prof["ms_upull"] > 0 else None,
                   "note": "operand-row gathers of the two pulls (E x B x s each)"},
        "algorithmic_bytes_per_step": alg / steps, "kernel_ms_per_step": kern_ms / steps,
        "rounds_per_step": prof["rounds"] / steps,
        "timing": "per-kernel CUDA events on the engine stream, in a replay of the timed steps "
                  "(the headline value is timed without per-kernel events; each timed step is "
                  "enqueued behind a device start gate, so e0..e1 is device time only)",
        "breakdown_ms_per_step": {k2: prof[k2] / steps for k2 in ("ms_prep", "ms_vpull", "ms_upull", "ms_control")},
        "peak_source": peak_src,
        "timed_step_ms": [round(x, 3) for x in prof.get("timed_step_ms", [])],
        "profiled_step_ms": [round(x, 3) for x in prof.get("step_ms", [])],
        "timed_step_rounds": prof.get("timed_step_rounds"),
    }


def c3_leg(n_sources, dev, stream, flush_buf, peak, peak_src):
    """Config c3 (HBM regime): one timed batch of the config's bench sources
    (device-resident), a profiled replay on a quarter of them for the roofline."""
    import torch

    import paper_2312_06724_b200 as bh
    from paper_2312_06724_b200 import _capi
    from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

    cfg = CONFIGS["c3"]
    t0 = time.perf_counter()
    g = make_graph(cfg, device=dev.index)
    t_graph = time.perf_counter() - t0
    meta = bh.build_index_meta(g, cfg.alpha)
    eps = cfg.epsilons[0]
    src = bench_sources(cfg.u_count, n_sources)
    r = Runner(g, meta, src, eps, cfg.k, "fp32", 0, 0, 1, "weak", len(src), dev, stream, flush_buf)
    r.run_steps(1, False)  # warm-up (engine + graph instantiation)
    launches0 = _capi.kernel_launches()
    ms, tprof, traces = r.run_steps(1, False, use_gate=True)
    launches = _capi.kernel_launches() - launches0
    sub = Runner(g, meta, src[: max(1, n_sources // 4)], eps, cfg.k, "fp32", 0, 0, 1, "weak",
                 max(1, n_sources // 4), dev, stream, flush_buf)
    pms, prof, ptraces = sub.run_steps(1, True)
    alg = sum(algorithmic_bytes(g, t, prof["rounds"], 4) for t in ptraces)
    roof = roofline_block(g, prof, pms, 1, 4, alg, peak, peak_src, "ncu_c3_round_kernels")
    roof["profiled_on"] = f"{len(sub.src_t)} of the {n_sources} sources (per-kernel event replay)"
    out = {"config": f"c3: |U|={cfg.u_count}, |V|={cfg.v_count}, |E|={cfg.edge_count} Chung-Lu beta 2.1, "
                     f"int weights, alpha={cfg.alpha}, eps={eps}, {n_sources} sources, top-{cfg.k}, fp32",
           "value": n_sources / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "slots": int(tprof["slots"]),
           "rounds": int(tprof["rounds"]), "gpu_launches": int(launches), "graph_build_s": round(t_graph, 1),
           "roofline": roof}
    del r, sub
    _capi._graph_cache.clear()
    del g
    torch.cuda.empty_cache()
    return out


def c1_leg(n_queries: int = 16):
    """Config c1 (configs[0], the reference's CPU-runnable case): single-query
    latency through the public API (one source per call, fp64, the cluster
    small path), beside the bit-exact C port on ONE host core for the same
    sources."""
    import torch

    import paper_2312_06724_b200 as bh
    from oracle import cpu_oracle as O
    from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

    cfg = CONFIGS["c1"]
    g = make_graph(cfg, device=torch.cuda.current_device())
    meta = bh.build_index_meta(g, cfg.alpha)
    eps = cfg.epsilons[0]
    src = bench_sources(cfg.u_count, n_queries)
    bh.bhpp_query_batch(g, meta, src[:1], eps, k=cfg.k, dtype="fp64")  # warm
    ts = []
    for s in src:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bh.bhpp_query_batch(g, meta, [int(s)], eps, k=cfg.k, dtype="fp64")
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    og = O.OracleGraph(g)
    eb = float(meta.eps_split_policy(eps))
    t0 = time.perf_counter()
    for s in src[:4]:
        og.bhpp_query(int(s), cfg.alpha, meta.lam, eb, eps - eb)
    cpu_ms = (time.perf_counter() - t0) / 4 * 1e3
    med = float(np.median(ts)) * 1e3
    return {"config": "c1: |U|=1000, |V|=1500, |E|=10000, alpha=0.15, eps=1e-6, fp64, one source per call",
            "ms_per_query": med, "queries_per_s": 1e3 / med, "queries": len(src),
            "path": "bhpp_query_batch with one source (thread-block-cluster small path)",
            "cpu_one_core_ms_per_query": cpu_ms, "cpu_kind": "port (oracle/bhpp_oracle.c, 1 thread)"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2312_06724_b200 as bh
    from paper_2312_06724_b200 import _capi

    rank, world, local = dist_env()
    # test hooks for the multi-rank path on a one-GPU box (never set by the driver):
    # BH_BENCH_DEVICE pins every rank to one device, BH_DIST_BACKEND=gloo because
    # NCCL refuses two ranks on one device
    if os.environ.get("BH_BENCH_DEVICE"):
        local = int(os.environ["BH_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("BH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)

    cfg, g, src, total = workload(args.config, rank, world, args.scaling, args.batch)
    meta = bh.build_index_meta(g, cfg.alpha)
    eps = cfg.epsilons[0]
    k = cfg.k
    stream = torch.cuda.Stream(device=dev)
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    peak, peak_src = peak_hbm()

    def runner(dtype):
        return Runner(g, meta, src, eps, k, dtype, args.slots, rank, world, args.scaling, total, dev, stream,
                      flush_buf)

    r32 = runner(args.dtype)
    n_local = r32.n
    ms, launches, prof, clk, traces_all, pms = r32.measure(args.steps, args.warmup, clocks_index=local)
    value = total * args.steps / (ms / 1e3)
    s_bytes = 4 if args.dtype == "fp32" else 8
    alg = sum(algorithmic_bytes(g, t, prof["rounds"] // args.steps, s_bytes) for t in traces_all)
    roof = roofline_block(g, prof, pms, args.steps, s_bytes, alg, peak, peak_src, "ncu_round_kernels")

    e2e_src = src  # strong: the whole batch (sharded inside); weak: this rank's sources
    e2e_n = max(args.steps, 10)
    e2e_ms, e2e_steps = e2e_leg(g, meta, e2e_src, eps, k, args.dtype, args.slots, rank, world, args.scaling, dev,
                                stream, flush_buf, e2e_n)
    e2e_value = total * e2e_n / (e2e_ms / 1e3)
    n_in = len(src)

    fp64 = None
    if not args.no_fp64 and args.dtype != "fp64":
        st64 = max(2, args.steps // 2)
        r64 = runner("fp64")
        ms64, _, prof64, _, tr64, _ = r64.measure(st64, 1)
        alg64 = sum(algorithmic_bytes(g, t, prof64["rounds"] // st64, 8) for t in tr64)
        k64 = prof64["ms_prep"] + prof64["ms_vpull"] + prof64["ms_upull"]
        e64_ms, e64_steps = e2e_leg(g, meta, e2e_src, eps, k, "fp64", args.slots, rank, world, args.scaling, dev,
                                    stream, flush_buf, max(3, st64))
        fp64 = {"value": total * st64 / (ms64 / 1e3), "unit": UNIT, "ms_per_step": ms64 / st64,
                "roofline_achieved_gbs": alg64 / (k64 / 1e3) / 1e9 if k64 else None,
                "e2e": {"value": total * max(3, st64) / (e64_ms / 1e3), "unit": UNIT,
                        "ms_per_step": e64_ms / max(3, st64), "step_ms": e64_steps,
                        "h2d_bytes_per_step": int(n_in * 4),
                        "d2h_bytes_per_step": int(n_in * k * (4 + 8) + n_in * _capi.TRACE_DTYPE.itemsize)}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        eb = float(meta.eps_split_policy(eps))
        cpu = cpu_leg(g, src, cfg.alpha, eb, eps - eb, meta.lam, args.cpu_seconds)

    c1 = None
    if rank == 0 and world == 1 and args.config == "c2":
        c1 = c1_leg()

    hbm = None
    if world == 1 and not args.no_c3 and args.config == "c2":
        hbm = c3_leg(args.c3_sources, dev, stream, flush_buf, peak, peak_src)

    if rank == 0:
        t0 = traces_all[0]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32" if args.dtype == "fp32" else "f64",
            "data": f"synthetic (seeded Chung-Lu stand-in for {cfg.name}; reference sampler for sources)",
            "config": config_json(cfg, n_local, world, prof.get("slots", 0), k, args.scaling, total),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(n_in * 4),
                    "d2h_bytes_per_step": int(n_in * k * (4 + 8) + n_in * _capi.TRACE_DTYPE.itemsize),
                    "ms_per_step": e2e_ms / e2e_n, "steps": e2e_n, "step_ms": e2e_steps,
                    "path": ("bhpp_query_sharded (numpy in, device shard + packed all-gather, numpy out)"
                             if args.scaling == "strong" and world > 1 else
                             "bhpp_query_batch (numpy sources in, numpy top-k / traces out), one call per step"
                             + (" + host all-gather of the shards" if world > 1 else ""))},
            "gpu_launches": int(launches),
            "clocks": clk,
            "fp64": fp64,
            "hbm_regime": hbm,
            "latency_c1": c1,
            "trace_sample": {"sel_b": int(t0["sel_b"][0]), "seq_b": int(t0["seq_b"][0]), "sel_f": int(t0["sel_f"][0]),
                             "pi_iters": int(t0["pi_iters"][0]), "n_p_f": int(t0["n_p_f"][0])} if len(t0) else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":  # the CPU reference arm: rank 0 alone does the work
            run_reference(args)
            return
        try:
            import torch

            have = torch.cuda.device_count()
        except Exception:  # noqa: BLE001
            have = 0
        if have < args.gpus and not os.environ.get("BH_BENCH_DEVICE"):
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible CUDA devices, found {have}", file=sys.stderr)
            sys.exit(2)
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
