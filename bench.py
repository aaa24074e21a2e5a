#!/usr/bin/env python
"""bench.py -- BHPP source queries/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N   (one rank per GPU, NCCL)

Workload (N=1): BASELINE.json configs[1] ("c2"): seeded Chung-Lu bipartite
graph |U|=1e5, |V|=2e5, |E|=2e6, exponent 2.2, integer weights U{1..10},
alpha=0.15, eps=1e-7, 64 sources drawn like the reference's bench
(cli.py:415-417), top-50 per query.  A step = one SS-BI-PUSH pass (backward
push, forward push, power iteration, combine, top-k) over the 64 sources.
Weak scaling: every rank runs its own 64 sources on a replica of the graph;
the per-shard top-k is all-gathered with NCCL inside the step.

value   : queries/s, inputs resident in HBM, device-timed (CUDA events on the
          engine stream, L2 flushed with a 256 MiB write between steps,
          outside the timed interval), max over ranks.
e2e     : same metric through the public host API bhpp_query_batch (numpy
          sources in, numpy top-k/traces out; H2D and D2H inside the timing).
roofline: the round kernels (K1 prep + K2 V pull + K3 U pull), algorithmic
          bytes of SURVEY.md section 8(d) / their CUDA-event time.
cpu_baseline / --impl reference: the bit-exact C port of the reference
          (oracle/) on all host cores, the reference's thread-pool pattern.
"""

from __future__ import annotations

import argparse
import json
import os
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
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 side measurement")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def workload(cfg_name: str, rank: int):
    from paper_2312_06724_b200.rng import substream
    from paper_2312_06724_b200.synth import CONFIGS, bench_sources, make_graph

    cfg = CONFIGS[cfg_name]
    g = make_graph(cfg)
    n = cfg.n_sources or cfg.u_count
    if rank == 0:
        src = bench_sources(cfg.u_count, n)
    else:
        src = substream(0, "bench-queries", rank).choice(cfg.u_count, n, replace=False).astype(np.int64)
    return cfg, g, src


def config_json(cfg, n_local, world, slots, k):
    return {
        "workload": f"{cfg.name}: |U|={cfg.u_count}, |V|={cfg.v_count}, |E|={cfg.edge_count} Chung-Lu "
                    f"beta_u={cfg.beta_u} beta_v={cfg.beta_v} weights={cfg.weights}, alpha={cfg.alpha}, "
                    f"eps={cfg.epsilons[0]}, {n_local} sources/GPU, top-{k}",
        "queries_per_gpu": int(n_local),
        "global_batch": int(n_local * world),
        "top_k": int(k),
        "slots": int(slots),
        "parallelism": f"query-shard x{world} (graph replicated)",
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


def _ncu_kernels():
    p = REPO / "profiles" / "r01_ncu_round_kernels.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text())["kernels"]
    except Exception:
        return None


def ncu_round_traffic():
    """DRAM bytes (read + write) of one round's K1+K2+K3+K1a from the committed
    ncu capture (profiles/r01_ncu_round_kernels.json), or None."""
    ks = _ncu_kernels()
    if not ks:
        return None
    return 1e6 * sum(v.get("dram_read_MB", 0) + v.get("dram_write_MB", 0)
                     for k, v in ks.items() if k.startswith(("k_push", "k_pull", "k_combine")))


def ncu_vpull_traffic():
    """DRAM bytes (read + write) of one V-pull launch from the same capture."""
    ks = _ncu_kernels()
    if not ks:
        return None
    for k, v in ks.items():  # k_pull*<B, T, SIDE, ...>: SIDE 0 is the V pull
        if k.startswith("k_pull") and k.split("<", 1)[1].split(",")[2].strip().rstrip(">") == "0":
            return 1e6 * (v.get("dram_read_MB", 0) + v.get("dram_write_MB", 0))
    return None


def c3_hbm_reference(peak):
    """DRAM throughput of the round kernels in the HBM-resident regime (config c3,
    operands larger than L2) from the committed ncu capture
    (profiles/r01_ncu_c3_round_kernels.json), as fractions of the HBM peak."""
    p = REPO / "profiles" / "r01_ncu_c3_round_kernels.json"
    if not p.exists() or not peak:
        return None
    try:
        ks = json.loads(p.read_text())["kernels"]
    except Exception:
        return None
    out = {}
    for k, v in ks.items():
        gbs = (v["dram_read_MB"] + v["dram_write_MB"]) / 1e3 / (v["time_us"] / 1e6)
        out[k] = {"dram_gbs": round(gbs, 1), "frac": round(gbs / peak, 3)}
    return {"config": "c3 (|E|=1e8, 128 slots): operands exceed L2, gathers served by HBM",
            "source": "profiles/r01_ncu_c3_round_kernels.json (ncu --set full, one launch each)",
            "kernels": out}


def peak_hbm():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
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

    cfg, g, src = workload(args.config, 0)
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
        "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Chung-Lu, configs[1])",
        "config": config_json(cfg, len(src), 1, 0, cfg.k),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{per_step} queries per step ({threads} threads) of the bench sources, "
                                   "bit-exact C port of the reference (oracle/), host wall clock"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference is pure Python (numpy/scipy); its path is timed through its bit-exact C port",
    }
    print(json.dumps(line), flush=True)


# -----------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2312_06724_b200 as bh
    from paper_2312_06724_b200 import _capi
    from paper_2312_06724_b200.bhpp_query import query_batch_device, query_wait
    from paper_2312_06724_b200.distributed import gather_results

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    cfg, g, src = workload(args.config, rank)
    meta = bh.build_index_meta(g, cfg.alpha)
    eps = cfg.epsilons[0]
    eps_b = float(meta.eps_split_policy(eps))
    eps_f = eps - eps_b
    k = cfg.k
    n = len(src)
    stream = torch.cuda.Stream(device=dev)
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # device-side start gate for the timed steps (graph mode only: the eager
    # round loop synchronises inside the call)
    gated = not os.environ.get("BH_NO_GRAPH") and not os.environ.get("BH_BENCH_NO_GATE")
    gate = torch.zeros(1, dtype=torch.int32).pin_memory()

    def measure(dtype: str, steps: int, warmup: int):
        """Timed steps (device events around each step only), then the same
        steps replayed with per-kernel events for the roofline breakdown."""
        dg = _capi.device_graph(g, dtype, device=local)
        src_t = torch.from_numpy(src.astype(np.int32)).to(dev)
        tk_i = torch.empty((n, k), dtype=torch.int32, device=dev)
        tk_s = torch.empty((n, k), dtype=torch.float64, device=dev)
        tr = torch.empty((n, _capi.TRACE_DTYPE.itemsize), dtype=torch.uint8, device=dev)
        all_i = torch.empty((world * n, k), dtype=torch.int32, device=dev)
        all_s = torch.empty((world * n, k), dtype=torch.float64, device=dev)

        def step(async_=False):
            query_batch_device(dg, meta, eps_b, eps_f, src_t.data_ptr(), n, k, tk_i.data_ptr(), tk_s.data_ptr(),
                               tr.data_ptr(), slots=args.slots or None, stream=stream.cuda_stream, async_=async_)
            if world > 1:  # gather the shard top-k on the same stream (NCCL)
                with torch.cuda.stream(stream):
                    dist.all_gather_into_tensor(all_i, tk_i)
                    dist.all_gather_into_tensor(all_s, tk_s)

        def run_steps(nsteps, profiled, use_gate=False):
            _capi.set_profiling(profiled)
            ms = 0.0
            per_step = []
            prof = {"ms_prep": 0.0, "ms_vpull": 0.0, "ms_upull": 0.0, "ms_control": 0.0, "rounds": 0, "slots": 0}
            traces = []
            for _ in range(nsteps):
                with torch.cuda.stream(stream):
                    flush_buf.fill_(1.0)  # evict L2 (256 MiB > 126 MB) outside the timed interval
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                if use_gate and gated and not profiled:
                    # the whole step is enqueued behind a gate before the device
                    # starts it: e0..e1 is device time only, no host submission gaps
                    gate[0] = 0
                    _capi.check(_capi.lib().bh_stream_gate(stream.cuda_stream, gate.data_ptr()))
                    e0.record(stream)
                    step(async_=True)
                    e1.record(stream)
                    gate[0] = 1
                    query_wait(dg)
                else:
                    e0.record(stream)
                    step()
                    e1.record(stream)
                e1.synchronize()
                ms += e0.elapsed_time(e1)
                per_step.append(e0.elapsed_time(e1))
                st = dg.last_run_stats()
                prof.setdefault("step_rounds", []).append(int(st["rounds"]))
                for key in ("ms_prep", "ms_vpull", "ms_upull", "ms_control", "rounds"):
                    prof[key] += st[key]
                prof["slots"] = st["slots"]
                traces.append(tr.cpu().numpy().copy().view(_capi.TRACE_DTYPE).reshape(-1))
            _capi.set_profiling(False)
            prof["step_ms"] = per_step
            return ms, prof, traces

        # warm-up: ungated first (graph instantiation, first NCCL use), the last one gated
        run_steps(max(1, warmup - 1), False)
        if warmup > 1:
            run_steps(1, False, use_gate=True)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        clocks = Clocks(local) if not os.environ.get("BH_BENCH_NO_CLOCKS") else None
        if clocks:
            clocks.start()
        launches0 = _capi.kernel_launches()
        ms, tprof, traces_all = run_steps(steps, False, use_gate=True)
        launches = _capi.kernel_launches() - launches0
        clk = clocks.stop() if clocks else {"sm_mhz": None, "reasons": ["not sampled (BH_BENCH_NO_CLOCKS)"]}
        torch.cuda.synchronize(dev)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        pms, prof, ptraces = run_steps(steps, True)
        prof["timed_step_ms"] = tprof["step_ms"]
        prof["timed_step_rounds"] = tprof["step_rounds"]
        return ms, launches, prof, clk, ptraces, pms

    # headline: fp32 storage / fp64 accumulation
    ms, launches, prof, clk, traces_all, pms = measure(args.dtype, args.steps, args.warmup)
    value = world * n * args.steps / (ms / 1e3)
    s_bytes = 4 if args.dtype == "fp32" else 8
    alg = sum(algorithmic_bytes(g, t, prof["rounds"] // args.steps, s_bytes) for t in traces_all)
    kern_ms = prof["ms_prep"] + prof["ms_vpull"] + prof["ms_upull"]
    # dominant kernel: the V pull, SURVEY 8(d) bytes of one SpMM half per launch
    B_slots = prof.get("slots", 0) or n
    v_bytes = g.edge_count * (4 + s_bytes) + (g.v_count + 1) * 4 + B_slots * s_bytes * (g.u_count + g.v_count)
    v_launch_us = prof["ms_vpull"] * 1e3 / max(1, prof["rounds"])
    v_achieved = v_bytes / (v_launch_us / 1e6) / 1e9 if v_launch_us > 0 else None
    achieved = alg / (kern_ms / 1e3) / 1e9 if kern_ms > 0 else None
    peak, peak_src = peak_hbm()

    # e2e through the public host API (numpy in, numpy out; copies inside)
    e2e_ms = 0.0
    e2e_steps = []
    for _ in range(2):
        bh.bhpp_query_batch(g, meta, src, eps, k=k, dtype=args.dtype, slots=args.slots or None,
                            stream=stream.cuda_stream)
    e2e_n = max(args.steps, 10)  # e2e steps are cheap: at least 10 samples
    gc_events = [0]
    if os.environ.get("BH_BENCH_E2E_DIAG"):
        import gc
        gc.callbacks.append(lambda phase, info: gc_events.__setitem__(0, gc_events[0] + (phase == "start")))
    for _ in range(e2e_n):
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        th0 = time.perf_counter()
        e0.record(stream)
        res = bh.bhpp_query_batch(g, meta, src, eps, k=k, dtype=args.dtype, slots=args.slots or None,
                                  stream=stream.cuda_stream)
        th1 = time.perf_counter()
        if world > 1:
            from paper_2312_06724_b200.distributed import gather_results as _gr
            with torch.cuda.stream(stream):
                _gr(res.topk_index, res.topk_score, res.traces, world * n, rank, world, device=dev)
        e1.record(stream)
        th2 = time.perf_counter()
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        e2e_steps.append(round(e0.elapsed_time(e1), 3))
        if os.environ.get("BH_BENCH_E2E_DIAG"):
            print(f"[e2e diag] event {e0.elapsed_time(e1):.3f} ms, host call {1e3 * (th1 - th0):.3f} ms, "
                  f"engine {1e3 * res.timing['total']:.3f} ms, to e1 {1e3 * (th2 - th0):.3f} ms, gc {gc_events[0]}",
                  file=sys.stderr, flush=True)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * n * e2e_n / (e2e_ms / 1e3)

    fp64 = None
    if not args.no_fp64 and args.dtype != "fp64":
        st64 = max(2, args.steps // 2)
        ms64, _, prof64, _, tr64, _ = measure("fp64", st64, 1)
        alg64 = sum(algorithmic_bytes(g, t, prof64["rounds"] // st64, 8) for t in tr64)
        k64 = prof64["ms_prep"] + prof64["ms_vpull"] + prof64["ms_upull"]
        fp64 = {"value": world * n * st64 / (ms64 / 1e3), "unit": UNIT, "ms_per_step": ms64 / st64,
                "roofline_achieved_gbs": alg64 / (k64 / 1e3) / 1e9 if k64 else None}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_leg(g, src, cfg.alpha, eps_b, eps_f, meta.lam, args.cpu_seconds)

    if rank == 0:
        t0 = traces_all[0]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.dtype == "fp32" else "f64",
            "data": "synthetic (seeded Chung-Lu stand-in for configs[1]; reference sampler for sources)",
            "config": config_json(cfg, n, world, prof.get("slots", 0), k),
            "roofline": {
                "bound": "hbm", "achieved": v_achieved, "peak": peak, "unit": "GB/s",
                "frac": v_achieved / peak if v_achieved else None, "traffic": ncu_vpull_traffic(),
                "kernel": "K2 V pull (k_pull_sw, SIDE_V), the dominant kernel",
                "algorithmic_bytes_per_launch": v_bytes,
                "algorithmic_model": "E(i+s) + (|V|+1) o + B s (|U| + |V|), i = o = 4 (SURVEY 8(d), one SpMM half)",
                "launch_us": v_launch_us, "launches": int(prof["rounds"]),
                "share_of_step": prof["ms_vpull"] / pms if pms else None,
                "traffic_note": "DRAM read+write bytes of one V-pull launch from one ncu --set full capture "
                                "(profiles/r01_ncu_round_kernels.json, cold cache)",
                "round": {
                    "unit": "push/PI round = K1 push + K2 V-pull + K3 U-pull + K1a combine (SURVEY 8(d) unit)",
                    "achieved_gbs": achieved, "frac": achieved / peak if achieved else None,
                    "algorithmic_bytes_per_round": alg / max(1, prof["rounds"]),
                    "traffic_per_round": ncu_round_traffic(),
                    "share_of_step": kern_ms / pms if pms else None,
                },
                "gather": {"bytes_per_round": 2 * g.edge_count * prof.get("slots", 0) * s_bytes,
                           "achieved_tbs": (2 * g.edge_count * prof.get("slots", 0) * s_bytes * prof["rounds"]
                                            / ((prof["ms_vpull"] + prof["ms_upull"]) / 1e3) / 1e12)
                           if prof["ms_vpull"] + prof["ms_upull"] > 0 else None,
                           "note": "operand-row gathers of the two pulls (E x B x s each), L2-served; "
                                   "tools/gather_bench.cu ceiling 13-17 TB/s"},
                "algorithmic_bytes_per_step": alg / args.steps, "kernel_ms_per_step": kern_ms / args.steps,
                "rounds_per_step": prof["rounds"] / args.steps,
                "timing": "per-kernel CUDA events on the engine stream, in a replay of the timed steps "
                          "(the headline value is timed without per-kernel events; each timed step is "
                          "enqueued behind a device start gate, so e0..e1 is device time only)",
                "breakdown_ms_per_step": {k2: prof[k2] / args.steps for k2 in ("ms_prep", "ms_vpull", "ms_upull", "ms_control")},
                "peak_source": peak_src,
                "hbm_regime_reference": c3_hbm_reference(peak),
                "timed_step_ms": [round(x, 3) for x in prof.get("timed_step_ms", [])],
                "profiled_step_ms": [round(x, 3) for x in prof.get("step_ms", [])],
                "timed_step_rounds": prof.get("timed_step_rounds"),
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(n * 4),
                    "d2h_bytes_per_step": int(n * k * (4 + 8) + n * _capi.TRACE_DTYPE.itemsize),
                    "ms_per_step": e2e_ms / e2e_n, "steps": e2e_n, "step_ms": e2e_steps,
                    "path": "bhpp_query_batch (numpy sources in, numpy top-k / traces out), one call per step"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "fp64": fp64,
            "trace_sample": {"sel_b": int(t0["sel_b"][0]), "seq_b": int(t0["seq_b"][0]), "sel_f": int(t0["sel_f"][0]),
                             "pi_iters": int(t0["pi_iters"][0]), "n_p_f": int(t0["n_p_f"][0])},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
