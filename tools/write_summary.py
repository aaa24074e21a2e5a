"""profiles/<round>_summary.md from the measurement set of tools/measure_round.sh.

    python tools/write_summary.py gpurun_out/bench_final.json gpurun_out/launches_bench.csv \
        gpurun_out/prof_round_final.ncu-rep > profiles/r01_summary.md
"""
import json
import subprocess
import sys

bench, launches, rep = sys.argv[1:4]
d = json.loads(open(bench).read().strip().splitlines()[-1])
r = d["roofline"]
b = r["breakdown_ms_per_step"]
launch = subprocess.run([sys.executable, "tools/ncu_summary.py", launches], capture_output=True, text=True).stdout
tab = subprocess.run([sys.executable, "tools/ncu_extract.py", rep], capture_output=True, text=True).stdout
steps = d["steps"]
print(f"""# Round 1 profiles (B200, sm_100a) -- config c2, fp32 storage / fp64 accumulation, B = 64 slots

Build: `k_pull_sw` pulls (shared-memory windows; V 7 rows in flight at 4 blocks/SM, U 8 rows at 4 blocks/SM), predicated
elementwise K1/K1a (one node per thread; K1 4 blocks/SM, K1a software-pipelined at 3; r_A := 0 and est += alpha r in K1a),
K4 with one load round trip, one CUDA graph per batch (WHILE node, PDL launches; K5 under an IF node on a
branch parallel to the next round's K1..K1a).
Commands: `tools/measure_round.sh` (bench line, reference arm, launch list, ncu full set).

## Bench line (`python bench.py`: {steps} timed steps, {d['warmup']} warm-up)

- value **{d['value']:.0f} queries/s** (device-timed steps {r['timed_step_ms']} ms, each enqueued
  behind a device start gate); e2e through the public numpy API **{d['e2e']['value']:.0f} queries/s**;
  fp64 mode {d['fp64']['value']:.0f} queries/s; SM clock {d['clocks']['sm_mhz']} MHz, no throttle reasons.
- CPU baseline (bit-exact C port of the reference, {d['cpu_baseline']['cores']} host threads):
  {d['cpu_baseline']['value']:.1f} queries/s -> e2e / CPU = {d['e2e']['value'] / d['cpu_baseline']['value']:.0f}x.
- Per-step CUDA-event breakdown (replay of the timed steps with per-kernel events):
  prep (K1+K1a) {b['ms_prep']:.2f} ms, V pull {b['ms_vpull']:.2f} ms, U pull {b['ms_upull']:.2f} ms,
  control (K4+K5) {b['ms_control']:.2f} ms; {r['launches'] // steps} rounds per step.
- Roofline, dominant kernel (K2 V pull, {100 * r['share_of_step']:.0f} % of the replayed step):
  {r['algorithmic_bytes_per_launch'] / 1e6:.1f} MB algorithmic per launch (SURVEY 8(d), one SpMM half) /
  {r['launch_us']:.1f} us = {r['achieved']:.0f} GB/s = **{r['frac']:.3f}** of the measured {r['peak']:.0f} GB/s;
  ncu DRAM traffic per launch {r['traffic'] / 1e6:.1f} MB (cold cache).  The pull is an L2-served
  gather: {r['gather']['achieved_tbs']:.2f} TB/s of operand rows (E x B x s per pull) against the 13-17 TB/s
  ceiling of `tools/gather_bench.cu`; latency-bound (issue ~52 %, < 1 eligible warp per scheduler);
  `r01_pull_variants.md` lists the transports tried (TMA gather4, cp.async ring, fused combine).
- Round unit (K1+K2+K3+K1a, SURVEY 8(d) push/PI round): {r['round']['achieved_gbs']:.0f} GB/s =
  {r['round']['frac']:.3f} of peak; ncu traffic {r['round']['traffic_per_round'] / 1e6:.0f} MB vs
  {r['round']['algorithmic_bytes_per_round'] / 1e6:.0f} MB algorithmic per round.

## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, `BH_NO_GRAPH=1 python bench.py --steps 2 --warmup 1 --no-cpu --no-fp64`)

Raw: `r01_launches_bench_c2.csv.gz` (also holds the IndexMeta power iteration, `k_pull_small<1, double>`).
Serialised cold-cache launch times; the kernel shares agree with the CUDA-event breakdown.

```
{launch}```

## ncu --set full, one launch of each round kernel (round 70 of a batch)

Raw per-kernel metrics: `r01_ncu_round_kernels.json` (bench.py reads the DRAM bytes from it).

{tab}
Reading:
- The two pulls are ~58 % of device time; each gathers 2e6 operand rows of 256 B per round from
  L2 (~69 % L2 hit); k_pull_sw executes 19-20 warp instructions per edge on the V side and 16 on
  the U side (22.5 / 18 for the round-1 baseline k_pull).
- K1/K1a are latency-bound elementwise passes.  Moving the residue zeroing and the estimate
  update from K1 into K1a (K1a re-takes K1's threshold decision on the same r), predicating the
  per-slot logic and running one node per thread at 4 blocks/SM took prep from 6.5 to 5.6 ms per step.
- K4 is latency-bound control (~8 us per round).  K5 runs only after rounds where a slot
  finished, under a CUDA-graph IF node, concurrently with the next round's K1..K1a.  A finished
  slot is refilled one round later.  Its radix select no longer uses a 64-bit shared atomic,
  which compiled to a CAS loop.  In the eager launch list below, K5 is still launched every
  round and is a no-op when no slot finished.
""")
