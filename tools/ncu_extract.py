"""Summarise ncu reports into profiles/: per-kernel time, DRAM bytes, key rates.

    python tools/ncu_extract.py gpurun_out/prof.ncu-rep > profiles/<name>.md
    python tools/ncu_extract.py --traffic gpurun_out/prof.ncu-rep > profiles/roofline_traffic.json
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time_us", 1e-3),
    ("dram__bytes_read.sum", "dram_read_MB", 1.0),
    ("dram__bytes_write.sum", "dram_write_MB", 1.0),
    ("smsp__inst_executed.sum", "warp_inst_M", 1e-6),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1.0),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct", 1.0),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct", 1.0),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_throughput_pct", 1.0),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
    ("launch__grid_size", "grid", 1.0),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    units = dict(zip(h, r[1]))
    return [dict(zip(h, x)) for x in r[2:]], units


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def main():
    traffic = "--traffic" in sys.argv
    rep = [a for a in sys.argv[1:] if not a.startswith("--")][0]
    data, units = rows(rep)
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        for k, short, scale in KEYS:
            v = to_float(d.get(k, ""))
            if v is None:
                continue
            u = units.get(k, "")
            if k.startswith("dram__bytes"):
                scale = {"byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3, "GB": 1e3}.get(u, 1.0)
            if k == "gpu__time_duration.sum":
                scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
            agg[name][short].append(v * scale)
    if traffic:
        per = {n: {s: sum(v) / len(v) for s, v in m.items()} for n, m in agg.items()}
        json.dump({"source": rep, "kernels": per}, sys.stdout, indent=1)
        return
    cols = [s for _, s, _ in KEYS]
    print("| kernel | launches | " + " | ".join(cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    for n, m in agg.items():
        cnt = len(m["time_us"])
        vals = [f"{sum(m[c]) / len(m[c]):.3g}" if m[c] else "-" for c in cols]
        print(f"| {n} | {cnt} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
