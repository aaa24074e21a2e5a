"""Merge gpurun_out/cfg_<config>.json (tools/run_configs.py output) into a markdown table + JSON.

    python tools/configs_table.py c1 c5 c3 c4 > profiles/<round>_configs.md
"""
import json
import sys
from pathlib import Path

rows, raw = [], {}
for c in sys.argv[1:]:
    d = json.loads(Path(f"gpurun_out/cfg_{c}.json").read_text().strip().splitlines()[-1])
    raw[c] = d
    gr = d["graph"]
    for r in d["runs"]:
        p = r.get("parity", {})
        tm = r["trace_mean"]
        rel = next((v for k, v in p.items() if k.endswith("topk_max_rel_err")), None)
        rows.append(f"| {c} | {gr['u']:.0e} / {gr['v']:.0e} / {gr['e']:.0e} | {r['eps']:g} | {d['dtype']} | "
                    f"{r['n_sources']} | {r['queries_per_s']:.1f} | {r['slots']} | {r['rounds']} | "
                    f"{tm['sel_b']:.1f} / {tm['seq_b']:.1f} / {tm['sel_f']:.1f} / {tm['pi_iters']:.1f} | "
                    f"{'pass' if p.get('pass') else 'FAIL'} ({p.get('sources')}) | {p.get('fp64_max_abs_err', 0):.1e} | "
                    f"{'identical' if p.get('fp64_traces_identical') else 'DIFFER'} | {rel:.1e} |")
print("| config | |U| / |V| / |E| | eps | dtype | sources | queries/s | slots | rounds | "
      "mean sel_b / seq_b / sel_f / PI | oracle parity (P) | fp64 max abs err | traces | top-k max rel err |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
print()
print("Host-side one-off costs: " + "; ".join(
    f"{c} graph {d['graph_build_s']:.1f} s (seeded generator + device CSR canonicalisation), "
    f"device IndexMeta {d['meta_s']:.2f} s" for c, d in raw.items()))
Path("gpurun_out/configs_merged.json").write_text(json.dumps(raw, indent=1))
