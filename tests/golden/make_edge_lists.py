"""Golden cases for load_edge_list, produced by the REFERENCE (bigraph.py:272-350).

Run in the dev container (where /root/reference exists):
    python tests/golden/make_edge_lists.py
Writes edge_lists.json: for each case its input (text, how it is passed,
delimiter, default weight) and the reference's outcome -- the graph's labels,
U-side CSR, ws and fingerprint, or the exception type and message.
"""

from __future__ import annotations

import io
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import bipush  # noqa: E402

rng = np.random.default_rng(20240601)
big = []
for i in range(1500):
    u, v = f"user{rng.integers(0, 60)}", f"item{rng.integers(0, 90)}"
    w = rng.choice([f"{rng.random() * 10:.17g}", f"{rng.integers(1, 10)}", f"{rng.random():.3e}", f"+{rng.random():.4f}"])
    sep = rng.choice([" ", "\t", "  ", " \t "])
    big.append(f"{u}{sep}{v}{sep}{w}")
    if rng.random() < 0.05:
        big.append("# comment " + str(i))
    if rng.random() < 0.03:
        big.append("   ")

CASES = [
    ("basic", "a x 1\nb x 2.5\n# note\n\na y 0.1\na x 0.5\n", "text", None, None),
    ("crlf_cr_tabs", "a\tx\t1\r\nb x 2\rc  y   3  \r\n\x0bd\x0cz\x1c4\x1f\n", "bytes", None, None),
    ("comma_empty_field", "a,,1\nb,x,2\n", "text", ",", None),
    ("multichar_delim", "a::x::1.5\nb::x::.5\nc::y::5.\n", "path", "::", None),
    ("default_weight", "a x\nb x 3\nc y\n", "text", None, 2.0),
    ("two_cols_no_default", "a x 1\nb y\n", "text", None, None),
    ("bad_weight", "a x 1\nb y abc\n", "text", None, None),
    ("inf_weight", "a x inf\n", "text", None, None),
    ("underscore_weight", "a x 1_000\nb x 2\n", "text", None, None),
    ("hex_weight", "a x 0x10\n", "text", None, None),
    ("negative_weight", "a x 1\nb x -1\n", "text", None, None),
    ("zero_weight", "a x 0\n", "bytes", None, None),
    ("underflow_weight", "a x 1e-400\n", "text", None, None),
    ("subnormal_weight", "a x 1e-310\nb x 4.9e-324\n", "text", None, None),
    ("both_sides_later", "a b 1\nb c 1\n", "text", None, None),
    ("both_sides_same_line", "a a 1\n", "text", None, None),
    ("four_columns", "a x 1 2\n", "text", None, None),
    ("only_comments", "# x\n\n   \n", "text", None, None),
    ("non_ascii", "café x 1\nnaïve y 2 \n", "path", None, None),
    ("bad_default", "a x\n", "text", None, 0.0),
    ("plus_signs_exponents", "a x +1\nb x 1E+2\nc x 2e-3\nd y 0001.2500\n", "text", None, None),
    ("random_1500_lines", "\n".join(big) + "\n", "bytes", None, None),
]


def run(text, how, delimiter, default_weight):
    if how == "text":
        return bipush.load_edge_list(io.StringIO(text), delimiter=delimiter, default_weight=default_weight)
    if how == "bytes":
        return bipush.load_edge_list(io.BytesIO(text.encode("utf-8")), delimiter=delimiter,
                                     default_weight=default_weight)
    with tempfile.NamedTemporaryFile("wb", suffix=".txt", delete=False) as f:
        f.write(text.encode("utf-8"))
    try:
        return bipush.load_edge_list(f.name, delimiter=delimiter, default_weight=default_weight)
    finally:
        Path(f.name).unlink()


out = []
for name, text, how, delim, dw in CASES:
    rec = {"name": name, "text": text, "how": how, "delimiter": delim, "default_weight": dw}
    try:
        g = run(text, how, delim, dw)
        rec["ok"] = {"u_labels": list(g.u_labels), "v_labels": list(g.v_labels),
                     "u_indptr": g.u_indptr.tolist(), "u_indices": g.u_indices.tolist(),
                     "u_weights_hex": [float(x).hex() for x in g.u_weights],
                     "ws_u_hex": [float(x).hex() for x in g.ws_u], "fingerprint": g.fingerprint}
    except Exception as e:  # noqa: BLE001 -- the reference's error is the expected outcome
        rec["error"] = {"type": type(e).__name__, "message": str(e)}
    out.append(rec)
(HERE / "edge_lists.json").write_text(json.dumps(out, indent=1))
print(f"{len(out)} cases:", ", ".join(f"{r['name']}={'ok' if 'ok' in r else r['error']['type']}" for r in out))
