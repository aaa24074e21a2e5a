"""load_edge_list (reference bigraph.py:272-350) against reference-produced cases.

tests/golden/edge_lists.json holds, per case, the input and what the
reference produced (labels, U-side CSR bits, ws bits, fingerprint) or raised.
Both parser paths must reproduce it: the native one (bh_edge_list_parse, ASCII
input with plain decimal weights) and the reference-semantics line loop (every
other input and every error).  Host-only: runs without a GPU.
"""

import io
import json
import tempfile
from pathlib import Path

import numpy as np
import pytest

import paper_2312_06724_b200 as bh
from paper_2312_06724_b200 import bigraph

CASES = json.loads((Path(__file__).resolve().parent / "golden" / "edge_lists.json").read_text())


def load(case, tmp_path):
    text, how = case["text"], case["how"]
    kw = dict(delimiter=case["delimiter"], default_weight=case["default_weight"])
    if how == "text":
        return bh.load_edge_list(io.StringIO(text), **kw)
    if how == "bytes":
        return bh.load_edge_list(io.BytesIO(text.encode("utf-8")), **kw)
    p = tmp_path / "edges.txt"
    p.write_bytes(text.encode("utf-8"))
    return bh.load_edge_list(p, **kw)


def check(case, tmp_path):
    if "error" in case:
        with pytest.raises(bh.DataError) as ei:
            load(case, tmp_path)
        assert type(ei.value).__name__ == case["error"]["type"]
        assert str(ei.value) == case["error"]["message"]
        return
    g = load(case, tmp_path)
    ok = case["ok"]
    assert list(g.u_labels) == ok["u_labels"] and list(g.v_labels) == ok["v_labels"]
    assert g.u_indptr.tolist() == ok["u_indptr"] and g.u_indices.tolist() == ok["u_indices"]
    assert [float(x).hex() for x in g.u_weights] == ok["u_weights_hex"]
    assert [float(x).hex() for x in g.ws_u] == ok["ws_u_hex"]
    assert g.fingerprint == ok["fingerprint"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_matches_reference(case, tmp_path):
    check(case, tmp_path)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_python_loop_matches_reference(case, tmp_path, monkeypatch):
    monkeypatch.setattr(bigraph, "_edge_list_native", lambda *a: None)
    check(case, tmp_path)


def test_native_path_taken_for_plain_ascii(monkeypatch):
    seen = []
    orig = bigraph._edge_list_native

    def spy(*a):
        r = orig(*a)
        seen.append(r is not None)
        return r

    monkeypatch.setattr(bigraph, "_edge_list_native", spy)
    bh.load_edge_list(io.StringIO("a x 1\nb y 2.5e-3\n"))
    bh.load_edge_list(io.StringIO("a x 1_0\n"))
    assert seen == [True, False]


def test_native_parser_scales():
    """A 2e5-line file: native and Python paths agree bit for bit."""
    rng = np.random.default_rng(1)
    u = rng.integers(0, 5000, 200000)
    v = rng.integers(0, 9000, 200000)
    w = rng.random(200000) * 5 + 0.01
    text = "".join(f"u{a}\tv{b}\t{float(c)!r}\n" for a, b, c in zip(u, v, w))
    g1 = bh.load_edge_list(io.StringIO(text))
    orig = bigraph._edge_list_native
    try:
        bigraph._edge_list_native = lambda *a: None
        g2 = bh.load_edge_list(io.StringIO(text))
    finally:
        bigraph._edge_list_native = orig
    assert g1.fingerprint == g2.fingerprint
    assert np.array_equal(g1.ws_v.view(np.uint64), g2.ws_v.view(np.uint64))
