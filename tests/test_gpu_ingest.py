"""Device graph canonicalisation (bh_csr_build) against the host constructor.

The host constructor is pinned to the reference (tests/test_host.py and the
golden fixtures); the device build must give bit-identical CSR arrays and ws
sums, and the same errors, on the configurations' graphs and on adversarial
edge lists (shuffled input order, non-integer weights whose sums depend on
accumulation order, hubs, a repeated pair).
"""

import numpy as np
import pytest

from golden_io import config_graph
from paper_2312_06724_b200 import BipartiteGraph, DataError
from paper_2312_06724_b200.synth import chung_lu_edges

pytestmark = pytest.mark.gpu

FIELDS = ("u_indptr", "u_indices", "u_weights", "v_indptr", "v_indices", "v_weights", "ws_u", "ws_v",
          "deg_u", "deg_v")


def same(a, b):
    assert a.edge_count == b.edge_count and a.u_count == b.u_count and a.v_count == b.v_count
    for f in FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        assert x.dtype == y.dtype, f
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), f  # bitwise
    assert a.fingerprint == b.fingerprint


def edges_of(g):
    eu = np.repeat(np.arange(g.u_count), np.diff(g.u_indptr))
    return eu, g.u_indices.astype(np.int64), g.u_weights.copy()


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c4s"])
def test_device_build_matches_host_on_configs(cfg):
    g = config_graph(cfg)
    eu, ev, ew = edges_of(g)
    perm = np.random.default_rng(5).permutation(eu.size)  # input order must not matter
    d = BipartiteGraph.from_arrays(g.u_count, g.v_count, eu[perm], ev[perm], ew[perm], device=0)
    same(g, d)


def test_order_sensitive_weight_sums_bit_identical():
    eu, ev, _ = chung_lu_edges(3000, 5000, 60000, 2.1, 1.9, "unit", 11)
    ew = np.random.default_rng(2).random(eu.size) * 10.0 + 1e-3  # sums depend on addition order
    h = BipartiteGraph.from_arrays(3000, 5000, eu, ev, ew)
    d = BipartiteGraph.from_arrays(3000, 5000, eu, ev, ew, device=0)
    same(h, d)


def test_device_build_errors_match_host():
    eu = np.array([0, 1, 1, 0])
    ev = np.array([0, 0, 1, 0])  # (0, 0) twice
    ew = np.ones(4)
    for dev in (None, 0):
        with pytest.raises(DataError, match="duplicate edge passed to constructor"):
            BipartiteGraph.from_arrays(2, 2, eu, ev, ew, device=dev)
    for dev in (None, 0):  # v1 has no edge
        with pytest.raises(DataError, match="isolated node on V side: 'v1'"):
            BipartiteGraph.from_arrays(2, 2, np.array([0, 1]), np.array([0, 0]), np.ones(2), device=dev)
    with pytest.raises(DataError, match="out of range on the V side"):
        BipartiteGraph.from_arrays(2, 2, np.array([0, 1]), np.array([0, 2]), np.ones(2), device=0)


def test_bpgr_round_trip_on_device():
    g = config_graph("c2s")
    d = BipartiteGraph.from_bytes(g.to_bytes(), device=0)
    same(g, d)
