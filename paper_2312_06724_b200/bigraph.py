"""Host-side weighted bipartite graph: the upload source of the device graph store.

Mirrors the CSR core of the reference ``bipush.BipartiteGraph``
(pkg/src/bipush/bigraph.py:40-111): canonical (u, v)-sorted U-CSR, the V-CSR
mirror, per-node weight sums ``ws_u``/``ws_v`` (np.bincount in canonical edge
order, so they are bit-identical to the reference's), degrees, labels, the
BPGR serialisation (bigraph.py:192-251) and its sha256 ``fingerprint``
(bigraph.py:260-263).  Because the bytes are identical, an ``IndexMeta`` built
by either package validates against a graph from the other.

The device engine also accepts a reference ``bipush.BipartiteGraph`` directly:
it only reads the attributes listed in ``CSR_ATTRS``.

Unlike the reference, large synthetic graphs can be built from integer arrays
without materialising Python label lists (``from_arrays``); labels are then
"u{i}" / "v{j}", exactly what the reference's ``synth_bipartite`` produces.
"""

from __future__ import annotations

import hashlib
import io
import struct
from functools import cached_property
from pathlib import Path

import numpy as np

CACHE_MAGIC = b"BPGR"
CACHE_VERSION = 1

CSR_ATTRS = (
    "u_count", "v_count", "edge_count", "u_indptr", "u_indices", "u_weights",
    "v_indptr", "v_indices", "v_weights", "ws_u", "ws_v",
)


class DataError(ValueError):
    """Malformed input data: bad edge lists, bad cache files, bad labels
    (same role as bipush.DataError, bigraph.py:30-31)."""


def _frozen(a):
    a = np.ascontiguousarray(a)
    a.setflags(write=False)
    return a


class IndexLabels:
    """Read-only label sequence ``prefix + str(i)`` without a Python list."""

    __slots__ = ("prefix", "n")

    def __init__(self, prefix: str, n: int):
        self.prefix = prefix
        self.n = int(n)

    def __len__(self):
        return self.n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(self.n))]
        i = int(i)
        if i < 0:
            i += self.n
        if not 0 <= i < self.n:
            raise IndexError(i)
        return f"{self.prefix}{i}"

    def __iter__(self):
        p = self.prefix
        return (f"{p}{i}" for i in range(self.n))

    def index_of(self, label):
        if isinstance(label, str) and label.startswith(self.prefix):
            tail = label[len(self.prefix):]
            if tail.isdigit() and (tail == "0" or not tail.startswith("0")):
                i = int(tail)
                if i < self.n:
                    return i
        return None


class BipartiteGraph:
    """Immutable weighted bipartite graph in CSR form for both sides.

    Same constructor, validation order and error messages as the reference
    (bigraph.py:53-111).
    """

    def __init__(self, u_labels, v_labels, edge_u, edge_v, edge_w, *, device: int | None = None):
        """``device``: build the canonical CSR arrays on that CUDA device
        (bh_csr_build: two radix sorts of the packed pair keys) instead of with
        host sorts; the arrays and ws sums are bit-identical either way."""
        if not isinstance(u_labels, IndexLabels):
            u_labels = list(u_labels)
        if not isinstance(v_labels, IndexLabels):
            v_labels = list(v_labels)
        eu = np.asarray(edge_u, dtype=np.int64)
        ev = np.asarray(edge_v, dtype=np.int64)
        ew = np.asarray(edge_w, dtype=np.float64)
        if eu.size == 0:
            raise DataError("empty graph: at least one edge is required")
        if not (eu.size == ev.size == ew.size):
            raise DataError("edge arrays have mismatched lengths")
        if not (isinstance(u_labels, IndexLabels) and isinstance(v_labels, IndexLabels)):
            ul, vl = list(u_labels), list(v_labels)
            if len(set(ul)) != len(ul) or len(set(vl)) != len(vl):
                raise DataError("duplicate node label within one side")
            both = set(ul) & set(vl)
            if both:
                raise DataError(f"label appears on both sides: {sorted(both)[0]!r}")
        elif u_labels.prefix == v_labels.prefix:
            raise DataError("label appears on both sides")
        n_u, n_v = len(u_labels), len(v_labels)
        if eu.min() < 0 or eu.max() >= n_u:
            raise DataError("edge endpoint out of range on the U side")
        if ev.min() < 0 or ev.max() >= n_v:
            raise DataError("edge endpoint out of range on the V side")
        if not np.isfinite(ew).all() or (ew <= 0).any():
            raise DataError("edge weights must be positive and finite")

        self.u_count = n_u
        self.v_count = n_v
        self.u_labels = u_labels
        self.v_labels = v_labels

        if device is not None:
            self._build_on_device(eu, ev, ew, int(device))
            return
        # Canonical order: rows sorted by (u, v).  A stable argsort of the
        # unique pair key is the same permutation as the reference's lexsort.
        key = eu * n_v + ev
        order = np.argsort(key, kind="stable")
        eu, ev, ew, key = eu[order], ev[order], ew[order], key[order]
        if key.size > 1 and (key[1:] == key[:-1]).any():
            raise DataError("duplicate edge passed to constructor")
        self.edge_count = int(eu.size)

        self.deg_u = _frozen(np.bincount(eu, minlength=n_u))
        self.deg_v = _frozen(np.bincount(ev, minlength=n_v))
        self._check_isolated()

        self.u_indptr = _frozen(np.concatenate(([0], np.cumsum(self.deg_u))).astype(np.int64))
        self.u_indices = _frozen(ev.astype(np.int32))
        self.u_weights = _frozen(ew)

        vorder = np.argsort(ev * n_u + eu, kind="stable")
        self.v_indptr = _frozen(np.concatenate(([0], np.cumsum(self.deg_v))).astype(np.int64))
        self.v_indices = _frozen(eu[vorder].astype(np.int32))
        self.v_weights = _frozen(ew[vorder])

        # bincount accumulates in canonical edge order -> identical bits to
        # the reference's ws_u / ws_v (bigraph.py:107-108).
        self.ws_u = _frozen(np.bincount(eu, weights=ew, minlength=n_u))
        self.ws_v = _frozen(np.bincount(ev, weights=ew, minlength=n_v))

    def _check_isolated(self):
        if (self.deg_u == 0).any():
            i = int(np.flatnonzero(self.deg_u == 0)[0])
            raise DataError(f"isolated node on U side: {self.u_labels[i]!r}")
        if (self.deg_v == 0).any():
            i = int(np.flatnonzero(self.deg_v == 0)[0])
            raise DataError(f"isolated node on V side: {self.v_labels[i]!r}")

    def _build_on_device(self, eu, ev, ew, device: int):
        from . import _capi

        out = _capi.csr_build(self.u_count, self.v_count, eu, ev, ew, device)
        if out is None:
            raise DataError("duplicate edge passed to constructor")
        self.edge_count = int(eu.size)
        self.deg_u = _frozen(np.diff(out["u_indptr"]))
        self.deg_v = _frozen(np.diff(out["v_indptr"]))
        self._check_isolated()
        for k in ("u_indptr", "u_indices", "u_weights", "v_indptr", "v_indices", "v_weights", "ws_u", "ws_v"):
            setattr(self, k, _frozen(out[k]))

    # -- construction helpers ------------------------------------------------

    @classmethod
    def from_arrays(cls, u_count: int, v_count: int, edge_u, edge_v, edge_w, device: int | None = None):
        """Graph with labels "u{i}" / "v{j}" (the reference synth convention)."""
        return cls(IndexLabels("u", u_count), IndexLabels("v", v_count), edge_u, edge_v, edge_w, device=device)

    @classmethod
    def from_edges(cls, u_labels, v_labels, triples):
        """(u_index, v_index, weight) triples; repeated pairs merge by summing
        weights in first-seen order (bigraph.py:115-130)."""
        merged: dict[tuple[int, int], float] = {}
        for ui, vi, w in triples:
            k = (int(ui), int(vi))
            merged[k] = merged.get(k, 0.0) + float(w)
        if not merged:
            raise DataError("empty graph: at least one edge is required")
        eu = np.fromiter((k[0] for k in merged), dtype=np.int64, count=len(merged))
        ev = np.fromiter((k[1] for k in merged), dtype=np.int64, count=len(merged))
        ew = np.fromiter(merged.values(), dtype=np.float64, count=len(merged))
        return cls(u_labels, v_labels, eu, ev, ew)

    # -- label lookup --------------------------------------------------------

    @cached_property
    def _u_index(self):
        return {lab: i for i, lab in enumerate(self.u_labels)}

    def u_id(self, label) -> int:
        if isinstance(self.u_labels, IndexLabels):
            i = self.u_labels.index_of(label)
            if i is not None:
                return i
            raise DataError(f"unknown U-side label: {label!r}")
        try:
            return self._u_index[label]
        except KeyError:
            raise DataError(f"unknown U-side label: {label!r}") from None

    @cached_property
    def _v_index(self):
        return {lab: i for i, lab in enumerate(self.v_labels)}

    def v_id(self, label) -> int:
        if isinstance(self.v_labels, IndexLabels):
            i = self.v_labels.index_of(label)
            if i is not None:
                return i
            raise DataError(f"unknown V-side label: {label!r}")
        try:
            return self._v_index[label]
        except KeyError:
            raise DataError(f"unknown V-side label: {label!r}") from None

    # -- normalised operators (bigraph.py:148-188), host-side scipy views ------
    # The device store keeps only the two prescaled value arrays (graph_store.cu);
    # these are for host callers that use the reference's operator attributes.

    @cached_property
    def u_step(self):
        """Row-stochastic |U| x |V| CSR: w(u, v) / ws(u)."""
        import scipy.sparse as sp

        data = self.u_weights / np.repeat(self.ws_u, self.deg_u)
        return sp.csr_matrix((data, self.u_indices.astype(np.int64), self.u_indptr), shape=(self.u_count, self.v_count))

    @cached_property
    def v_step(self):
        """Row-stochastic |V| x |U| CSR: w(u, v) / ws(v)."""
        import scipy.sparse as sp

        data = self.v_weights / np.repeat(self.ws_v, self.deg_v)
        return sp.csr_matrix((data, self.v_indices.astype(np.int64), self.v_indptr), shape=(self.v_count, self.u_count))

    @cached_property
    def u_step_t(self):
        return self.u_step.T.tocsr()

    @cached_property
    def v_step_t(self):
        return self.v_step.T.tocsr()

    @cached_property
    def recv_uv(self) -> np.ndarray:
        """Per U-CSR slot: w(u, v) / ws(v)."""
        return _frozen(self.u_weights / self.ws_v[self.u_indices])

    @cached_property
    def recv_vu(self) -> np.ndarray:
        """Per V-CSR slot: w(u, v) / ws(u)."""
        return _frozen(self.v_weights / self.ws_u[self.v_indices])

    # -- serialisation (BPGR v1, bigraph.py:192-251) ---------------------------

    def _label_blob(self, labels) -> bytes:
        enc = [lab.encode("utf-8") for lab in labels]
        out = bytearray()
        for b in enc:
            out += struct.pack("<I", len(b))
            out += b
        return bytes(out)

    def to_bytes(self) -> bytes:
        out = io.BytesIO()
        out.write(CACHE_MAGIC)
        out.write(struct.pack("<I", CACHE_VERSION))
        out.write(struct.pack("<QQQ", self.u_count, self.v_count, self.edge_count))
        out.write(self.u_indptr.astype("<i8").tobytes())
        out.write(self.u_indices.astype("<i4").tobytes())
        out.write(self.u_weights.astype("<f8").tobytes())
        out.write(self._label_blob(self.u_labels))
        out.write(self._label_blob(self.v_labels))
        return out.getvalue()

    @classmethod
    def from_bytes(cls, buf: bytes, device: int | None = None) -> "BipartiteGraph":
        if len(buf) < 4 + 4 + 24 or buf[:4] != CACHE_MAGIC:
            raise DataError("not a graph cache file (bad magic)")
        (version,) = struct.unpack_from("<I", buf, 4)
        if version != CACHE_VERSION:
            raise DataError(f"unsupported graph cache version: {version}")
        u_count, v_count, edge_count = struct.unpack_from("<QQQ", buf, 8)
        off = 32
        try:
            indptr = np.frombuffer(buf, dtype="<i8", count=u_count + 1, offset=off).copy()
            off += 8 * (u_count + 1)
            indices = np.frombuffer(buf, dtype="<i4", count=edge_count, offset=off).copy()
            off += 4 * edge_count
            weights = np.frombuffer(buf, dtype="<f8", count=edge_count, offset=off).copy()
            off += 8 * edge_count
        except ValueError:
            raise DataError("truncated graph cache file") from None
        labels = []
        for _ in range(u_count + v_count):
            if off + 4 > len(buf):
                raise DataError("truncated graph cache label table")
            (n,) = struct.unpack_from("<I", buf, off)
            off += 4
            if off + n > len(buf):
                raise DataError("truncated graph cache label table")
            labels.append(buf[off: off + n].decode("utf-8"))
            off += n
        if off != len(buf):
            raise DataError("trailing bytes after graph cache payload")
        if indptr[0] != 0 or indptr[-1] != edge_count or (np.diff(indptr) < 0).any():
            raise DataError("corrupt adjacency offsets in graph cache")
        eu = np.repeat(np.arange(u_count, dtype=np.int64), np.diff(indptr))
        return cls(labels[:u_count], labels[u_count:], eu, indices.astype(np.int64), weights, device=device)

    def save(self, path) -> None:
        Path(path).write_bytes(self.to_bytes())

    @classmethod
    def load(cls, path, device: int | None = None) -> "BipartiteGraph":
        return cls.from_bytes(Path(path).read_bytes(), device=device)

    @cached_property
    def fingerprint(self) -> str:
        """Hex sha256 of the canonical serialisation (bigraph.py:260-263)."""
        return hashlib.sha256(self.to_bytes()).hexdigest()

    def __repr__(self):
        return f"BipartiteGraph(u={self.u_count}, v={self.v_count}, edges={self.edge_count})"


# -- text edge lists (bigraph.py:272-350) --------------------------------------

def _edge_lines_reference(lines, delimiter, default_weight):
    """The reference's per-line loop restated: labels in first-seen order per
    side, (u, v, w) triples, every error message of bigraph.py:322-344."""
    u_index: dict[str, int] = {}
    v_index: dict[str, int] = {}
    triples: list[tuple[int, int, float]] = []
    for lineno, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        cols = line.split(delimiter)
        if len(cols) == 3:
            try:
                w = float(cols[2])
            except ValueError:
                raise DataError(f"line {lineno}: bad weight {cols[2]!r}") from None
        elif len(cols) == 2:
            if default_weight is None:
                raise DataError(f"line {lineno}: two columns but no default weight configured")
            w = float(default_weight)
        else:
            raise DataError(f"line {lineno}: expected 2 or 3 columns, got {len(cols)}")
        if not np.isfinite(w) or w <= 0:
            raise DataError(f"line {lineno}: weight must be positive, got {w}")
        ul, vl = cols[0], cols[1]
        if ul in v_index:
            raise DataError(f"line {lineno}: label appears on both sides: {ul!r}")
        if vl in u_index:
            raise DataError(f"line {lineno}: label appears on both sides: {vl!r}")
        ui = u_index.setdefault(ul, len(u_index))
        vi = v_index.setdefault(vl, len(v_index))
        triples.append((ui, vi, w))
    if not triples:
        raise DataError("empty graph: no data lines found")
    return list(u_index), list(v_index), triples


def _edge_list_native(data: bytes, delimiter, default_weight):
    """bh_edge_list_parse on the raw bytes: (u_labels, v_labels, eu, ev, ew) with
    repeated pairs already merged, or None when the input needs the Python loop."""
    import ctypes as C

    from . import _capi

    L = _capi.lib()
    h = C.c_void_p()
    err = C.c_int64(0)
    sep = None if delimiter is None else delimiter.encode("ascii")
    rc = L.bh_edge_list_parse(data, len(data), sep, 0 if sep is None else len(sep),
                              int(default_weight is not None), float(default_weight or 0.0),
                              C.byref(h), C.byref(err))
    if rc == _capi.BH_EFALLBACK:
        return None
    _capi.check(rc)
    try:
        n = [C.c_int64() for _ in range(5)]
        _capi.check(L.bh_edge_list_sizes(h, *[C.byref(x) for x in n]))
        n_u, n_v, bu, bv, n_e = (x.value for x in n)
        ublob, vblob = C.create_string_buffer(max(1, bu)), C.create_string_buffer(max(1, bv))
        uend, vend = np.empty(n_u, np.int64), np.empty(n_v, np.int64)
        eu, ev, ew = np.empty(n_e, np.int64), np.empty(n_e, np.int64), np.empty(n_e, np.float64)
        _capi.check(L.bh_edge_list_export(h, ublob, _capi.ptr(uend), vblob, _capi.ptr(vend),
                                          _capi.ptr(eu), _capi.ptr(ev), _capi.ptr(ew)))
    finally:
        L.bh_edge_list_free(h)

    def labels(blob, ends):
        raw = blob.raw[: int(ends[-1]) if ends.size else 0].decode("ascii")
        starts = np.concatenate(([0], ends[:-1])).tolist()
        return [raw[a:b] for a, b in zip(starts, ends.tolist())]

    return labels(ublob, uend), labels(vblob, vend), eu, ev, ew


def load_edge_list(source, delimiter=None, default_weight=None, device: int | None = None) -> "BipartiteGraph":
    """Text edge list -> graph (reference bigraph.py:272-350, same arguments,
    same errors).  ASCII input with plain decimal weights is parsed by the
    native parser (bh_edge_list_parse); anything else, and every malformed
    file, goes through the reference-semantics line loop.  ``device`` builds
    the CSR on that GPU (see BipartiteGraph)."""
    if default_weight is not None and not (np.isfinite(default_weight) and default_weight > 0):
        raise DataError("default_weight must be positive and finite")
    if isinstance(source, (str, Path)):
        data = Path(source).read_bytes()
        text_lines = lambda: open(source, "r", encoding="utf-8")  # noqa: E731
    elif isinstance(source, (io.RawIOBase, io.BufferedIOBase)) or (
            hasattr(source, "read") and isinstance(source.read(0), bytes)):
        data = source.read()
        text_lines = lambda: io.TextIOWrapper(io.BytesIO(data), encoding="utf-8")  # noqa: E731
    else:
        text = source.read()
        data = text.encode("utf-8", "surrogatepass")
        text_lines = lambda: io.StringIO(text, newline=None)  # noqa: E731
    fast = None
    if delimiter is None or (isinstance(delimiter, str) and delimiter and delimiter.isascii()):
        fast = _edge_list_native(data, delimiter, default_weight)
    if fast is not None:
        u_labels, v_labels, eu, ev, ew = fast
        return BipartiteGraph(u_labels, v_labels, eu, ev, ew, device=device)
    with text_lines() as fh:
        u_labels, v_labels, triples = _edge_lines_reference(fh, delimiter, default_weight)
    merged: dict[tuple[int, int], float] = {}
    for ui, vi, w in triples:
        merged[(ui, vi)] = merged.get((ui, vi), 0.0) + w
    eu = np.fromiter((k[0] for k in merged), dtype=np.int64, count=len(merged))
    ev = np.fromiter((k[1] for k in merged), dtype=np.int64, count=len(merged))
    ew = np.fromiter(merged.values(), dtype=np.float64, count=len(merged))
    return BipartiteGraph(u_labels, v_labels, eu, ev, ew, device=device)
