"""Python mirror of the reference's counting interface over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj:
  TemporalGraph / parse_edge_list / generate_random_graph   graph.hpp:25-82
  GraphContext                                               indexes.hpp:95-105
  count_star_pair_at_center / count_star_pair                star_engine.hpp:35-46
  count_triangles_at_center / count_triangles                triangle_engine.hpp:20-36
  RunConfig / auto_degree_threshold / run_parallel           executor.hpp:36-74
  merge_census / MotifCensus / signatures                    motifs.hpp:136-206
Every count is computed by libtmotif_b200.so on the GPU; there is no CPU
counting path, and a missing library or device raises instead of falling back.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# TM_LIB overrides the library path (A/B runs of two builds of the same API)
LIB_PATH = os.environ.get("TM_LIB") or os.path.join(HERE, "libtmotif_b200.so")

TM_OK = 0
TM_ERR_INVALID = 1
TM_ERR_PARSE = 2
TM_ERR_OVERFLOW = 3
TM_ERR_CONFIG = 4
TM_ERR_CONSISTENCY = 10
TM_ERR_CUDA = 8
TM_ERR_LIMIT = 9


# ---- error types (types.hpp:35-63) -----------------------------------------
class ParseError(RuntimeError):
    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


class ConfigError(RuntimeError):
    pass


class CounterOverflowError(OverflowError):
    pass


class ConsistencyError(ArithmeticError):
    pass


class ClassificationError(ValueError):
    pass


class DeviceError(RuntimeError):
    pass


def _raise(rc: int, lib) -> None:
    if rc == TM_OK:
        return
    msg = lib.tm_last_error().decode() if lib is not None else ""
    if rc == TM_ERR_INVALID:
        raise ValueError(msg)
    if rc == TM_ERR_PARSE:
        line = int(lib.tm_parse_error_line())
        prefix = f"line {line}: "
        raise ParseError(line, msg[len(prefix):] if msg.startswith(prefix) else msg)
    if rc == TM_ERR_OVERFLOW:
        raise CounterOverflowError(msg or "motif counter overflow")
    if rc == TM_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == TM_ERR_CONSISTENCY:
        raise ConsistencyError(msg)
    if rc == TM_ERR_LIMIT:
        raise MemoryError(msg)
    raise DeviceError(msg or f"tmotif error {rc}")


# ---- library -----------------------------------------------------------------
class _Counters(C.Structure):
    _fields_ = [("star", C.c_uint64 * 24), ("pair", C.c_uint64 * 8), ("tri", C.c_uint64 * 24)]


class _RunConfig(C.Structure):
    _fields_ = [("delta", C.c_int64), ("workers", C.c_uint32), ("degree_threshold", C.c_int64),
                ("triangle_mode", C.c_int32), ("motifs", C.c_uint32), ("shard_target", C.c_uint64),
                ("center_begin", C.c_uint32), ("center_end", C.c_uint32),
                ("has_first_edge_t_end", C.c_int32), ("first_edge_t_end", C.c_int64)]


class _Timings(C.Structure):
    _fields_ = [("ingest_ms", C.c_double), ("index_ms", C.c_double), ("star_pair_ms", C.c_double),
                ("triangle_ms", C.c_double), ("merge_ms", C.c_double)]


_lib = None
VP = C.c_void_p


def lib():
    """Load libtmotif_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.tm_graph_build.argtypes = [VP, VP, VP, C.c_uint64, C.c_uint64, C.c_int, VP, C.POINTER(VP)]
    L.tm_graph_free.argtypes = [VP]
    L.tm_graph_node_count.argtypes = [VP]
    L.tm_graph_node_count.restype = C.c_uint64
    L.tm_graph_edge_count.argtypes = [VP]
    L.tm_graph_edge_count.restype = C.c_uint64
    L.tm_graph_stream.argtypes = [VP]
    L.tm_graph_stream.restype = VP
    L.tm_graph_degrees.argtypes = [VP, VP]
    L.tm_graph_sequence.argtypes = [VP, C.c_uint32, VP, VP, VP, VP, C.c_uint64, C.POINTER(C.c_uint64)]
    L.tm_pair_window.argtypes = [VP, C.c_uint32, C.c_uint32, C.c_int64, C.c_int64, VP, VP, VP,
                                 C.c_uint64, C.POINTER(C.c_uint64)]
    L.tm_auto_degree_threshold.argtypes = [VP, C.POINTER(C.c_uint64)]
    L.tm_count_star_pair.argtypes = [VP, C.c_int64, VP, VP]
    L.tm_count_triangles.argtypes = [VP, C.c_int64, C.c_int, VP]
    L.tm_count_star_pair_items.argtypes = [VP, C.c_int64, C.c_uint64, VP, VP, VP, VP, VP]
    L.tm_count_triangles_items.argtypes = [VP, C.c_int64, C.c_uint64, VP, VP, VP, VP, VP]
    L.tm_run_parallel.argtypes = [VP, C.POINTER(_RunConfig), C.POINTER(_Counters), VP,
                                  C.POINTER(_Timings)]
    L.tm_count_edges.argtypes = [VP, VP, VP, C.c_uint64, C.c_uint64, C.c_int, VP,
                                 C.POINTER(_RunConfig), C.POINTER(_Counters), VP, C.POINTER(_Timings)]
    L.tm_parse_edge_list.argtypes = [VP, C.c_uint64, C.c_int, C.c_int, VP, C.POINTER(VP)]
    L.tm_edge_list_info.argtypes = [VP, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_uint64)]
    L.tm_edge_list_device_arrays.argtypes = [VP, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP)]
    L.tm_edge_list_copy.argtypes = [VP, VP, VP, VP, VP]
    L.tm_parse_error_line.restype = C.c_uint64
    L.tm_edge_list_free.argtypes = [VP]
    L.tm_write_edge_list.argtypes = [VP, VP, VP, C.c_uint64, C.c_int, VP, VP, C.c_int, C.POINTER(C.c_uint64)]
    L.tm_count_edges_async.argtypes = [VP, VP, VP, C.c_uint64, C.c_uint64, VP, C.POINTER(_RunConfig),
                                       C.POINTER(C.c_uint64)]
    L.tm_count_edges_wait.argtypes = [C.c_uint64, C.POINTER(_Counters), VP]
    L.tm_async_h2d_bytes.argtypes = [C.POINTER(C.c_uint64)]
    L.tm_count_edges_time_slice.argtypes = [VP, VP, VP, C.c_uint64, C.c_uint64, C.c_int, VP,
                                            C.POINTER(_RunConfig), C.c_int, C.c_int64, C.c_int, C.c_int64,
                                            C.POINTER(_Counters), C.POINTER(_Timings)]
    L.tm_partition_centers.argtypes = [VP, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint32)]
    L.tm_merge_census.argtypes = [VP, VP, VP, C.c_int, VP]
    L.tm_signature.argtypes = [C.c_int, C.c_char_p]
    L.tm_cell_signature.argtypes = [C.c_int, C.c_int]
    L.tm_signature_label.argtypes = [C.c_int, C.c_char_p]
    L.tm_generate_random_graph.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_uint64, VP, VP, VP]
    L.tm_run_stats.argtypes = [VP, VP]
    L.tm_last_error.restype = C.c_char_p
    L.tm_debug_acc_bias.argtypes = [C.c_uint64]
    L.tm_kernel_launches.restype = C.c_uint64
    L.tm_kernel_timing_enable.argtypes = [C.c_int]
    L.tm_kernel_timing_get.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    _lib = L
    return L


def kernel_launches() -> int:
    return int(lib().tm_kernel_launches())


def kernel_timing(enable: Optional[bool] = None, reset: bool = False):
    L = lib()
    if reset:
        L.tm_kernel_timing_reset()
    if enable is not None:
        L.tm_kernel_timing_enable(1 if enable else 0)


def kernel_time(name: str) -> Tuple[float, int]:
    ms, n = C.c_double(0), C.c_uint64(0)
    lib().tm_kernel_timing_get(name.encode(), C.byref(ms), C.byref(n))
    return ms.value, n.value


# ---- taxonomy (motifs.hpp) -------------------------------------------------------
class Direction(enum.IntEnum):
    outward = 0
    inward = 1


class StarType(enum.IntEnum):
    isolated_first = 0
    isolated_second = 1
    isolated_third = 2


class TriangleType(enum.IntEnum):
    closing_first = 0
    closing_middle = 1
    closing_last = 2


class TriangleMode(enum.IntEnum):
    count_all = 0
    removal = 1


def triangle_mode_name(mode: TriangleMode) -> str:
    return "countall" if mode == TriangleMode.count_all else "removal"


def complement(d: Direction) -> Direction:
    return Direction(1 - int(d))


_SIGS: Optional[List[str]] = None


def all_signatures() -> List[str]:
    """The 36 valid signatures in lexicographic order (motifs.cpp:196)."""
    global _SIGS
    if _SIGS is None:
        L = lib()
        buf = C.create_string_buffer(9)
        out = []
        for k in range(36):
            L.tm_signature(k, buf)
            out.append(buf.value.decode())
        _SIGS = out
    return list(_SIGS)


def signature_index(sig: str) -> Optional[int]:
    try:
        return all_signatures().index(sig)
    except ValueError:
        return None


def _check_sig(s: str) -> str:
    if len(s) != 8 or s[2] != "|" or s[5] != "|" or any(c not in "123" for c in s[:2] + s[3:5] + s[6:]):
        raise ClassificationError("malformed signature: " + s)
    return s


def canonical_signature(edges: Sequence[Tuple[int, int]]) -> str:
    """canonical_signature (motifs.cpp:49-77): first-appearance relabeling."""
    seen: List[int] = []
    labels = []
    for a, b in edges:
        if a == b:
            raise ClassificationError("self-loop edge in triple")
        for node in (a, b):
            if node not in seen:
                if len(seen) == 3:
                    raise ClassificationError("edge triple spans more than 3 nodes")
                seen.append(node)
            labels.append(seen.index(node) + 1)
    return "|".join(f"{labels[2 * k]}{labels[2 * k + 1]}" for k in range(3))


def signature_category(sig: str) -> str:
    s = _check_sig(sig)
    labs = [int(c) for c in s if c != "|"]
    if max(labs) == 2:
        return "pair"
    pairs = {tuple(sorted((labs[2 * k], labs[2 * k + 1]))) for k in range(3)}
    return "triangle" if len(pairs) == 3 else "star"


def cell_signature(kind: str, cell: int) -> str:
    k = {"star": 0, "pair": 1, "tri": 2}[kind]
    return all_signatures()[lib().tm_cell_signature(k, cell)]


def star_cell_signature(t, d1, d2, d3) -> str:
    return cell_signature("star", StarCounter.index(t, d1, d2, d3))


def pair_cell_signature(d1, d2, d3) -> str:
    return cell_signature("pair", PairCounter.index(d1, d2, d3))


def tri_cell_signature(t, di, dj, dk) -> str:
    return cell_signature("tri", TriCounter.index(t, di, dj, dk))


def label_for_signature(sig: str) -> str:
    idx = signature_index(sig)
    if idx is None:
        raise ClassificationError("unknown signature: " + sig)
    buf = C.create_string_buffer(16)
    lib().tm_signature_label(idx, buf)
    return buf.value.decode()


class _Cells:
    cell_count = 0

    def __init__(self, cells=None):
        self.cells = np.zeros(self.cell_count, np.uint64) if cells is None else \
            np.array(cells, dtype=np.uint64).reshape(self.cell_count)

    def __eq__(self, other):
        return isinstance(other, type(self)) and bool((self.cells == other.cells).all())

    def add(self, other):
        s = self.cells.astype(object) + other.cells.astype(object)
        if any(v >= 2 ** 64 for v in s):
            raise CounterOverflowError("motif counter overflow")
        self.cells = np.array(s, dtype=np.uint64)

    def __repr__(self):
        return f"{type(self).__name__}({self.cells.tolist()})"


class StarCounter(_Cells):
    cell_count = 24

    @staticmethod
    def index(t, d1, d2, d3):
        return ((int(t) * 2 + int(d1)) * 2 + int(d2)) * 2 + int(d3)

    def at(self, t, d1, d2, d3):
        return int(self.cells[self.index(t, d1, d2, d3)])


class PairCounter(_Cells):
    cell_count = 8

    @staticmethod
    def index(d1, d2, d3):
        return (int(d1) * 2 + int(d2)) * 2 + int(d3)

    def at(self, d1, d2, d3):
        return int(self.cells[self.index(d1, d2, d3)])


class TriCounter(_Cells):
    cell_count = 24

    @staticmethod
    def index(t, di, dj, dk):
        return ((int(t) * 2 + int(di)) * 2 + int(dj)) * 2 + int(dk)

    def at(self, t, di, dj, dk):
        return int(self.cells[self.index(t, di, dj, dk)])


@dataclass
class CenterStarResult:
    star: StarCounter = field(default_factory=StarCounter)
    pair: PairCounter = field(default_factory=PairCounter)

    def add(self, other: "CenterStarResult"):
        self.star.add(other.star)
        self.pair.add(other.pair)


@dataclass
class CensusMeta:
    input: str = ""
    edge_count: int = 0
    triangle_mode: str = ""
    workers: int = 0


class MotifCensus:
    """signature -> count over the 36-signature domain (motifs.hpp:168-190)."""

    def __init__(self, counts=None, delta: int = 0):
        self.counts = np.zeros(36, np.uint64) if counts is None else np.array(counts, np.uint64)
        self.delta = delta
        self.meta = CensusMeta()

    def count(self, sig: str) -> int:
        idx = signature_index(sig)
        if idx is None:
            raise ClassificationError("unknown signature: " + sig)
        return int(self.counts[idx])

    def count_at(self, k: int) -> int:
        return int(self.counts[k])

    def total(self) -> int:
        """checked sum (motifs.cpp:239-243)."""
        s = int(sum(int(c) for c in self.counts))
        if s >= 1 << 64:
            raise CounterOverflowError("motif counter overflow")
        return s

    def same_counts(self, other: "MotifCensus") -> bool:
        return bool((self.counts == other.counts).all())

    def as_dict(self) -> Dict[str, int]:
        return {s: int(c) for s, c in zip(all_signatures(), self.counts)}


def merge_census(star: StarCounter, pair: PairCounter, tri: TriCounter,
                 tri_mode: TriangleMode = TriangleMode.count_all) -> MotifCensus:
    """merge_census (motifs.cpp:233-281) via the C-ABI."""
    s = np.ascontiguousarray(star.cells, np.uint64)
    p = np.ascontiguousarray(pair.cells, np.uint64)
    t = np.ascontiguousarray(tri.cells, np.uint64)
    out = np.zeros(36, np.uint64)
    L = lib()
    _raise(L.tm_merge_census(s.ctypes.data, p.ctypes.data, t.ctypes.data, int(tri_mode),
                             out.ctypes.data), L)
    return MotifCensus(out)


# ---- graph (graph.hpp) -------------------------------------------------------------
class TemporalGraph:
    """Edge arrays in ingestion order (ordinal = index) plus the id map.

    TemporalGraph::build (graph.cpp:13-44) validates and sorts; here the
    sort happens on the GPU inside GraphContext.build, and `edges()` (the
    (t, ordinal)-sorted view) is provided for tests only.
    """

    def __init__(self, node_ids: Sequence[str], src, dst, t, dropped_self_loops: int = 0):
        self.node_ids = list(node_ids)
        self._index = {}
        for u, name in enumerate(self.node_ids):
            if name in self._index:
                raise ValueError("duplicate node id: " + name)
            self._index[name] = u
        self.src = np.ascontiguousarray(src, np.uint32)
        self.dst = np.ascontiguousarray(dst, np.uint32)
        self.t = np.ascontiguousarray(t, np.int64)
        n = len(self.node_ids)
        if len(self.src) and ((self.src == self.dst).any()):
            i = int(np.nonzero(self.src == self.dst)[0][0])
            raise ValueError(f"self-loop edge at ingestion index {i}")
        if len(self.src) and (int(self.src.max()) >= n or int(self.dst.max()) >= n):
            raise ValueError("edge endpoint out of range")
        self._dropped = dropped_self_loops

    @classmethod
    def from_arrays(cls, n: int, src, dst, t) -> "TemporalGraph":
        g = cls.__new__(cls)
        g.node_ids = None
        g._index = None
        g._n = int(n)
        g.src = np.ascontiguousarray(src, np.uint32)
        g.dst = np.ascontiguousarray(dst, np.uint32)
        g.t = np.ascontiguousarray(t, np.int64)
        g._dropped = 0
        return g

    def node_count(self) -> int:
        return len(self.node_ids) if self.node_ids is not None else self._n

    def edge_count(self) -> int:
        return len(self.src)

    def node_id(self, u: int) -> str:
        return self.node_ids[u] if self.node_ids is not None else str(u)

    def find_node(self, name: str) -> Optional[int]:
        if self._index is None:
            try:
                u = int(name)
            except ValueError:
                return None
            return u if 0 <= u < self._n else None
        return self._index.get(name)

    def dropped_self_loops(self) -> int:
        return self._dropped

    def degrees(self) -> np.ndarray:
        n = self.node_count()
        return (np.bincount(self.src, minlength=n) + np.bincount(self.dst, minlength=n)).astype(np.uint64)

    def edges(self):
        """(t, ordinal)-sorted (src, dst, t, ordinal) arrays."""
        order = np.lexsort((np.arange(len(self.t)), self.t))
        return self.src[order], self.dst[order], self.t[order], order.astype(np.uint64)


def parse_edge_list(text: str, drop_self_loops: bool = True) -> TemporalGraph:
    """parse_edge_list (graph.cpp:77-124): 'SRC DST T' lines, '#' comments."""
    node_ids: List[str] = []
    index: Dict[str, int] = {}
    src, dst, ts = [], [], []
    dropped = 0

    def intern(tok):
        if tok in index:
            return index[tok]
        index[tok] = len(node_ids)
        node_ids.append(tok)
        return index[tok]

    for line_no, line in enumerate(text.split("\n"), start=1):
        if line.endswith("\r"):
            line = line[:-1]
        f = line.split()
        if not f or f[0].startswith("#"):
            continue
        if len(f) < 3:
            raise ParseError(line_no, "expected 3 tokens: SRC DST T")
        tok = f[2]
        try:
            # std::from_chars<int64_t>: optional '-', ASCII digits, whole field
            body = tok[1:] if tok.startswith("-") else tok
            if not body or any(c not in "0123456789" for c in body):
                raise ValueError
            tv = int(tok)
            if not -(2 ** 63) <= tv < 2 ** 63:
                raise ValueError
        except ValueError:
            raise ParseError(line_no, f"malformed timestamp '{tok}'")
        if f[0] == f[1]:
            if not drop_self_loops:
                raise ParseError(line_no, f"self-loop edge '{f[0]}'")
            dropped += 1
            continue
        s = intern(f[0])
        d = intern(f[1])
        src.append(s)
        dst.append(d)
        ts.append(tv)
    return TemporalGraph(node_ids, np.array(src, np.uint32), np.array(dst, np.uint32),
                         np.array(ts, np.int64), dropped)


class EdgeList:
    """A parsed edge list resident on the GPU (tm_parse_edge_list): the
    reference's parse_edge_list output -- ingestion-order edges, dense node
    ids by first appearance, dropped self-loop tally -- with the edge arrays
    left in device memory for GraphContext.build_device / count_edges_device."""

    def __init__(self, handle, lib_):
        self._h = handle
        self._L = lib_
        n, m, dr, ib = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _raise(lib_.tm_edge_list_info(handle, C.byref(n), C.byref(m), C.byref(dr), C.byref(ib)), lib_)
        self.n, self.m, self.dropped_self_loops, self._id_bytes = n.value, m.value, dr.value, ib.value

    def device_arrays(self) -> Tuple[int, int, int]:
        s, d, t = VP(), VP(), VP()
        _raise(self._L.tm_edge_list_device_arrays(self._h, C.byref(s), C.byref(d), C.byref(t)), self._L)
        return s.value or 0, d.value or 0, t.value or 0

    def to_graph(self) -> TemporalGraph:
        src = np.zeros(self.m, np.uint32)
        dst = np.zeros(self.m, np.uint32)
        t = np.zeros(self.m, np.int64)
        ids = C.create_string_buffer(self._id_bytes + 1)
        _raise(self._L.tm_edge_list_copy(self._h, src.ctypes.data, dst.ctypes.data, t.ctypes.data, ids), self._L)
        names = ids.raw[:self._id_bytes].decode("utf-8", "surrogateescape").split("\n") if self.n else []
        return TemporalGraph(names, src, dst, t, self.dropped_self_loops)

    def close(self):
        if self._h:
            self._L.tm_edge_list_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def parse_edge_list_gpu(text, drop_self_loops: bool = True, stream: Optional[int] = None) -> EdgeList:
    """parse_edge_list (graph.cpp:73-116) on the GPU; `text` is str or bytes
    (host), or (pointer, nbytes[, is_device=True]).  Raises ParseError like
    the reference."""
    L = lib()
    h = VP()
    if isinstance(text, tuple):
        ptr, nbytes = text[0], text[1]
        on_dev = text[2] if len(text) > 2 else True
        _raise(L.tm_parse_edge_list(ptr, nbytes, int(on_dev), int(drop_self_loops), stream, C.byref(h)), L)
    else:
        buf = text.encode("utf-8", "surrogateescape") if isinstance(text, str) else bytes(text)
        _raise(L.tm_parse_edge_list(buf, len(buf), 0, int(drop_self_loops), stream, C.byref(h)), L)
    return EdgeList(h, L)


def write_edge_list_gpu(src, dst, t, stream: Optional[int] = None) -> bytes:
    """write_edge_list (graph.cpp:170) on the GPU for decimal node ids."""
    L = lib()
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    t = np.ascontiguousarray(t, np.int64)
    nb = C.c_uint64(0)
    _raise(L.tm_write_edge_list(src.ctypes.data, dst.ctypes.data, t.ctypes.data, len(src), 0, stream, None, 0,
                                C.byref(nb)), L)
    buf = C.create_string_buffer(nb.value + 1)
    _raise(L.tm_write_edge_list(src.ctypes.data, dst.ctypes.data, t.ctypes.data, len(src), 0, stream, buf, 0,
                                C.byref(nb)), L)
    return buf.raw[:nb.value]


def write_edge_list_device(n_edges: int, src_ptr: int, dst_ptr: int, t_ptr: int, out_ptr: Optional[int] = None,
                           stream: Optional[int] = None) -> int:
    """Device-to-device write_edge_list: returns the byte count; writes into
    out_ptr (device) when given."""
    L = lib()
    nb = C.c_uint64(0)
    _raise(L.tm_write_edge_list(src_ptr, dst_ptr, t_ptr, n_edges, 1, stream, out_ptr, 1, C.byref(nb)), L)
    return nb.value


def load_edge_list(path: str, drop_self_loops: bool = True) -> TemporalGraph:
    with open(path, "r", encoding="utf-8") as f:
        return parse_edge_list(f.read(), drop_self_loops)


def generate_random_graph(nodes: int, edges: int, t_max: int, seed: int) -> TemporalGraph:
    """generate_random_graph (graph.cpp:140-168), bit-identical output."""
    src = np.zeros(edges, np.uint32)
    dst = np.zeros(edges, np.uint32)
    t = np.zeros(edges, np.int64)
    L = lib()
    rc = L.tm_generate_random_graph(nodes, edges, t_max, seed, src.ctypes.data, dst.ctypes.data,
                                    t.ctypes.data)
    if rc:
        raise ValueError(L.tm_last_error().decode())
    return TemporalGraph([str(u) for u in range(nodes)], src, dst, t)


def write_edge_list(graph: TemporalGraph) -> str:
    s, d, t, _ = graph.edges()
    return "".join(f"{graph.node_id(int(a))} {graph.node_id(int(b))} {int(c)}\n" for a, b, c in zip(s, d, t))


# ---- device context (indexes.hpp:95-105) -------------------------------------------
@dataclass
class IncidentEdge:
    t: int
    ordinal: int
    other: int
    dir: Direction


class GraphContext:
    """Device-resident graph + indexes.  Build with GraphContext.build(graph)."""

    def __init__(self, graph: TemporalGraph, handle, lib_):
        self.graph = graph
        self._h = handle
        self._lib = lib_

    @classmethod
    def build(cls, graph: TemporalGraph, stream: Optional[int] = None) -> "GraphContext":
        L = lib()
        h = VP()
        rc = L.tm_graph_build(graph.src.ctypes.data, graph.dst.ctypes.data, graph.t.ctypes.data,
                              graph.edge_count(), graph.node_count(), 0, stream, C.byref(h))
        _raise(rc, L)
        return cls(graph, h, L)

    @classmethod
    def build_device(cls, n: int, src_ptr: int, dst_ptr: int, t_ptr: int, m: int,
                     stream: Optional[int] = None) -> "GraphContext":
        L = lib()
        h = VP()
        _raise(L.tm_graph_build(src_ptr, dst_ptr, t_ptr, m, n, 1, stream, C.byref(h)), L)
        return cls(None, h, L)

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            self._lib.tm_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def node_count(self) -> int:
        return int(self._lib.tm_graph_node_count(self._h))

    def edge_count(self) -> int:
        return int(self._lib.tm_graph_edge_count(self._h))

    def degrees(self) -> np.ndarray:
        out = np.zeros(self.node_count(), np.uint64)
        _raise(self._lib.tm_graph_degrees(self._h, out.ctypes.data), self._lib)
        return out

    def degree(self, u: int) -> int:
        n = C.c_uint64(0)
        self._lib.tm_graph_sequence(self._h, u, None, None, None, None, 0, C.byref(n))
        return int(n.value)

    def sequence(self, u: int) -> List[IncidentEdge]:
        s = self.degree(u)
        t = np.zeros(max(s, 1), np.int64); o = np.zeros(max(s, 1), np.uint64)
        x = np.zeros(max(s, 1), np.uint32); d = np.zeros(max(s, 1), np.uint8)
        n = C.c_uint64(0)
        _raise(self._lib.tm_graph_sequence(self._h, u, t.ctypes.data, o.ctypes.data, x.ctypes.data,
                                           d.ctypes.data, s, C.byref(n)), self._lib)
        return [IncidentEdge(int(t[k]), int(o[k]), int(x[k]), Direction(int(d[k]))) for k in range(s)]

    def edges_in_window(self, v: int, w: int, lo: int, hi: int):
        """PairEdgeIndex::edges_in_window: [(t, ordinal, dir_rel_v)]."""
        cap = self.edge_count() + 1
        t = np.zeros(cap, np.int64); o = np.zeros(cap, np.uint64); d = np.zeros(cap, np.uint8)
        n = C.c_uint64(0)
        _raise(self._lib.tm_pair_window(self._h, v, w, lo, hi, t.ctypes.data, o.ctypes.data,
                                        d.ctypes.data, cap, C.byref(n)), self._lib)
        k = int(n.value)
        return [(int(t[i]), int(o[i]), Direction(int(d[i]))) for i in range(k)]

    def run_stats(self) -> Dict[str, int]:
        """Work counters of the last counting run on this graph."""
        out = np.zeros(8, np.uint64)
        _raise(self._lib.tm_run_stats(self._h, out.ctypes.data), self._lib)
        keys = ["star_first_candidates", "star_third_candidates", "short_wedges", "long_first_edges",
                "long_wedges", "long_group_lookups"]
        stats = {k: int(v) for k, v in zip(keys, out)}
        if out[6] or out[7]:  # instrumented builds only (-DTM_TRI_STATS)
            stats["long_empty_lookups"] = int(out[6])
            stats["long_iterations"] = int(out[7]) & 0xFFFFFFFF
            stats["long_iterations_with_lookup"] = int(out[7]) >> 32
        return stats

    def partition(self, world: int, rank: int) -> Tuple[int, int]:
        b, e = C.c_uint32(0), C.c_uint32(0)
        _raise(self._lib.tm_partition_centers(self._h, world, rank, C.byref(b), C.byref(e)), self._lib)
        return int(b.value), int(e.value)


def full_star_range(s: int) -> Tuple[int, int]:
    return (0, s - 2 if s >= 3 else 0)


def full_triangle_range(s: int) -> Tuple[int, int]:
    return (0, s - 1 if s >= 2 else 0)


def _items(nodes, ranges):
    n = np.ascontiguousarray(nodes, np.uint32)
    b = np.ascontiguousarray([r[0] for r in ranges], np.uint64)
    e = np.ascontiguousarray([r[1] for r in ranges], np.uint64)
    return n, b, e


def count_star_pair_items(ctx: GraphContext, delta: int, nodes, ranges) -> List[CenterStarResult]:
    n, b, e = _items(nodes, ranges)
    k = len(n)
    st = np.zeros(max(k, 1) * 24, np.uint64); pr = np.zeros(max(k, 1) * 8, np.uint64)
    if k:
        _raise(ctx._lib.tm_count_star_pair_items(ctx._h, delta, k, n.ctypes.data, b.ctypes.data,
                                                 e.ctypes.data, st.ctypes.data, pr.ctypes.data), ctx._lib)
    return [CenterStarResult(StarCounter(st[i * 24:(i + 1) * 24]), PairCounter(pr[i * 8:(i + 1) * 8]))
            for i in range(k)]


def count_star_pair_at_center(ctx: GraphContext, u: int, delta: int,
                              first_edges: Tuple[int, int]) -> CenterStarResult:
    """count_star_pair_at_center (star_engine.cpp:64)."""
    return count_star_pair_items(ctx, delta, [u], [first_edges])[0]


def count_star_pair(ctx: GraphContext, delta: int) -> CenterStarResult:
    """count_star_pair (star_engine.cpp:129)."""
    st = np.zeros(24, np.uint64); pr = np.zeros(8, np.uint64)
    _raise(ctx._lib.tm_count_star_pair(ctx._h, delta, st.ctypes.data, pr.ctypes.data), ctx._lib)
    return CenterStarResult(StarCounter(st), PairCounter(pr))


def count_triangles_items(ctx: GraphContext, delta: int, nodes, ranges, live=None) -> List[TriCounter]:
    n, b, e = _items(nodes, ranges)
    k = len(n)
    out = np.zeros(max(k, 1) * 24, np.uint64)
    lv = None if live is None else np.ascontiguousarray(live, np.uint8)
    if k:
        _raise(ctx._lib.tm_count_triangles_items(ctx._h, delta, k, n.ctypes.data, b.ctypes.data,
                                                 e.ctypes.data, lv.ctypes.data if lv is not None else None,
                                                 out.ctypes.data), ctx._lib)
    return [TriCounter(out[i * 24:(i + 1) * 24]) for i in range(k)]


def count_triangles_at_center(ctx: GraphContext, u: int, delta: int, first_edges: Tuple[int, int],
                              live=None) -> TriCounter:
    """count_triangles_at_center (triangle_engine.cpp:20)."""
    return count_triangles_items(ctx, delta, [u], [first_edges], live)[0]


def count_triangles(ctx: GraphContext, delta: int, mode: TriangleMode = TriangleMode.count_all) -> TriCounter:
    """count_triangles (triangle_engine.cpp:64)."""
    out = np.zeros(24, np.uint64)
    _raise(ctx._lib.tm_count_triangles(ctx._h, delta, int(mode), out.ctypes.data), ctx._lib)
    return TriCounter(out)


# ---- executor (executor.hpp) ---------------------------------------------------------
@dataclass
class MotifFilter:
    star: bool = True
    pair: bool = True
    triangle: bool = True

    def mask(self) -> int:
        return (1 if self.star else 0) | (2 if self.pair else 0) | (4 if self.triangle else 0)


NO_SHARDING = 2 ** 63 - 1


@dataclass
class RunConfig:
    delta: int = 0
    workers: int = 1
    degree_threshold: Optional[int] = None  # None: auto top-20 rule
    triangle_mode: TriangleMode = TriangleMode.count_all
    motifs: MotifFilter = field(default_factory=MotifFilter)
    shard_target: int = 4096
    light_batch: int = 64
    # time-slice partition: count only instances whose earliest edge has t < this
    first_edge_t_end: Optional[int] = None

    def to_c(self, center_begin: int = 0, center_end: int = 0) -> _RunConfig:
        thr = -1 if self.degree_threshold is None else min(int(self.degree_threshold), NO_SHARDING)
        m = self.motifs.mask()  # 0 = the empty filter: an all-zero census (executor.cpp:28-29)
        has_t = 0 if self.first_edge_t_end is None else 1
        return _RunConfig(int(self.delta), int(self.workers), thr, int(self.triangle_mode), m,
                          int(self.shard_target), center_begin, center_end, has_t,
                          int(self.first_edge_t_end or 0))


@dataclass
class PhaseTimings:
    ingest_ms: float = 0.0
    index_ms: float = 0.0
    star_pair_ms: float = 0.0
    triangle_ms: float = 0.0
    merge_ms: float = 0.0

    def total_ms(self) -> float:
        return self.ingest_ms + self.index_ms + self.star_pair_ms + self.triangle_ms + self.merge_ms


def auto_degree_threshold(ctx: GraphContext) -> int:
    v = C.c_uint64(0)
    _raise(ctx._lib.tm_auto_degree_threshold(ctx._h, C.byref(v)), ctx._lib)
    return int(v.value)


@dataclass
class HeavyNode:
    node: int
    shards: List[Tuple[int, int]]


@dataclass
class SchedulePlan:
    """executor.hpp:20-33."""
    heavy: List[HeavyNode] = field(default_factory=list)
    light: List[int] = field(default_factory=list)
    thr_d: int = 0
    shard_target: int = 0
    run_star_pair: bool = True
    run_triangle: bool = True


def plan_schedule(ctx: GraphContext, thr_d: int, shard_target: int, motifs: MotifFilter) -> SchedulePlan:
    """plan_schedule (executor.cpp:23-52): heavy centers (degree > thr_d)
    sharded over their star first-edge range, the rest light.  The reference's
    CPU work plan, for callers that drive the per-center API themselves; the
    device passes parallelise over records and wedges instead."""
    if shard_target < 1:
        raise ConfigError("shard_target must be >= 1")
    plan = SchedulePlan(thr_d=thr_d, shard_target=shard_target,
                        run_star_pair=motifs.star or motifs.pair, run_triangle=motifs.triangle)
    deg = ctx.degrees()
    heavy = np.nonzero(deg > thr_d)[0]
    plan.light = [int(u) for u in np.nonzero(deg <= thr_d)[0]]
    for u in heavy:
        b, e = full_star_range(int(deg[u]))
        plan.heavy.append(HeavyNode(int(u), [(x, min(x + shard_target, e)) for x in range(b, e, shard_target)]))
    return plan


@dataclass
class RawCounters:
    star: StarCounter
    pair: PairCounter
    tri: TriCounter

    def as_array(self) -> np.ndarray:
        return np.concatenate([self.star.cells, self.pair.cells, self.tri.cells]).astype(np.uint64)

    @classmethod
    def from_array(cls, a) -> "RawCounters":
        a = np.asarray(a, np.uint64)
        return cls(StarCounter(a[:24]), PairCounter(a[24:32]), TriCounter(a[32:56]))


def run_parallel_raw(ctx: GraphContext, config: RunConfig, center_begin: int = 0, center_end: int = 0,
                     timings: Optional[PhaseTimings] = None):
    """run_parallel over a center partition; returns (RawCounters, census or None)."""
    L = ctx._lib
    cfg = config.to_c(center_begin, center_end)
    raw = _Counters()
    census = np.zeros(36, np.uint64)
    tm = _Timings()
    _raise(L.tm_run_parallel(ctx._h, C.byref(cfg), C.byref(raw), census.ctypes.data, C.byref(tm)), L)
    if timings is not None:
        timings.star_pair_ms, timings.triangle_ms, timings.merge_ms = tm.star_pair_ms, tm.triangle_ms, tm.merge_ms
    rc = RawCounters(StarCounter(np.frombuffer(raw.star, np.uint64)),
                     PairCounter(np.frombuffer(raw.pair, np.uint64)),
                     TriCounter(np.frombuffer(raw.tri, np.uint64)))
    full = center_begin == 0 and (center_end == 0 or center_end == ctx.node_count()) \
        and config.first_edge_t_end is None
    return rc, (census if full else None)


def run_parallel(ctx: GraphContext, config: RunConfig, timings: Optional[PhaseTimings] = None) -> MotifCensus:
    """run_parallel (executor.cpp:149-215) -- GPU HARE replacement."""
    _, census = run_parallel_raw(ctx, config, timings=timings)
    mc = MotifCensus(census, config.delta)
    mc.meta.edge_count = ctx.edge_count()
    mc.meta.triangle_mode = triangle_mode_name(config.triangle_mode)
    mc.meta.workers = config.workers
    return mc


def count_edges(n: int, src, dst, t, config: RunConfig, stream: Optional[int] = None,
                timings: Optional[PhaseTimings] = None, raw_out: Optional[np.ndarray] = None,
                center: Tuple[int, int] = (0, 0)):
    """One full step from HOST edge arrays: H2D copy + build + count + free."""
    L = lib()
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    t = np.ascontiguousarray(t, np.int64)
    cfg = config.to_c(*center)
    raw = _Counters()
    census = np.zeros(36, np.uint64)
    tm = _Timings()
    # phase timings only when asked for: they add events and a host sync
    rc = L.tm_count_edges(src.ctypes.data, dst.ctypes.data, t.ctypes.data, len(src), n, 0, stream,
                          C.byref(cfg), C.byref(raw), census.ctypes.data,
                          C.byref(tm) if timings is not None else None)
    _raise(rc, L)
    if raw_out is not None:
        raw_out[:24] = np.frombuffer(raw.star, np.uint64)
        raw_out[24:32] = np.frombuffer(raw.pair, np.uint64)
        raw_out[32:56] = np.frombuffer(raw.tri, np.uint64)
    if timings is not None:
        timings.ingest_ms, timings.index_ms, timings.star_pair_ms = tm.ingest_ms, tm.index_ms, tm.star_pair_ms
        timings.triangle_ms, timings.merge_ms = tm.triangle_ms, tm.merge_ms
    return census


class PendingCensus:
    """A census submitted with count_edges_async; result() waits for it.  Keeps
    the host arrays alive until their copy to the device has been waited for."""

    def __init__(self, ticket: int, arrays):
        self.ticket = ticket
        self._arrays = arrays
        self._census = None

    def result(self, raw_out: Optional[np.ndarray] = None) -> np.ndarray:
        if self._census is None:
            L = lib()
            raw = _Counters()
            census = np.zeros(36, np.uint64)
            _raise(L.tm_count_edges_wait(self.ticket, C.byref(raw), census.ctypes.data), L)
            self._raw = np.concatenate([np.frombuffer(raw.star, np.uint64), np.frombuffer(raw.pair, np.uint64),
                                        np.frombuffer(raw.tri, np.uint64)])
            self._census = census
            self._arrays = None
        if raw_out is not None:
            raw_out[:56] = self._raw
        return self._census


def async_h2d_bytes() -> int:
    """Input bytes the last count_edges_async batch put on the host->device
    link (tm_async_h2d_bytes: 16 per edge, 12 when its timestamps travel
    packed)."""
    L = lib()
    b = C.c_uint64(0)
    _raise(L.tm_async_h2d_bytes(C.byref(b)), L)
    return int(b.value)


def count_edges_async(n: int, src, dst, t, config: RunConfig, stream: Optional[int] = None) -> PendingCensus:
    """Pipelined count_edges for batches streamed from host memory
    (tm_count_edges_async): the copy of this batch overlaps the previous
    batch's census.  src/dst/t should live in pinned memory."""
    L = lib()
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    t = np.ascontiguousarray(t, np.int64)
    cfg = config.to_c()
    ticket = C.c_uint64(0)
    _raise(L.tm_count_edges_async(src.ctypes.data, dst.ctypes.data, t.ctypes.data, len(src), n, stream,
                                  C.byref(cfg), C.byref(ticket)), L)
    return PendingCensus(ticket.value, (src, dst, t))


def count_edges_device(n: int, m: int, src_ptr: int, dst_ptr: int, t_ptr: int, config: RunConfig,
                       stream: Optional[int] = None, center: Tuple[int, int] = (0, 0),
                       raw_out: Optional[np.ndarray] = None, timings: Optional[PhaseTimings] = None):
    """One full step from device-resident edge arrays (pointers)."""
    L = lib()
    cfg = config.to_c(*center)
    raw = _Counters()
    census = np.zeros(36, np.uint64)
    tm = _Timings()
    rc = L.tm_count_edges(src_ptr, dst_ptr, t_ptr, m, n, 1, stream, C.byref(cfg), C.byref(raw),
                          census.ctypes.data, C.byref(tm) if timings is not None else None)
    _raise(rc, L)
    if raw_out is not None:
        raw_out[:24] = np.frombuffer(raw.star, np.uint64)
        raw_out[24:32] = np.frombuffer(raw.pair, np.uint64)
        raw_out[32:56] = np.frombuffer(raw.tri, np.uint64)
    if timings is not None:
        timings.ingest_ms, timings.index_ms, timings.star_pair_ms = tm.ingest_ms, tm.index_ms, tm.star_pair_ms
        timings.triangle_ms, timings.merge_ms = tm.triangle_ms, tm.merge_ms
    return census


def count_edges_time_slice(n: int, src, dst, t, config: RunConfig, t_lo: Optional[int] = None,
                           t_hi: Optional[int] = None, m: Optional[int] = None,
                           stream: Optional[int] = None) -> RawCounters:
    """One rank's share of a time-sliced census (tm_count_edges_time_slice):
    the instances whose earliest edge has t in [t_lo, t_hi).  src/dst/t are
    numpy host arrays, or device pointers (ints) together with `m`."""
    L = lib()
    cfg = config.to_c()
    raw = _Counters()
    tm_ = _Timings()
    if m is None:
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        t = np.ascontiguousarray(t, np.int64)
        args = (src.ctypes.data, dst.ctypes.data, t.ctypes.data, len(src), n, 0)
    else:
        args = (src, dst, t, m, n, 1)
    _raise(L.tm_count_edges_time_slice(*args, stream, C.byref(cfg), int(t_lo is not None), int(t_lo or 0),
                                       int(t_hi is not None), int(t_hi or 0), C.byref(raw), None), L)
    return RawCounters(StarCounter(np.frombuffer(raw.star, np.uint64)),
                       PairCounter(np.frombuffer(raw.pair, np.uint64)),
                       TriCounter(np.frombuffer(raw.tri, np.uint64)))
