"""TEST INFRASTRUCTURE ONLY: CPU checkers for the GPU temporal-motif path.

`Oracle` wraps oracle/liboracle.so (plain-C restatement of the reference's
FAST-Star / FAST-Tri / brute-force enumerator); `Reference` wraps
oracle/_ref/libtmotif_ref.so (the reference's own sources compiled in place).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtmotif_ref.so")

u64p = C.POINTER(C.c_uint64)


def build(quiet: bool = True) -> None:
    """Build liboracle.so and (if /root/reference exists) _ref/libtmotif_ref.so."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def _arr(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(C.c_void_p)


class _Graph:
    def __init__(self, lib, handle, n, m):
        self._lib, self.h, self.n, self.m = lib, handle, n, m


class Oracle:
    """ctypes view of liboracle.so."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_build.restype = C.c_void_p
        L.orc_build.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_free.argtypes = [C.c_void_p]
        for f in ("orc_star_pair_at_center",):
            getattr(L, f).argtypes = [C.c_void_p, C.c_uint32, C.c_int64, C.c_uint64, C.c_uint64,
                                      C.c_void_p, C.c_void_p]
        L.orc_triangles_at_center.argtypes = [C.c_void_p, C.c_uint32, C.c_int64, C.c_uint64,
                                              C.c_uint64, C.c_void_p, C.c_void_p]
        L.orc_count_star_pair.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.orc_count_triangles.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        L.orc_merge_census.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.orc_census_bruteforce.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_census_bruteforce_before.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        L.orc_signature.argtypes = [C.c_int, C.c_char_p]
        L.orc_cell_signature.argtypes = [C.c_int, C.c_int]
        L.orc_auto_degree_threshold.restype = C.c_uint64
        L.orc_auto_degree_threshold.argtypes = [C.c_void_p]
        L.orc_degree.restype = C.c_uint64
        L.orc_degree.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_sequence.restype = C.c_uint64
        L.orc_sequence.argtypes = [C.c_void_p, C.c_uint32] + [C.c_void_p] * 4
        L.orc_pair_window.restype = C.c_uint64
        L.orc_pair_window.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_int64, C.c_int64,
                                      C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_generate_random_graph.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_uint64,
                                                C.c_void_p, C.c_void_p, C.c_void_p]
        self.L = L

    # -- graph -----------------------------------------------------------
    def build_graph(self, n, src, dst, t):
        s, ps = _arr(src, np.uint32)
        d, pd = _arr(dst, np.uint32)
        tt, pt = _arr(t, np.int64)
        h = self.L.orc_build(n, len(s), ps, pd, pt)
        if not h:
            raise ValueError("invalid edge list (self-loop or endpoint out of range)")
        g = _Graph(self.L, h, n, len(s))
        return g

    def free(self, g):
        if g.h:
            self.L.orc_free(g.h)
            g.h = None

    def degree(self, g, u):
        return int(self.L.orc_degree(g.h, u))

    def sequence(self, g, u):
        s = self.degree(g, u)
        t = np.zeros(s, np.int64); o = np.zeros(s, np.uint64)
        other = np.zeros(s, np.uint32); d = np.zeros(s, np.uint8)
        self.L.orc_sequence(g.h, u, t.ctypes.data, o.ctypes.data, other.ctypes.data, d.ctypes.data)
        return t, o, other, d

    def pair_window(self, g, v, w, lo, hi):
        cap = g.m
        t = np.zeros(max(cap, 1), np.int64); o = np.zeros(max(cap, 1), np.uint64)
        d = np.zeros(max(cap, 1), np.uint8)
        k = self.L.orc_pair_window(g.h, v, w, lo, hi, t.ctypes.data, o.ctypes.data, d.ctypes.data)
        return t[:k], o[:k], d[:k]

    def auto_degree_threshold(self, g):
        return int(self.L.orc_auto_degree_threshold(g.h))

    # -- counters ----------------------------------------------------------
    def star_pair_at_center(self, g, u, delta, begin, end):
        st = np.zeros(24, np.uint64); pr = np.zeros(8, np.uint64)
        rc = self.L.orc_star_pair_at_center(g.h, u, delta, begin, end, st.ctypes.data, pr.ctypes.data)
        if rc:
            raise OverflowError("oracle counter overflow")
        return st, pr

    def triangles_at_center(self, g, u, delta, begin, end, live=None):
        tr = np.zeros(24, np.uint64)
        lv = None
        if live is not None:
            lv = np.ascontiguousarray(live, np.uint8)
        rc = self.L.orc_triangles_at_center(g.h, u, delta, begin, end,
                                            lv.ctypes.data if lv is not None else None, tr.ctypes.data)
        if rc:
            raise OverflowError("oracle counter overflow")
        return tr

    def count_star_pair(self, g, delta):
        st = np.zeros(24, np.uint64); pr = np.zeros(8, np.uint64)
        if self.L.orc_count_star_pair(g.h, delta, st.ctypes.data, pr.ctypes.data):
            raise OverflowError("oracle counter overflow")
        return st, pr

    def count_triangles(self, g, delta, removal=False):
        tr = np.zeros(24, np.uint64)
        if self.L.orc_count_triangles(g.h, delta, int(removal), tr.ctypes.data):
            raise OverflowError("oracle counter overflow")
        return tr

    def merge_census(self, star, pair, tri, removal=False):
        st, _ = _arr(star, np.uint64); pr, _ = _arr(pair, np.uint64); tr, _ = _arr(tri, np.uint64)
        out = np.zeros(36, np.uint64)
        rc = self.L.orc_merge_census(st.ctypes.data, pr.ctypes.data, tr.ctypes.data, int(removal),
                                     out.ctypes.data)
        if rc == 5:
            raise ArithmeticError("consistency error")
        if rc:
            raise OverflowError("overflow")
        return out

    def census(self, g, delta, removal=False):
        st, pr = self.count_star_pair(g, delta)
        tr = self.count_triangles(g, delta, removal)
        return self.merge_census(st, pr, tr, removal)

    def census_bruteforce(self, g, delta):
        out = np.zeros(36, np.uint64)
        if self.L.orc_census_bruteforce(g.h, delta, out.ctypes.data):
            raise OverflowError("overflow")
        return out

    def census_bruteforce_before(self, g, delta, t_end):
        """Brute-force census of the instances whose earliest edge has t < t_end."""
        out = np.zeros(36, np.uint64)
        if self.L.orc_census_bruteforce_before(g.h, delta, t_end, out.ctypes.data):
            raise OverflowError("overflow")
        return out

    def signatures(self):
        out = []
        buf = C.create_string_buffer(9)
        for k in range(36):
            self.L.orc_signature(k, buf)
            out.append(buf.value.decode())
        return out

    def cell_signature(self, kind, cell):
        return int(self.L.orc_cell_signature(kind, cell))

    def generate_random_graph(self, nodes, m, t_max, seed):
        src = np.zeros(m, np.uint32); dst = np.zeros(m, np.uint32); t = np.zeros(m, np.int64)
        if self.L.orc_generate_random_graph(nodes, m, t_max, seed, src.ctypes.data, dst.ctypes.data,
                                            t.ctypes.data):
            raise ValueError("bad generator parameters")
        return src, dst, t


class Reference:
    """ctypes view of oracle/_ref/libtmotif_ref.so (the reference's own code)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        L = C.CDLL(REF_SO)
        L.ref_build.restype = C.c_void_p
        L.ref_build.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_counters.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_star_pair_at_center.argtypes = [C.c_void_p, C.c_uint32, C.c_int64, C.c_uint64,
                                              C.c_uint64, C.c_void_p, C.c_void_p]
        L.ref_triangles_at_center.argtypes = [C.c_void_p, C.c_uint32, C.c_int64, C.c_uint64,
                                              C.c_uint64, C.c_void_p, C.c_void_p]
        L.ref_run_parallel.argtypes = [C.c_void_p, C.c_int64, C.c_uint, C.c_int64, C.c_int, C.c_int,
                                       C.c_uint64, C.c_void_p]
        L.ref_oracle_census.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.ref_auto_degree_threshold.restype = C.c_uint64
        L.ref_auto_degree_threshold.argtypes = [C.c_void_p]
        L.ref_signature.argtypes = [C.c_int, C.c_char_p]
        L.ref_pipeline.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int64, C.c_uint, C.c_void_p, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)]
        L.ref_generate_random_graph.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_uint64,
                                                C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_parse_edge_list.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_char_p, C.c_void_p, C.c_void_p, C.c_char_p]
        self.L = L

    def build_graph(self, n, src, dst, t):
        s, ps = _arr(src, np.uint32); d, pd = _arr(dst, np.uint32); tt, pt = _arr(t, np.int64)
        h = self.L.ref_build(n, len(s), ps, pd, pt)
        if not h:
            raise ValueError("reference rejected the edge list")
        return _Graph(self.L, h, n, len(s))

    def free(self, g):
        if g.h:
            self.L.ref_free(g.h)
            g.h = None

    def counters(self, g, delta, removal=False):
        st = np.zeros(24, np.uint64); pr = np.zeros(8, np.uint64); tr = np.zeros(24, np.uint64)
        rc = self.L.ref_counters(g.h, delta, int(removal), st.ctypes.data, pr.ctypes.data, tr.ctypes.data)
        if rc:
            raise RuntimeError(f"reference error {rc}")
        return st, pr, tr

    def star_pair_at_center(self, g, u, delta, begin, end):
        st = np.zeros(24, np.uint64); pr = np.zeros(8, np.uint64)
        self.L.ref_star_pair_at_center(g.h, u, delta, begin, end, st.ctypes.data, pr.ctypes.data)
        return st, pr

    def triangles_at_center(self, g, u, delta, begin, end, live=None):
        tr = np.zeros(24, np.uint64)
        lv = None if live is None else np.ascontiguousarray(live, np.uint8)
        self.L.ref_triangles_at_center(g.h, u, delta, begin, end,
                                       lv.ctypes.data if lv is not None else None, tr.ctypes.data)
        return tr

    def run_parallel(self, g, delta, workers=1, thr=-1, removal=False, motifs=7, shard_target=0):
        out = np.zeros(36, np.uint64)
        rc = self.L.ref_run_parallel(g.h, delta, workers, thr, int(removal), motifs, shard_target,
                                     out.ctypes.data)
        if rc:
            raise RuntimeError(f"reference error {rc}")
        return out

    def oracle_census(self, g, delta):
        out = np.zeros(36, np.uint64)
        self.L.ref_oracle_census(g.h, delta, out.ctypes.data)
        return out

    def auto_degree_threshold(self, g):
        return int(self.L.ref_auto_degree_threshold(g.h))

    def signatures(self):
        buf = C.create_string_buffer(9)
        out = []
        for k in range(36):
            self.L.ref_signature(k, buf)
            out.append(buf.value.decode())
        return out

    def pipeline(self, n, src, dst, t, delta, workers):
        s, ps = _arr(src, np.uint32); d, pd = _arr(dst, np.uint32); tt, pt = _arr(t, np.int64)
        out = np.zeros(36, np.uint64)
        mb, mc = C.c_double(0), C.c_double(0)
        rc = self.L.ref_pipeline(n, len(s), ps, pd, pt, delta, workers, out.ctypes.data,
                                 C.byref(mb), C.byref(mc))
        if rc:
            raise RuntimeError(f"reference error {rc}")
        return out, mb.value, mc.value

    def generate_random_graph(self, nodes, m, t_max, seed):
        src = np.zeros(m, np.uint32); dst = np.zeros(m, np.uint32); t = np.zeros(m, np.int64)
        if self.L.ref_generate_random_graph(nodes, m, t_max, seed, src.ctypes.data, dst.ctypes.data,
                                            t.ctypes.data):
            raise ValueError("bad generator parameters")
        return src, dst, t

    def parse_edge_list(self, text: bytes, drop_self_loops: bool = True):
        """The reference's parse_edge_list: (node_ids, src, dst, t, dropped)
        in ingestion order, or raises ValueError((line, message))."""
        lines = text.count(b"\n") + 1
        counts = np.zeros(3, np.uint64)
        src = np.zeros(lines, np.uint32); dst = np.zeros(lines, np.uint32); t = np.zeros(lines, np.int64)
        ids = C.create_string_buffer(len(text) + 1)
        ids_len = np.zeros(1, np.uint64)
        err_line = np.zeros(1, np.uint64)
        err = C.create_string_buffer(512)
        rc = self.L.ref_parse_edge_list(text, len(text), int(drop_self_loops), counts.ctypes.data,
                                        src.ctypes.data, dst.ctypes.data, t.ctypes.data, ids,
                                        ids_len.ctypes.data, err_line.ctypes.data, err)
        if rc:
            raise ValueError((int(err_line[0]), err.value.decode("utf-8", "surrogateescape")))
        n, m, dropped = (int(x) for x in counts)
        names = ids.raw[:int(ids_len[0])].decode("utf-8", "surrogateescape").split("\n") if n else []
        return names, src[:m], dst[:m], t[:m], dropped
