"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU checkers.

* ``Oracle``   : liboracle.so, the plain-C restatement of the reference path
                 (oracle.c; every function cites the reference file:line).
* ``RefLib``   : oracle/_ref/libgraphlet_ref.so, the reference's OWN sources
                 (/root/reference/proj/src/*.cpp) compiled in place by
                 oracle/Makefile plus a thin extern "C" driver.  Present only
                 where it was built; tests skip when absent.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgraphlet_ref.so")

MICRO_FIELDS = ("edge_id", "x3", "x4", "x5", "x7", "x10", "t", "s_u", "s_v", "d_e")
MICRO_DTYPE = np.dtype([(f, "<u8") for f in MICRO_FIELDS])


def _x_from(arr) -> list:
    return [int(arr[2 * i]) | (int(arr[2 * i + 1]) << 64) for i in range(len(arr) // 2)]


class _OrGraph(C.Structure):
    _fields_ = [("n", C.c_uint64), ("m", C.c_uint64), ("dmax", C.c_uint32),
                ("offsets", C.POINTER(C.c_uint64)), ("adj_id", C.POINTER(C.c_uint32)),
                ("adj_deg", C.POINTER(C.c_uint32)), ("degree", C.POINTER(C.c_uint32)),
                ("inverse_map", C.POINTER(C.c_uint64))]


def _pairs(pairs):
    p = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint64).reshape(-1, 2))
    a = np.ascontiguousarray(p[:, 0])
    b = np.ascontiguousarray(p[:, 1])
    return a, b, p.shape[0]


class Oracle:
    """liboracle.so wrapper; one instance per graph."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                raise RuntimeError(f"{ORACLE_SO} missing; run make -C oracle")
            L = C.CDLL(ORACLE_SO)
            vp = C.c_void_p
            L.or_build_graph.argtypes = [vp, vp, C.c_uint64, C.POINTER(_OrGraph)]
            L.or_build_graph.restype = C.c_int
            L.or_free_graph.argtypes = [C.POINTER(_OrGraph)]
            L.or_orient_edges.argtypes = [C.POINTER(_OrGraph), vp, vp]
            L.or_count.argtypes = [C.POINTER(_OrGraph), C.c_int, vp, vp]
            L.or_count.restype = C.c_int
            L.or_process_edge_bsearch.argtypes = [C.POINTER(_OrGraph), C.c_uint32, C.c_uint32, vp]
            L.or_process_edge_hash_one.argtypes = [C.POINTER(_OrGraph), C.c_uint32, C.c_uint32, C.c_uint64, vp]
            L.or_edges_hash.argtypes = [C.POINTER(_OrGraph), vp, C.c_uint64, vp]
            L.or_time_sample.argtypes = [C.POINTER(_OrGraph), C.c_int, vp, C.c_uint64, C.POINTER(C.c_uint64)]
            L.or_time_sample.restype = C.c_double
            L.or_brute_force_global.argtypes = [C.POINTER(_OrGraph), C.c_uint32, vp]
            L.or_brute_force_global.restype = C.c_int
            L.or_global_from_unrestricted.argtypes = [vp, C.c_uint64, C.c_uint64, vp]
            L.or_global_from_unrestricted.restype = C.c_int
            L.or_generate_rmat.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                           C.c_uint64, C.c_int, vp]
            L.or_generate_rmat.restype = C.c_int
            L.or_generate_ba.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.POINTER(C.POINTER(C.c_uint64)),
                                         C.POINTER(C.c_uint64)]
            L.or_generate_ba.restype = C.c_int
            L.or_free_pairs.argtypes = [vp]
            cls._lib = L
        return cls._lib

    def __init__(self, pairs):
        L = self.lib()
        a, b, k = _pairs(pairs)
        self.g = _OrGraph()
        if L.or_build_graph(a.ctypes.data, b.ctypes.data, k, C.byref(self.g)) != 0:
            raise OverflowError("graph exceeds 32-bit vertex id space")

    def __del__(self):
        try:
            self.lib().or_free_graph(C.byref(self.g))
        except Exception:
            pass

    @property
    def n(self):
        return int(self.g.n)

    @property
    def m(self):
        return int(self.g.m)

    def degrees(self):
        return np.ctypeslib.as_array(self.g.degree, shape=(self.n,)).copy() if self.n else np.zeros(0, np.uint32)

    def labels(self):
        return np.ctypeslib.as_array(self.g.inverse_map, shape=(self.n,)).copy() if self.n else np.zeros(0, np.uint64)

    def csr(self):
        off = np.ctypeslib.as_array(self.g.offsets, shape=(self.n + 1,)).copy()
        adj = (np.ctypeslib.as_array(self.g.adj_id, shape=(2 * self.m,)).copy()
               if self.m else np.zeros(0, np.uint32))
        return off, adj

    def orient_edges(self):
        v = np.zeros(self.m, np.uint32)
        u = np.zeros(self.m, np.uint32)
        self.lib().or_orient_edges(C.byref(self.g), v.ctypes.data, u.ctypes.data)
        return v, u

    def count(self, threads: int = 1, micro: bool = False):
        X = np.zeros(36, np.uint64)
        rec = np.zeros(self.m, MICRO_DTYPE) if micro else None
        rc = self.lib().or_count(C.byref(self.g), threads, X.ctypes.data,
                                 rec.ctypes.data if micro else None)
        if rc != 0:
            raise ArithmeticError("oracle count consistency/overflow error")
        return (_x_from(X), rec) if micro else _x_from(X)

    def edge_bsearch(self, v, u):
        r = np.zeros(5, np.uint64)
        self.lib().or_process_edge_bsearch(C.byref(self.g), int(v), int(u), r.ctypes.data)
        return [int(x) for x in r]

    def edge_hash(self, v, u, eid):
        r = np.zeros(5, np.uint64)
        self.lib().or_process_edge_hash_one(C.byref(self.g), int(v), int(u), int(eid), r.ctypes.data)
        return [int(x) for x in r]

    def edges_hash(self, edge_ids):
        """{t, s_u, s_v, x7, x10} per listed edge id (hash pipeline)."""
        ids = np.ascontiguousarray(edge_ids, dtype=np.uint64)
        out = np.zeros((len(ids), 5), np.uint64)
        self.lib().or_edges_hash(C.byref(self.g), ids.ctypes.data, len(ids), out.ctypes.data)
        return out

    def time_sample(self, edge_ids, threads: int):
        ids = np.ascontiguousarray(edge_ids, dtype=np.uint64)
        cs = C.c_uint64()
        secs = self.lib().or_time_sample(C.byref(self.g), threads, ids.ctypes.data, len(ids), C.byref(cs))
        return float(secs), int(cs.value)

    def brute_force(self, cap: int = 64):
        X = np.zeros(36, np.uint64)
        if self.lib().or_brute_force_global(C.byref(self.g), cap, X.ctypes.data) != 0:
            raise ValueError("brute force census capped")
        return _x_from(X)


def global_from_unrestricted(Cs, n, m):
    L = Oracle.lib()
    arr = np.zeros(34, np.uint64)
    for i, v in enumerate(Cs):
        arr[2 * i] = v & ((1 << 64) - 1)
        arr[2 * i + 1] = v >> 64
    X = np.zeros(36, np.uint64)
    if L.or_global_from_unrestricted(arr.ctypes.data, n, m, X.ctypes.data) != 0:
        raise ArithmeticError("count consistency error")
    return _x_from(X)


def generate_rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
                  seed: int = 1, threads: int = 0) -> np.ndarray:
    """(count, 2) uint64 labels, identical to the product's gl_generate_rmat."""
    L = Oracle.lib()
    count = edge_factor << scale
    out = np.empty((count, 2), np.uint64)
    if L.or_generate_rmat(scale, edge_factor, a, b, c, seed, threads or (os.cpu_count() or 1), out.ctypes.data):
        raise ValueError("bad RMAT parameters")
    return out


def generate_ba(n: int, attach: int, seed: int = 1) -> np.ndarray:
    """(count, 2) uint64 labels, identical to the product's gl_generate_ba."""
    L = Oracle.lib()
    p = C.POINTER(C.c_uint64)()
    cnt = C.c_uint64()
    if L.or_generate_ba(n, attach, seed, C.byref(p), C.byref(cnt)):
        raise ValueError("bad BA parameters")
    k = int(cnt.value)
    if k == 0:
        return np.zeros((0, 2), np.uint64)
    try:
        return np.ctypeslib.as_array(p, shape=(2 * k,)).copy().reshape(k, 2)
    finally:
        L.or_free_pairs(p)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefLib:
    """The reference's own code (compiled from /root/reference sources)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not ref_available():
                raise RuntimeError(f"{REF_SO} missing (reference sources not compiled here)")
            L = C.CDLL(REF_SO)
            vp = C.c_void_p
            L.ref_build.argtypes = [vp, vp, C.c_uint64]
            L.ref_build.restype = vp
            L.ref_free.argtypes = [vp]
            L.ref_n.argtypes = [vp]
            L.ref_n.restype = C.c_uint64
            L.ref_m.argtypes = [vp]
            L.ref_m.restype = C.c_uint64
            L.ref_dmax.argtypes = [vp]
            L.ref_dmax.restype = C.c_uint32
            L.ref_orient.argtypes = [vp, vp, vp, vp, vp]
            L.ref_degrees.argtypes = [vp, vp]
            L.ref_parse.argtypes = [C.c_char_p, C.c_uint64, vp, C.c_uint64, C.POINTER(C.c_uint64)]
            L.ref_parse.restype = C.c_int64
            L.ref_edge_records.argtypes = [vp, C.c_int, vp]
            L.ref_count.argtypes = [vp, C.c_int, vp, vp]
            L.ref_count.restype = C.c_int
            L.ref_time_sample.argtypes = [vp, C.c_int, vp, C.c_uint64, C.POINTER(C.c_uint64)]
            L.ref_time_sample.restype = C.c_double
            L.ref_brute.argtypes = [vp, C.c_uint32, vp]
            L.ref_brute.restype = C.c_int
            L.ref_brute_edges.argtypes = [vp, vp]
            L.ref_last_error.restype = C.c_char_p
            L.ref_edges.argtypes = [vp, C.c_int, vp, C.c_uint64, vp]
            L.ref_edges.restype = C.c_int
            cls._lib = L
        return cls._lib

    def __init__(self, pairs):
        L = self.lib()
        a, b, k = _pairs(pairs)
        self.h = L.ref_build(a.ctypes.data, b.ctypes.data, k)
        if not self.h:
            raise RuntimeError(L.ref_last_error().decode())

    def __del__(self):
        try:
            if self.h:
                self.lib().ref_free(self.h)
        except Exception:
            pass

    @property
    def n(self):
        return int(self.lib().ref_n(self.h))

    @property
    def m(self):
        return int(self.lib().ref_m(self.h))

    def orient(self):
        m = self.m
        v, u = np.zeros(m, np.uint32), np.zeros(m, np.uint32)
        vl, ul = np.zeros(m, np.uint64), np.zeros(m, np.uint64)
        self.lib().ref_orient(self.h, v.ctypes.data, u.ctypes.data, vl.ctypes.data, ul.ctypes.data)
        return v, u, vl, ul

    def degrees(self):
        d = np.zeros(self.n, np.uint32)
        self.lib().ref_degrees(self.h, d.ctypes.data)
        return d

    def edge_records(self, variant: int = 0):
        out = np.zeros((self.m, 6), np.uint64)
        self.lib().ref_edge_records(self.h, variant, out.ctypes.data)
        return out

    def count(self, threads: int = 1, micro: bool = False):
        X = np.zeros(36, np.uint64)
        rec = np.zeros(self.m, MICRO_DTYPE) if micro else None
        rc = self.lib().ref_count(self.h, threads, X.ctypes.data, rec.ctypes.data if micro else None)
        if rc != 0:
            raise ArithmeticError(self.lib().ref_last_error().decode())
        return (_x_from(X), rec) if micro else _x_from(X)

    def edges(self, edge_ids, threads: int = 1):
        """The reference's process_edge_hash for the listed edge ids:
        (k, 7) rows {v label, u label, t, s_u, s_v, x7, x10}."""
        ids = np.ascontiguousarray(edge_ids, dtype=np.uint64)
        out = np.zeros((len(ids), 7), np.uint64)
        if self.lib().ref_edges(self.h, threads, ids.ctypes.data, len(ids), out.ctypes.data) != 0:
            raise RuntimeError(self.lib().ref_last_error().decode())
        return out

    def time_sample(self, edge_ids, threads: int):
        ids = np.ascontiguousarray(edge_ids, dtype=np.uint64)
        cs = C.c_uint64()
        secs = self.lib().ref_time_sample(self.h, threads, ids.ctypes.data, len(ids), C.byref(cs))
        return float(secs), int(cs.value)

    def brute_force(self, cap: int = 64):
        X = np.zeros(36, np.uint64)
        if self.lib().ref_brute(self.h, cap, X.ctypes.data) != 0:
            raise ValueError(self.lib().ref_last_error().decode())
        return _x_from(X)

    def brute_edges(self):
        out = np.zeros((self.m, 6), np.uint64)
        self.lib().ref_brute_edges(self.h, out.ctypes.data)
        return out

    @classmethod
    def parse(cls, text):
        if isinstance(text, str):
            text = text.encode()
        L = cls.lib()
        cap = text.count(b"\n") + 2
        out = np.zeros(2 * cap, np.uint64)
        line = C.c_uint64()
        k = L.ref_parse(text, len(text), out.ctypes.data, cap, C.byref(line))
        if k < 0:
            return None, int(line.value), L.ref_last_error().decode()
        return out[: 2 * k].reshape(k, 2), 0, ""
