"""B200-native edge-centric k<=4 graphlet decomposition (arxiv 1608.05138).

Python mirror of the reference's C++ API for the counting path
(/root/reference/proj/include/graphlet/{graph,counts,kernels}.hpp), bound with
ctypes to the C-ABI in include/graphlet_b200.h (libgraphlet_b200.so, built
in-tree for sm_100a).  There is no CPU fallback: if the shared library is
missing, importing this package raises ImportError, and every counting call
needs a CUDA device.

Reference name             -> here
  load_edge_list(istream)  -> load_edge_list(text)          (graph.hpp:38)
  load_edge_list_file      -> load_edge_list_file(path)     (graph.hpp:39)
  build_graph(RawEdges)    -> Graph.build(pairs)            (graph.hpp:96)
  orient_edges(g)          -> Graph.orient_edges()          (graph.hpp:107)
  process_edge_* loop +
  accumulate/merge/global  -> Graph.count()                 (kernels.hpp:99-102,
                                                             counts.hpp:49-70)
  micro_counts(rec, n)     -> Graph.micro_records()         (counts.hpp:90)
  global_from_unrestricted -> global_from_unrestricted()    (counts.hpp:69)
  graphlet_name(i)         -> graphlet_name(i)              (counts.hpp:64)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "GraphletError", "ParseError", "CountConsistencyError", "CountOverflowError",
    "CudaError", "Graph", "load_edge_list", "load_edge_list_file", "parse_edge_list_device", "generate_rmat",
    "generate_rmat_device", "generate_gnm", "generate_ba", "global_from_unrestricted",
    "graphlet_name", "GRAPHLET_NAMES", "MICRO_DTYPE", "MOTIF_DTYPE", "local_three_counts", "lib_path", "LIB",
]

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    # GRAPHLET_B200_LIB selects another in-tree build of the same library
    # (e.g. libgraphlet_b200_prof.so, the phase-instrumented variant)
    return os.path.join(_HERE, os.environ.get("GRAPHLET_B200_LIB", "libgraphlet_b200.so"))


if not os.path.exists(lib_path()):
    raise ImportError(
        f"{lib_path()} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(make -C paper_1608_05138_b200/csrc). There is no CPU fallback.")

LIB = C.CDLL(lib_path())

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)


class _U128(C.Structure):
    _fields_ = [("lo", C.c_uint64), ("hi", C.c_uint64)]


class _GV(C.Structure):
    _fields_ = [("x", _U128 * 18)]


class _UC(C.Structure):
    _fields_ = [("c", _U128 * 17)]


MICRO_FIELDS = ("edge_id", "x3", "x4", "x5", "x7", "x10", "t", "s_u", "s_v", "d_e")
MICRO_DTYPE = np.dtype([(f, "<u8") for f in MICRO_FIELDS])
# EdgeMotifRecord (counts.hpp:20-35), hash pipeline (kernels.cpp:143-156)
MOTIF_DTYPE = np.dtype([("edge_id", "<u4"), ("t", "<u4"), ("s_u", "<u4"), ("s_v", "<u4"),
                        ("x7", "<u8"), ("x10", "<u8"), ("work_units", "<u8")])

GRAPHLET_NAMES = {
    1: "edge", 2: "2-node-independent", 3: "triangle", 4: "2-star", 5: "3-node-1-edge",
    6: "3-node-independent", 7: "4-clique", 8: "chordal-cycle", 9: "tailed-triangle",
    10: "4-cycle", 11: "3-star", 12: "4-path", 13: "4-node-1-triangle", 14: "4-node-2-edge",
    15: "4-node-2-star", 16: "4-node-1-edge", 17: "4-node-independent",
}


def graphlet_name(i: int) -> str:
    """counts.cpp:47-68 -- class id to readable name ("?" when unknown)."""
    return GRAPHLET_NAMES.get(i, "?")


def _sig(name, res, *args):
    f = getattr(LIB, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("gl_last_error", C.c_char_p)
_sig("gl_last_error_line", C.c_uint64)
_sig("gl_version", C.c_char_p)
_sig("gl_free", None, C.c_void_p)
_sig("gl_load_edge_list", C.c_int, C.c_char_p, C.c_size_t, C.POINTER(_u64p), _u64p)
_sig("gl_load_edge_list_file", C.c_int, C.c_char_p, C.POINTER(_u64p), _u64p)
_sig("gl_parse_edge_list_device", C.c_int, C.c_char_p, C.c_size_t, C.c_int, C.POINTER(_u64p), _u64p)
_sig("gl_graph_build_text", C.c_int, C.c_void_p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p))
_sig("gl_generate_rmat", C.c_int, C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
     C.c_uint64, C.POINTER(_u64p), _u64p)
_sig("gl_generate_rmat_device", C.c_int, C.c_uint32, C.c_uint32, C.c_double, C.c_double,
     C.c_double, C.c_uint64, C.c_int, C.c_void_p, C.c_uint64)
_sig("gl_generate_gnm", C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(_u64p), _u64p)
_sig("gl_generate_ba", C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, C.POINTER(_u64p), _u64p)
_sig("gl_graph_build", C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p))
_sig("gl_graph_build_device", C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p))
_sig("gl_graph_free", None, C.c_void_p)
_sig("gl_graph_num_vertices", C.c_uint64, C.c_void_p)
_sig("gl_graph_num_edges", C.c_uint64, C.c_void_p)
_sig("gl_graph_max_degree", C.c_uint32, C.c_void_p)
_sig("gl_graph_degrees", C.c_int, C.c_void_p, C.c_void_p)
_sig("gl_graph_labels", C.c_int, C.c_void_p, C.c_void_p)
_sig("gl_graph_csr", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
_sig("gl_orient_edges", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
_sig("gl_count", C.c_int, C.c_void_p, C.POINTER(_GV), C.POINTER(_UC))
_sig("gl_partials_len", C.c_uint64, C.c_void_p, C.c_int)
_sig("gl_count_begin", C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p)
_sig("gl_count_mid", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
_sig("gl_triangle_counts_device", C.c_int, C.c_void_p, C.POINTER(C.c_void_p), _u64p)
_sig("gl_count_finish", C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
     C.POINTER(_UC), C.c_void_p)
_sig("gl_global_from_unrestricted", C.c_int, C.POINTER(_UC), C.c_uint64, C.c_uint64, C.POINTER(_GV))
_sig("gl_count_edges", C.c_int, C.c_void_p, C.POINTER(_GV), C.POINTER(_UC), C.c_void_p, C.c_void_p, C.c_void_p)
_sig("gl_micro_records", C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p)
_sig("gl_edge_motif_records", C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p)
_sig("gl_edge_counts", C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p)
_sig("gl_edge_counts_device", C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
     C.POINTER(C.c_void_p))
_sig("gl_last_timings", C.c_int, C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_uint32))
_sig("gl_last_work", C.c_int, C.c_void_p, _u64p)
_sig("gl_cycle_pieces", C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, _u64p)


class GraphletError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(GraphletError, ValueError):
    pass


class ParseError(GraphletError):
    """graphlet::parse_error (graph.hpp:23-33); .line is 1-based."""

    def __init__(self, code, msg, line):
        super().__init__(code, msg)
        self.line = line


class IOErrorGL(GraphletError, OSError):
    pass


class CudaError(GraphletError):
    pass


class CountConsistencyError(GraphletError):
    pass


class CountOverflowError(GraphletError, OverflowError):
    pass


class StateError(GraphletError):
    pass


_ERRS = {-1: InvalidArgument, -3: IOErrorGL, -4: CudaError, -5: CountConsistencyError,
         -6: CountOverflowError, -7: CudaError, -8: StateError}


def _check(rc: int):
    if rc == 0:
        return
    msg = (LIB.gl_last_error() or b"").decode(errors="replace")
    if rc == -2:
        raise ParseError(rc, msg, int(LIB.gl_last_error_line()))
    raise _ERRS.get(rc, GraphletError)(rc, msg)


def _take_pairs(ptr, count) -> np.ndarray:
    n = int(count.value)
    try:
        if n == 0:
            return np.zeros((0, 2), dtype=np.uint64)
        arr = np.ctypeslib.as_array(ptr, shape=(2 * n,)).copy()
        return arr.reshape(n, 2)
    finally:
        LIB.gl_free(ptr)


def load_edge_list(text) -> np.ndarray:
    """Parse an edge list held in memory -> (count, 2) uint64 pairs in file order."""
    if isinstance(text, str):
        text = text.encode()
    ptr, cnt = _u64p(), C.c_uint64()
    _check(LIB.gl_load_edge_list(text, len(text), C.byref(ptr), C.byref(cnt)))
    return _take_pairs(ptr, cnt)


def parse_edge_list_device(text, device: int = 0) -> np.ndarray:
    """load_edge_list (graph.cpp:47-85) executed on the GPU (parse.cu): same
    pairs, same ParseError line numbers and messages as load_edge_list."""
    if isinstance(text, str):
        text = text.encode()
    ptr, cnt = _u64p(), C.c_uint64()
    _check(LIB.gl_parse_edge_list_device(text, len(text), device, C.byref(ptr), C.byref(cnt)))
    return _take_pairs(ptr, cnt)


def load_edge_list_file(path: str) -> np.ndarray:
    ptr, cnt = _u64p(), C.c_uint64()
    _check(LIB.gl_load_edge_list_file(os.fsencode(path), C.byref(ptr), C.byref(cnt)))
    return _take_pairs(ptr, cnt)


def generate_rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
                  c: float = 0.19, seed: int = 1) -> np.ndarray:
    ptr, cnt = _u64p(), C.c_uint64()
    _check(LIB.gl_generate_rmat(scale, edge_factor, a, b, c, seed, C.byref(ptr), C.byref(cnt)))
    return _take_pairs(ptr, cnt)


def generate_rmat_device(scale: int, edge_factor: int, d_ptr: int, device: int = 0,
                         a: float = 0.57, b: float = 0.19, c: float = 0.19, seed: int = 1) -> int:
    """Write the same RMAT pair list straight into device memory at d_ptr."""
    count = edge_factor << scale
    _check(LIB.gl_generate_rmat_device(scale, edge_factor, a, b, c, seed, device,
                                       C.c_void_p(d_ptr), count))
    return count


def generate_gnm(n: int, m: int, seed: int = 1) -> np.ndarray:
    ptr, cnt = _u64p(), C.c_uint64()
    _check(LIB.gl_generate_gnm(n, m, seed, C.byref(ptr), C.byref(cnt)))
    return _take_pairs(ptr, cnt)


def generate_ba(n: int, attach: int, seed: int = 1) -> np.ndarray:
    ptr, cnt = _u64p(), C.c_uint64()
    _check(LIB.gl_generate_ba(n, attach, seed, C.byref(ptr), C.byref(cnt)))
    return _take_pairs(ptr, cnt)


def _to_int(u: _U128) -> int:
    return int(u.lo) | (int(u.hi) << 64)


def _from_int(v: int, u: _U128):
    if v < 0 or v >> 128:
        raise OverflowError("value does not fit an unsigned 128-bit count")
    u.lo = v & ((1 << 64) - 1)
    u.hi = v >> 64


def global_from_unrestricted(c, n: int, m: int) -> list[int]:
    """counts.cpp:86-111. c: 17 ints (C_0..C_16) -> X_0..X_17 (X_0 = 0)."""
    uc = _UC()
    for i in range(17):
        _from_int(int(c[i]), uc.c[i])
    gv = _GV()
    _check(LIB.gl_global_from_unrestricted(C.byref(uc), n, m, C.byref(gv)))
    return [_to_int(gv.x[i]) for i in range(18)]


@dataclass
class CountResult:
    X: list          # X_0..X_17 (python ints, exact 128-bit)
    C: list          # unrestricted C_0..C_16
    ms: list         # [triangles, cliques, cycles, epilogue, total] device ms
    launches: int
    work: list       # [tri adjacency reads, clique reads, cycle reads, edges finalised]


class Graph:
    """Device-resident preprocessed graph (graphlet::Graph, graph.hpp:41-93)."""

    def __init__(self, handle: int, device: int):
        self._h = C.c_void_p(handle)
        self.device = device

    @classmethod
    def build(cls, pairs, device: int = 0) -> "Graph":
        p = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint64).reshape(-1, 2))
        h = C.c_void_p()
        _check(LIB.gl_graph_build(p.ctypes.data_as(C.c_void_p), p.shape[0], device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def build_host_ptr(cls, host_ptr: int, count: int, device: int = 0) -> "Graph":
        """gl_graph_build on a raw (e.g. pinned) host pointer of 2*count labels."""
        h = C.c_void_p()
        _check(LIB.gl_graph_build(C.c_void_p(host_ptr), count, device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def build_text(cls, text, device: int = 0) -> "Graph":
        """Edge-list text (bytes / str, or a host pointer + length tuple) ->
        graph, parsed on the device (gl_graph_build_text)."""
        h = C.c_void_p()
        if isinstance(text, tuple):
            ptr, n = text
            _check(LIB.gl_graph_build_text(C.c_void_p(ptr), n, device, C.byref(h)))
        else:
            if isinstance(text, str):
                text = text.encode()
            _check(LIB.gl_graph_build_text(text, len(text), device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def build_device(cls, d_ptr: int, count: int, device: int = 0) -> "Graph":
        h = C.c_void_p()
        _check(LIB.gl_graph_build_device(C.c_void_p(d_ptr), count, device, C.byref(h)))
        return cls(h.value, device)

    def close(self):
        if self._h is not None and self._h.value:
            LIB.gl_graph_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def num_vertices(self) -> int:
        return int(LIB.gl_graph_num_vertices(self._h))

    def num_edges(self) -> int:
        return int(LIB.gl_graph_num_edges(self._h))

    def max_degree(self) -> int:
        return int(LIB.gl_graph_max_degree(self._h))

    def degrees(self) -> np.ndarray:
        out = np.zeros(self.num_vertices(), dtype=np.uint32)
        _check(LIB.gl_graph_degrees(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def labels(self) -> np.ndarray:
        out = np.zeros(self.num_vertices(), dtype=np.uint64)
        _check(LIB.gl_graph_labels(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def csr(self):
        off = np.zeros(self.num_vertices() + 1, dtype=np.uint64)
        adj = np.zeros(2 * self.num_edges(), dtype=np.uint32)
        _check(LIB.gl_graph_csr(self._h, off.ctypes.data_as(C.c_void_p), adj.ctypes.data_as(C.c_void_p)))
        return off, adj

    def orient_edges(self):
        m = self.num_edges()
        v = np.zeros(m, dtype=np.uint32)
        u = np.zeros(m, dtype=np.uint32)
        _check(LIB.gl_orient_edges(self._h, v.ctypes.data_as(C.c_void_p), u.ctypes.data_as(C.c_void_p)))
        return v, u

    def count(self) -> CountResult:
        gv, uc = _GV(), _UC()
        _check(LIB.gl_count(self._h, C.byref(gv), C.byref(uc)))
        return CountResult([_to_int(gv.x[i]) for i in range(18)], [_to_int(uc.c[i]) for i in range(17)],
                           *self.last_stats())

    def count_edges(self, t=None, x7=None, x10=None):
        """count() plus every edge's (t, x7, x10) into host arrays (allocated when
        None; pass pinned numpy views to make the early t/x7 copy asynchronous):
        t and x7 leave the device while the cycle pass runs (gl_count_edges)."""
        m = self.num_edges()

        def out(a, dt, name):
            if a is None:
                return np.zeros(m, dtype=dt)
            if (not isinstance(a, np.ndarray) or a.dtype != dt or not a.flags.c_contiguous or a.size < m
                    or not a.flags.writeable):
                raise ValueError(f"{name}: need a writeable C-contiguous {np.dtype(dt).name} array of >= {m}")
            return a
        t, x7, x10 = out(t, np.uint32, "t"), out(x7, np.uint64, "x7"), out(x10, np.uint64, "x10")
        gv, uc = _GV(), _UC()
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _check(LIB.gl_count_edges(self._h, C.byref(gv), C.byref(uc), p(t), p(x7), p(x10)))
        res = CountResult([_to_int(gv.x[i]) for i in range(18)], [_to_int(uc.c[i]) for i in range(17)],
                          *self.last_stats())
        return res, t[:m], x7[:m], x10[:m]

    def last_stats(self):
        ms = (C.c_float * 5)()
        nl = C.c_uint32()
        _check(LIB.gl_last_timings(self._h, ms, C.byref(nl)))
        w = (C.c_uint64 * 4)()
        _check(LIB.gl_last_work(self._h, w))
        return [float(x) for x in ms], int(nl.value), [int(x) for x in w]

    def cycle_pieces(self) -> np.ndarray:
        """Windowed-top work items of the last count: rows (a, c_lo, c_hi, wedge estimate)."""
        n = C.c_uint64()
        _check(LIB.gl_cycle_pieces(self._h, None, 0, C.byref(n)))
        out = np.zeros((n.value, 4), dtype=np.uint32)
        if n.value:
            _check(LIB.gl_cycle_pieces(self._h, out.ctypes.data_as(C.c_void_p), n.value, C.byref(n)))
        return out

    # sharded (one process per GPU) form -------------------------------------
    def partials_len(self, world: int) -> int:
        return int(LIB.gl_partials_len(self._h, world))

    def count_begin(self, rank: int, world: int, d_partials: int, stream: int = 0):
        _check(LIB.gl_count_begin(self._h, rank, world, C.c_void_p(d_partials), C.c_void_p(stream)))

    def count_mid(self, d_partials: int, stream: int = 0):
        _check(LIB.gl_count_mid(self._h, C.c_void_p(d_partials), C.c_void_p(stream)))

    def triangle_counts_device(self):
        p, n = C.c_void_p(), C.c_uint64()
        _check(LIB.gl_triangle_counts_device(self._h, C.byref(p), C.byref(n)))
        return p.value, int(n.value)

    def count_finish(self, d_partials_shard: int, edge_begin: int, edge_end: int, stream: int = 0) -> list:
        uc = _UC()
        _check(LIB.gl_count_finish(self._h, C.c_void_p(d_partials_shard), edge_begin, edge_end,
                                   C.byref(uc), C.c_void_p(stream)))
        return [_to_int(uc.c[i]) for i in range(17)]

    # per-edge output ---------------------------------------------------------
    def micro_records(self, first: int = 0, count: int | None = None, out=None) -> np.ndarray:
        """micro_counts (counts.cpp:122-136) rows of edge ids [first, first+count);
        `out`: optional caller buffer (e.g. a pinned host array) of MICRO_DTYPE."""
        if count is None:
            count = self.num_edges() - first
        if first < 0 or count < 0:
            raise ValueError("negative edge range")
        if out is None:
            out = np.zeros(count, dtype=MICRO_DTYPE)
        elif (not isinstance(out, np.ndarray) or out.dtype != MICRO_DTYPE or not out.flags.c_contiguous
              or out.size < count or not out.flags.writeable):
            raise ValueError(f"out: need a writeable C-contiguous MICRO_DTYPE array of >= {count} rows")
        _check(LIB.gl_micro_records(self._h, first, count, out.ctypes.data_as(C.c_void_p)))
        return out

    def edge_motif_records(self, first: int = 0, count: int | None = None) -> np.ndarray:
        """EdgeMotifRecord rows (t, s_u, s_v, x7, x10, work_units) of edge ids
        [first, first+count), identical to the reference's process_edge_hash
        (kernels.cpp:143-156) including its operation counter."""
        if count is None:
            count = self.num_edges() - first
        if first < 0 or count < 0:
            raise ValueError("negative edge range")
        out = np.zeros(count, dtype=MOTIF_DTYPE)
        _check(LIB.gl_edge_motif_records(self._h, first, count, out.ctypes.data_as(C.c_void_p)))
        return out

    def process_edge_hash(self, edge_id: int) -> np.void:
        """kernels.cpp:143-156 for one oriented edge id (after count())."""
        return self.edge_motif_records(edge_id, 1)[0]

    def edge_counts(self, first: int = 0, count: int | None = None, t=None, x7=None, x10=None):
        if count is None:
            count = self.num_edges() - first
        if first < 0 or count < 0:
            raise ValueError("negative edge range")

        def out(a, dt, name):
            # caller buffers are written through raw pointers: insist on the
            # exact dtype, C contiguity and room for `count` values
            if a is None:
                return np.zeros(count, dtype=dt)
            if not isinstance(a, np.ndarray) or a.dtype != dt or not a.flags.c_contiguous or a.size < count:
                raise ValueError(f"{name}: need a C-contiguous {np.dtype(dt).name} array of >= {count} values")
            if not a.flags.writeable:
                raise ValueError(f"{name}: array is read-only")
            return a

        t = out(t, np.uint32, "t")
        x7 = out(x7, np.uint64, "x7")
        x10 = out(x10, np.uint64, "x10")
        _check(LIB.gl_edge_counts(self._h, first, count, t.ctypes.data_as(C.c_void_p),
                                  x7.ctypes.data_as(C.c_void_p), x10.ctypes.data_as(C.c_void_p)))
        return t, x7, x10

    def edge_counts_device(self):
        t, a, b = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(LIB.gl_edge_counts_device(self._h, C.byref(t), C.byref(a), C.byref(b)))
        return t.value, a.value, b.value


def local_three_counts(rec, n: int):
    """counts.cpp:113-120: (x3, x4, x5) of one EdgeMotifRecord / MicroRecord row;
    std::invalid_argument (InvalidArgument here) when n < 2."""
    if n < 2:
        raise InvalidArgument(-1, "local_three_counts needs n >= 2")
    t, su, sv = int(rec["t"]), int(rec["s_u"]), int(rec["s_v"])
    return t, su + sv, n - (su + sv + t) - 2


def version() -> str:
    return LIB.gl_version().decode()
