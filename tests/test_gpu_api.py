"""GPU: boundary behaviour of the C-ABI -- the reference's error semantics,
call-sequence errors and caller-buffer validation (no counting parity here)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

gl = pytest.importorskip("paper_1608_05138_b200")


def test_vertex_id_space_is_invalid_argument(cuda_device, monkeypatch):
    """graph.cpp:103-104: >= 2^32-1 distinct labels -> std::invalid_argument
    (GL_ERR_INVALID).  GL_TEST_VERTEX_LIMIT lowers the bound to reach it."""
    monkeypatch.setenv("GL_TEST_VERTEX_LIMIT", "4")
    gl.Graph.build(np.array([[0, 1], [1, 2], [2, 0]], np.uint64), cuda_device)  # n = 3 < 4
    with pytest.raises(gl.InvalidArgument, match="vertex id space"):
        gl.Graph.build(np.array([[0, 1], [1, 2], [2, 3]], np.uint64), cuda_device)


def test_edge_id_space_is_invalid_argument(cuda_device, monkeypatch):
    """eid_t is u32 (common.hpp:14): m >= 2^32-1 is refused as invalid."""
    monkeypatch.setenv("GL_TEST_EDGE_LIMIT", "3")
    gl.Graph.build(np.array([[0, 1], [1, 2]], np.uint64), cuda_device)
    with pytest.raises(gl.InvalidArgument, match="edge id space"):
        gl.Graph.build(np.array([[0, 1], [1, 2], [2, 0]], np.uint64), cuda_device)


def test_slot_limit_is_invalid_argument(cuda_device, monkeypatch):
    """Device counting needs 2m < 2^32 adjacency slots: refused at load time
    with the reference's invalid_argument (GL_TEST_SLOT_LIMIT lowers 2^32-1)."""
    monkeypatch.setenv("GL_TEST_SLOT_LIMIT", "5")
    gl.Graph.build(np.array([[0, 1], [1, 2]], np.uint64), cuda_device)  # 2m = 4 < 6
    with pytest.raises(gl.InvalidArgument, match="counting limit"):
        gl.Graph.build(np.array([[0, 1], [1, 2], [2, 0]], np.uint64), cuda_device)  # 2m = 6


def test_degree_limit_is_overflow(cuda_device, monkeypatch):
    """The cycle windows count runs in 24 bits: max degree >= 2^24 is refused
    (GL_ERR_OVERFLOW) rather than miscounted (GL_TEST_DEGREE_LIMIT lowers it)."""
    star = np.array([[0, i] for i in range(1, 200)] + [[1, 2], [3, 4], [2, 3]], np.uint64)
    g = gl.Graph.build(star, cuda_device)
    monkeypatch.setenv("GL_TEST_DEGREE_LIMIT", "150")
    with pytest.raises(gl.CountOverflowError, match="max degree"):
        g.count()
    monkeypatch.delenv("GL_TEST_DEGREE_LIMIT")
    assert g.count().X[1] == g.num_edges()


def test_call_sequence_errors(cuda_device):
    import torch
    g = gl.Graph.build(gl.generate_rmat(10, 8, seed=2), cuda_device)
    st = torch.cuda.Stream()
    buf = torch.empty(2 * g.partials_len(1), dtype=torch.int64, device="cuda")
    with pytest.raises(gl.StateError):
        g.count_mid(buf.data_ptr(), st.cuda_stream)
    g.count_begin(0, 1, buf.data_ptr(), st.cuda_stream)
    g.count_mid(buf.data_ptr(), st.cuda_stream)
    with pytest.raises(gl.StateError, match="twice"):
        g.count_mid(buf.data_ptr(), st.cuda_stream)
    C = g.count_finish(buf.data_ptr(), 0, g.num_edges(), st.cuda_stream)
    assert gl.global_from_unrestricted(C, g.num_vertices(), g.num_edges()) == g.count().X
    # re-entry: begin twice on different streams before mid gives the same counts
    st2 = torch.cuda.Stream()
    g.count_begin(0, 1, buf.data_ptr(), st.cuda_stream)
    g.count_begin(0, 1, buf.data_ptr(), st2.cuda_stream)
    g.count_mid(buf.data_ptr(), st2.cuda_stream)
    C2 = g.count_finish(buf.data_ptr(), 0, g.num_edges(), st2.cuda_stream)
    assert C2 == C


def test_edge_counts_validates_caller_buffers(cuda_device):
    g = gl.Graph.build(gl.generate_rmat(9, 8, seed=4), cuda_device)
    g.count()
    m = g.num_edges()
    t, x7, x10 = g.edge_counts()
    with pytest.raises(ValueError):
        g.edge_counts(0, m, t=np.zeros(m, np.int64))  # wrong dtype
    with pytest.raises(ValueError):
        g.edge_counts(0, m, x7=np.zeros(m - 1, np.uint64))  # too short
    with pytest.raises(ValueError):
        g.edge_counts(0, m, x10=np.zeros(2 * m, np.uint64)[::2])  # not contiguous
    # first + count wraps around 2^64: refused by the C range check itself
    assert gl.LIB.gl_edge_counts(g._h, 5, 2**64 - 3, None, None, None) == -1
    t2, a, b = g.edge_counts(0, m, t=np.zeros(m + 5, np.uint32))
    assert np.array_equal(t2[:m], t)
    rec = np.zeros(m, gl.MICRO_DTYPE)
    assert np.array_equal(g.micro_records(out=rec), g.micro_records())


def test_count_sharded_world1_on_default_stream(cuda_device):
    """dist.count_sharded without a stream runs on its own stream ordered after
    the caller's (never the library's unordered NULL-stream mapping)."""
    from paper_1608_05138_b200.dist import count_sharded, sharded_step
    import torch
    g = gl.Graph.build(gl.generate_rmat(11, 16, seed=9), cuda_device)
    X, (b, e) = count_sharded(g, 0, 1)
    assert X == g.count().X and (b, e) == (0, g.num_edges())
    p = torch.empty(2 * g.partials_len(1), dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError, match="stream"):
        sharded_step(g, p, 0, 1, torch.cuda.default_stream())


def test_cpp_mirror_on_device(cuda_device, tmp_path):
    """include/graphlet_b200.hpp on the device: graph.hpp:56-79 accessors and
    process_edge_hash records (tests/cpp_gpu_check.cpp)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "cpp_gpu_check"
    libdir = os.path.dirname(gl.lib_path())
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp_gpu_check.cpp"), "-o", str(exe), "-L", libdir,
                    "-lgraphlet_b200", f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert out.strip() == "ok"


def test_edge_motif_records_match_reference_pipeline(cuda_device):
    """EdgeMotifRecord rows (t, s_u, s_v, x7, x10, work_units) equal the
    reference's own process_edge_hash records (oracle/_ref: the reference's
    sources compiled in place) on RMAT / BA graphs."""
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle as O
    for pairs in (gl.generate_rmat(10, 8, seed=3), gl.generate_ba(3000, 5, seed=2)):
        g = gl.Graph.build(pairs, cuda_device)
        g.count()
        rec = g.edge_motif_records()
        if not O.ref_available():
            pytest.skip("oracle/_ref not built (it ships with the snapshot from the build container)")
        ref = O.RefLib(pairs).edge_records(0)
        got = np.stack([rec[f].astype(np.uint64) for f in ("t", "s_u", "s_v", "x7", "x10", "work_units")], 1)
        assert np.array_equal(got, ref)
        assert np.array_equal(rec["edge_id"], np.arange(g.num_edges(), dtype=np.uint32))
        one = g.process_edge_hash(7)
        assert tuple(int(one[f]) for f in ("t", "x7", "x10", "work_units")) == tuple(int(x) for x in ref[7, [0, 3, 4, 5]])
        assert gl.local_three_counts(one, g.num_vertices())[0] == int(one["t"])


def test_count_edges_equals_count_then_copy(cuda_device):
    """gl_count_edges (t/x7 copied out during the cycle pass) == gl_count +
    gl_edge_counts, also into caller buffers, and again on a reused graph."""
    g = gl.Graph.build(gl.generate_rmat(12, 16, seed=6), cuda_device)
    ref = g.count()
    t, x7, x10 = (a.copy() for a in g.edge_counts())
    for _ in range(2):
        res, t2, x72, x102 = g.count_edges()
        assert res.X == ref.X and res.C == ref.C
        assert np.array_equal(t2, t) and np.array_equal(x72, x7) and np.array_equal(x102, x10)
    m = g.num_edges()
    bt, b7, b10 = np.zeros(m + 3, np.uint32), np.zeros(m, np.uint64), np.zeros(m, np.uint64)
    g.count_edges(bt, b7, b10)
    assert np.array_equal(bt[:m], t) and np.array_equal(b7, x7) and np.array_equal(b10, x10)
    with pytest.raises(ValueError):
        g.count_edges(t=np.zeros(m, np.int64))
