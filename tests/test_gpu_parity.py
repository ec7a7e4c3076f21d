"""GPU parity: the sm_100a pipeline vs the oracle / reference goldens, through the C-ABI.

Bit-exact is the bar everywhere: global X_1..X_17 (128-bit) and every
per-edge MicroRecord field (counts.cpp:122-136).
"""
import hashlib
import math
import os

import numpy as np
import pytest

from conftest import golden_cases, load_golden

pytestmark = pytest.mark.gpu

gl = pytest.importorskip("paper_1608_05138_b200")
from oracle import Oracle  # noqa: E402  (test infrastructure)

THREADS = max(1, min(32, os.cpu_count() or 1))


def gpu_count(pairs, device=0):
    g = gl.Graph.build(np.asarray(pairs, dtype=np.uint64).reshape(-1, 2), device)
    res = g.count()
    rec = g.micro_records() if g.num_edges() else np.zeros(0, gl.MICRO_DTYPE)
    return g, res, rec


def assert_partitions(X, n):
    assert X[1] + X[2] == math.comb(n, 2)
    assert sum(X[3:7]) == math.comb(n, 3)
    assert sum(X[7:18]) == math.comb(n, 4)


@pytest.mark.parametrize("name", golden_cases())
def test_golden(cuda_device, name):
    d = load_golden(name)
    g, res, rec = gpu_count(d["pairs"], cuda_device)
    assert g.num_vertices() == d["n"] and g.num_edges() == d["m"]
    assert [str(x) for x in res.X] == d["X"]
    assert hashlib.sha256(np.ascontiguousarray(rec).tobytes()).hexdigest() == d["micro_sha256"]
    if "micro" in d:
        assert rec.tolist() == [tuple(r) for r in d["micro"]]
    v, u = g.orient_edges()
    lab = g.labels()
    got = hashlib.sha256(lab[v].astype(np.uint64).tobytes() + lab[u].astype(np.uint64).tobytes()).hexdigest()
    assert got == d["edge_labels_sha256"]
    assert_partitions(res.X, d["n"])


def _er(n, p, seed):
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    mask = rng.random(len(iu[0])) < p
    return np.stack([iu[0][mask], iu[1][mask]], 1).astype(np.uint64)


def test_random_corpus_vs_oracle(cuda_device):
    """ER n in [5,60], p in {.1,.3,.5,.8,.95} and BA graphs: X and micro exact."""
    rng = np.random.default_rng(2024)
    for k in range(120):
        if k % 3 == 2:
            pairs = gl.generate_ba(int(rng.integers(5, 200)), int(rng.integers(1, 8)), seed=k)
        else:
            pairs = _er(int(rng.integers(5, 61)), [0.1, 0.3, 0.5, 0.8, 0.95][k % 5], k)
        o = Oracle(pairs)
        X, orec = o.count(micro=True)
        g, res, rec = gpu_count(pairs, cuda_device)
        assert res.X == X, k
        assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE)), k
        if o.n <= 25:
            assert res.X == o.brute_force()


@pytest.mark.parametrize("scale,ef", [(8, 16), (10, 8), (12, 16), (13, 16)])
def test_rmat_vs_oracle(cuda_device, scale, ef):
    pairs = gl.generate_rmat(scale, ef, seed=scale)
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))
    assert_partitions(res.X, o.n)


@pytest.mark.parametrize("n,k", [(5000, 5), (20000, 10)])
def test_ba_vs_oracle(cuda_device, n, k):
    pairs = gl.generate_ba(n, k, seed=1)
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))


def test_gnm_config0_vs_oracle(cuda_device):
    """BASELINE configs[0]: G(n=10k, m=100k)."""
    pairs = gl.generate_gnm(10000, 100000, seed=1)
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert g.num_edges() == 100000
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))


def test_edge_cases(cuda_device):
    # empty input
    g, res, rec = gpu_count(np.zeros((0, 2), np.uint64), cuda_device)
    assert g.num_vertices() == 0 and res.X == [0] * 18
    # only self loops: 3 isolated vertices
    g, res, rec = gpu_count([(5, 5), (6, 6), (7, 7), (7, 7)], cuda_device)
    assert g.num_vertices() == 3 and g.num_edges() == 0
    assert res.X[2] == 3 and res.X[6] == 1 and sum(res.X) == 4
    # empty graph on n=5 (SPEC oracle example): X2=10, X6=10, X17=5
    g, res, rec = gpu_count([(i, i) for i in range(5)], cuda_device)
    assert res.X[2] == 10 and res.X[6] == 10 and res.X[17] == 5
    # duplicates in both directions + label gaps + max label
    pairs = [(2**64 - 1, 0), (0, 2**64 - 1), (3, 3), (10**15, 0), (0, 10**15), (10**15, 2**64 - 1)]
    o = Oracle(pairs)
    X, orec = o.count(micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert res.X == X and np.array_equal(rec, orec.view(gl.MICRO_DTYPE))
    assert sorted(g.labels().tolist()) == sorted({0, 3, 10**15, 2**64 - 1})


@pytest.mark.parametrize("n", [5, 12, 40, 600, 800, 1000, 1200])
def test_complete_graphs_closed_form(cuda_device, n):
    """K_n: X3=C(n,3), X7=C(n,4); per edge t=n-2, x7=C(n-2,2), x10=0.
    |U(a)| = n-1-a covers every H-pass class: K_800/K_1000 the xl class in
    shared memory, K_1200 (|U(0)| = 1199 > 1088) its global-scratch path."""
    pairs = [(a, b) for a in range(n) for b in range(a + 1, n)]
    g, res, rec = gpu_count(pairs, cuda_device)
    X = res.X
    assert X[1] == math.comb(n, 2) and X[3] == math.comb(n, 3) and X[7] == math.comb(n, 4)
    assert all(X[i] == 0 for i in (2, 4, 5, 6, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17))
    assert (rec["t"] == n - 2).all() and (rec["x7"] == math.comb(n - 2, 2)).all() and (rec["x10"] == 0).all()


def test_hpass_smem_limit_across_graphs(cuda_device):
    """The xl H-pass kernel's dynamic shared-memory limit is a per-process
    attribute: a graph needing less (K_800, xl class in shared memory) must
    not lower it under a later graph needing more (K_1200, the whole opt-in
    size).  The round-2 regression: K_1200 -> K_800 -> K_1200 failed its
    last launch with 'invalid argument'."""
    for n in (1200, 800, 1200):
        pairs = [(a, b) for a in range(n) for b in range(a + 1, n)]
        g, res, rec = gpu_count(pairs, cuda_device)
        assert res.X[7] == math.comb(n, 4) and (rec["t"] == n - 2).all()


def test_cycles_and_stars_closed_form(cuda_device):
    for n in (5, 9, 100):
        g, res, rec = gpu_count([(i, (i + 1) % n) for i in range(n)], cuda_device)
        assert res.X[10] == 0 and res.X[3] == 0
    g, res, rec = gpu_count([(0, 1), (1, 2), (2, 3), (3, 0)], cuda_device)
    assert res.X[10] == 1 and (rec["x10"] == 1).all()
    for n in (3, 10, 3000):
        g, res, rec = gpu_count([(0, i) for i in range(1, n + 1)], cuda_device)
        assert res.X[11] == math.comb(n, 3) and res.X[4] == math.comb(n, 2)


def test_big_top_windows(cuda_device):
    """Hubs with > 512 wedges and ids > 32768 exercise k_cycle_big's multi-window path."""
    pairs = gl.generate_ba(60000, 6, seed=3)
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))


def test_multiwindow_half_counters(cuda_device):
    """n > 65536: big tops span several 64K-id windows of 16-bit counters."""
    pairs = gl.generate_ba(200000, 4, seed=11)
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert g.num_vertices() > 65536
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))


@pytest.mark.parametrize("mode", ["all", "off"])
@pytest.mark.parametrize("n,k,seed", [(60000, 6, 3), (200000, 4, 11), (30000, 12, 5)])
def test_sparse_big_windowed_hash(cuda_device, monkeypatch, mode, n, k, seed):
    """GL_SPARSE_BIG=all routes every big top (> 16384 wedges, |L(a)| < 65536)
    through the windowed block hash (KIND 3: c windows cut by wedge count and
    re-cut when over the cap); =off keeps them on dense windows."""
    monkeypatch.setenv("GL_SPARSE_BIG", mode)
    pairs = gl.generate_ba(n, k, seed=seed)
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))


def recut_graph(seed=1):
    """Top A (degree 500) over 100 b's (degree ~331) whose wedges crowd the low
    end of a wide c range: 1500 ids of degree 20 (C1) adjacent to 20 b's each
    hold 30000 wedges, then 58500 ids of degree 20-21 (a circulant C2, 3000 of
    them with one b) hold 3000.  A's first windowed-hash window (~30K ids by the
    uniform estimate) holds ~30K wedges > kHashWinMax (27306) and is re-cut."""
    rng = np.random.default_rng(seed)
    nb, n1, n2 = 100, 1500, 58500
    A = 0
    bs = np.arange(1, 1 + nb)
    c1 = np.arange(1 + nb, 1 + nb + n1)
    c2 = np.arange(1 + nb + n1, 1 + nb + n1 + n2)
    leaves = np.arange(c2[-1] + 1, c2[-1] + 1 + 400)
    e = [np.stack([np.full(nb, A), bs], 1), np.stack([np.full(400, A), leaves], 1)]
    for c in c1:
        e.append(np.stack([rng.choice(bs, 20, replace=False), np.full(20, c)], 1))
    i = np.arange(n2)
    for d in range(1, 11):
        e.append(np.stack([c2[i], c2[(i + d) % n2]], 1))
    pick = rng.choice(n2, 3000, replace=False)
    e.append(np.stack([rng.choice(bs, 3000), c2[pick]], 1))
    return np.concatenate(e).astype(np.uint64)


def test_sparse_big_recut(cuda_device, monkeypatch):
    """Windowed-hash re-cut path (see recut_graph) against the oracle."""
    monkeypatch.setenv("GL_SPARSE_BIG", "all")
    pairs = recut_graph()
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))


def test_hub_full_counters(cuda_device):
    """A hub with |L(a)| >= 65536 switches k_cycle_big to 32-bit counters
    (32K-id windows); leaves carry a sparse random graph plus a second hub so
    the hub's wedges close 4-cycles through many windows."""
    rng = np.random.default_rng(7)
    leaves = 70000
    hub = [(0, i) for i in range(1, leaves + 1)]
    hub2 = [(leaves + 1, int(i)) for i in rng.choice(np.arange(1, leaves + 1), 3000, replace=False)]
    ab = rng.integers(1, leaves + 1, size=(20000, 2))
    pairs = np.array(hub + hub2 + [tuple(map(int, r)) for r in ab], dtype=np.uint64)
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert g.max_degree() >= 65536
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))


def _piece_wedges(g, pieces):
    """Exact wedges a-b-c (b in L(a), c in N(b), c < a) with c in [lo, hi) of
    every piece row (a, lo, hi, est), from the CSR on the host."""
    off, adj = g.csr()
    off = off.astype(np.int64)
    n = g.num_vertices()
    row = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    key = row * n + adj.astype(np.int64)  # ascending: rows by id, each row ascending
    out = np.zeros(len(pieces), np.int64)
    for i, (a, lo, hi, _) in enumerate(pieces.astype(np.int64)):
        r = adj[off[a]:off[a + 1]].astype(np.int64)
        b = r[r < a]
        hi = min(hi, a)
        if hi > lo and len(b):
            out[i] = int((np.searchsorted(key, b * n + hi) - np.searchsorted(key, b * n + lo)).sum())
    return out


@pytest.mark.parametrize("graph,cap,sparse", [("ba60k", 3000, None), ("ba60k", 3000, "all"), ("ba200k", 4000, None),
                                              ("rmat13", 2000, None), ("rmat13", 2000, "all"), ("ba200k", 4000, "all")])
def test_cycle_pieces(cuda_device, monkeypatch, graph, cap, sparse):
    """Heavy windowed tops split into c-range pieces (GL_PIECE_WEDGES forces a
    small piece cap): counts stay bit-exact, the pieces of each top tile
    [0, a) without gaps or overlap, and a split top's pieces share its wedges."""
    monkeypatch.setenv("GL_PIECE_WEDGES", str(cap))
    if sparse:
        monkeypatch.setenv("GL_SPARSE_BIG", sparse)
    if graph == "hub":
        rng = np.random.default_rng(7)
        leaves = 70000
        hub = [(0, i) for i in range(1, leaves + 1)]
        hub2 = [(leaves + 1, int(i)) for i in rng.choice(np.arange(1, leaves + 1), 3000, replace=False)]
        ab = rng.integers(1, leaves + 1, size=(20000, 2))
        pairs = np.array(hub + hub2 + [tuple(map(int, r)) for r in ab], dtype=np.uint64)
    elif graph == "rmat13":
        pairs = gl.generate_rmat(13, 16, seed=13)
    else:
        n, k, seed = (60000, 6, 3) if graph == "ba60k" else (200000, 4, 11)
        pairs = gl.generate_ba(n, k, seed=seed)
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))
    P = g.cycle_pieces()
    P = P[P[:, 0] != 0xFFFFFFFF]  # empty pieces (coinciding cut points on the window grid)
    tops, counts = np.unique(P[:, 0], return_counts=True)
    assert counts.max() > 1, "no top was split"
    for a in tops[counts > 1]:
        rows = P[P[:, 0] == a]
        rows = rows[np.argsort(rows[:, 1], kind="stable")]
        assert rows[0, 1] == 0 and rows[-1, 2] == a
        assert np.array_equal(rows[1:, 1], rows[:-1, 2])  # contiguous tiling of [0, a)
    w = _piece_wedges(g, P)
    split = np.isin(P[:, 0], tops[counts > 1])
    # the pieces of a split top hold exactly its wedges
    whole = _piece_wedges(g, np.stack([tops, np.zeros_like(tops), tops, tops], 1))
    for a, tot in zip(tops[counts > 1], whole[counts > 1]):
        assert int(w[P[:, 0] == a].sum()) == int(tot)
    if sparse == "all":
        # windowed-hash tops cut at the quantiles of 2048 sampled wedges stay
        # near the cap (dense tops cut on their window grid: a window is the
        # smallest piece there)
        assert w[split].max() <= 3 * max(cap, int(P[split, 3].max()))


@pytest.mark.parametrize("graph,sparse,world,piece", [("rmat12", None, 2, None), ("ba60k", None, 2, None),
                                                      ("ba60k", "off", 2, None), ("ba60k", "all", 2, None),
                                                      ("ba60k", "all", 3, None), ("ba60k", None, 3, 2000),
                                                      ("rmat12", "all", 2, 1500)])
def test_sharded_equals_single(cuda_device, monkeypatch, graph, sparse, world, piece):
    """world=2/3 sharding emulated on one GPU: begin per rank, sum partial rows,
    finish per shard, sum unrestricted -> identical macro and micro (BA 60k
    with GL_SPARSE_BIG=all: the windowed-hash tops are split across ranks;
    with a piece cap: the c-range pieces of one top land on different ranks)."""
    import torch
    if sparse:
        monkeypatch.setenv("GL_SPARSE_BIG", sparse)
    if piece:
        monkeypatch.setenv("GL_PIECE_WEDGES", str(piece))
    pairs = gl.generate_rmat(12, 16, seed=5) if graph == "rmat12" else gl.generate_ba(60000, 6, seed=3)
    g = gl.Graph.build(pairs, cuda_device)
    full = g.count()
    full_rec = g.micro_records()
    plen = g.partials_len(world)
    parts, tris = [], []
    # every library call and every torch op on one stream, as in dist.sharded_step
    # (the library's own stream is non-blocking: torch's default stream would race it)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for rank in range(world):
            buf = torch.empty(2 * plen, dtype=torch.int64, device="cuda")
            g.count_begin(rank, world, buf.data_ptr(), st.cuda_stream)
            ptr, m = g.triangle_counts_device()
            tris.append(_copy_u32(ptr, m))
            parts.append(buf)
        # all-reduce of t (emulated), then each rank's share of the triangle sums
        tsum = sum(tris[1:], tris[0])
        for rank in range(world):
            g.count_begin(rank, world, parts[rank].data_ptr(), st.cuda_stream)
            ptr, m = g.triangle_counts_device()
            _write_u32(ptr, tsum)
            g.count_mid(parts[rank].data_ptr(), st.cuda_stream)
        total = sum(parts[1:], parts[0])
        from paper_1608_05138_b200.dist import shard_range
        Csum = [0] * 17
        recs = []
        for rank in range(world):
            b, e = shard_range(g.num_edges(), world, rank)
            shard = total[2 * b:2 * e].contiguous()
            Cr = g.count_finish(shard.data_ptr(), b, e, st.cuda_stream)
            Csum = [x + y for x, y in zip(Csum, Cr)]
            recs.append(g.micro_records(b, e - b))
    torch.cuda.synchronize()
    assert gl.global_from_unrestricted(Csum, g.num_vertices(), g.num_edges()) == full.X
    assert Csum == full.C
    assert np.array_equal(np.concatenate(recs), full_rec)


def _copy_u32(ptr, m):
    from paper_1608_05138_b200.dist import _tensor_from_ptr
    import torch
    return _tensor_from_ptr(ptr, m, torch.int32, torch.device("cuda", 0)).clone()


def _write_u32(ptr, src):
    from paper_1608_05138_b200.dist import _tensor_from_ptr
    import torch
    _tensor_from_ptr(ptr, src.numel(), torch.int32, torch.device("cuda", 0)).copy_(src)


def test_device_generated_graph_matches_host(cuda_device):
    import torch
    scale, ef = 11, 16
    host = gl.generate_rmat(scale, ef, seed=9)
    d = torch.empty(2 * (ef << scale), dtype=torch.int64, device="cuda")
    gl.generate_rmat_device(scale, ef, d.data_ptr(), cuda_device, seed=9)
    assert np.array_equal(d.cpu().numpy().view(np.uint64).reshape(-1, 2), host)
    g1 = gl.Graph.build_device(d.data_ptr(), ef << scale, cuda_device)
    g2 = gl.Graph.build(host, cuda_device)
    assert g1.count().X == g2.count().X


@pytest.mark.slow
@pytest.mark.parametrize("scale", [16, 17])
def test_rmat_full_parity_larger(cuda_device, scale):
    """Every micro record and X_1..X_17 vs the oracle's per-edge hash pipeline
    (the reference algorithm) at RMAT 16/17: hub tops, every cycle-kernel kind,
    several degree-tier windows, both block H-pass classes."""
    pairs = gl.generate_rmat(scale, 16, seed=100 + scale)
    o = Oracle(pairs)
    X, orec = o.count(threads=THREADS, micro=True)
    g, res, rec = gpu_count(pairs, cuda_device)
    assert res.X == X
    assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))


@pytest.mark.slow
def test_rmat20_properties_and_sample(cuda_device):
    """BASELINE configs[1] at full size: size-independent properties plus a
    sampled per-edge comparison with the oracle's hash pipeline."""
    pairs = gl.generate_rmat(20, 16, seed=1)
    g = gl.Graph.build(pairs, cuda_device)
    res = g.count()
    n, m = g.num_vertices(), g.num_edges()
    assert_partitions(res.X, n)
    t, x7, x10 = g.edge_counts()
    assert int(t.astype(np.uint64).sum()) == 3 * res.X[3]
    assert int(x7.sum()) == 6 * res.X[7]
    assert int(x10.sum()) == 4 * res.X[10]
    o = Oracle(pairs)
    rng = np.random.default_rng(0)
    ids = np.sort(rng.choice(m, size=300, replace=False)).astype(np.uint64)
    ref = o.edges_hash(ids)
    assert np.array_equal(ref[:, 0], t[ids].astype(np.uint64))
    assert np.array_equal(ref[:, 3], x7[ids])
    assert np.array_equal(ref[:, 4], x10[ids])


def test_cli_count_spec_examples(tmp_path):
    """SPEC cli cmd_count examples through the C++ driver: K4 -> "X7":"1";
    --micro on C4 -> 4 rows with x10 = 1; every golden graph's X matches."""
    import json
    import subprocess
    tool = os.path.join(os.path.dirname(gl.lib_path()), "graphlet_count")
    k4 = tmp_path / "k4.txt"
    k4.write_text("".join(f"{a} {b}\n" for a in range(4) for b in range(a + 1, 4)))
    doc = json.loads(subprocess.run([tool, "count", str(k4)], capture_output=True, text=True, check=True).stdout)
    assert doc["counts"]["X7"] == "1" and doc["n"] == 4 and doc["m"] == 6
    c4 = tmp_path / "c4.txt"
    c4.write_text("0 1\n1 2\n2 3\n3 0\n")
    micro = tmp_path / "micro.csv"
    subprocess.run([tool, "count", str(c4), "--micro", str(micro)], check=True, capture_output=True)
    rows = micro.read_text().strip().splitlines()
    assert rows[0].startswith("edge_id,") and len(rows) == 5
    assert all(r.split(",")[5] == "1" for r in rows[1:])
    for name in golden_cases():
        d = load_golden(name)
        f = tmp_path / f"{name}.txt"
        f.write_text("".join(f"{a} {b}\n" for a, b in d["pairs"]))
        if not d["pairs"]:
            continue
        doc = json.loads(subprocess.run([tool, "count", str(f)], capture_output=True, text=True,
                                        check=True).stdout)
        assert [doc["counts"][f"X{i}"] for i in range(1, 18)] == d["X"][1:], name


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("spec", ["rmat:13", "ba:60000:6:3"])
def test_sharded_ranks_share_gpu(cuda_device, tmp_path, world, spec):
    """The multi-rank path end to end: `world` processes (torchrun, gloo, all on
    cuda:0) each count their cost-balanced share, exchange t / partial rows /
    128-bit sums, and finalise their edge shard; the shards' micro records and
    X equal the single-process count."""
    import json
    import subprocess
    import sys
    from _dist_worker import make_pairs
    pairs = make_pairs(gl, spec)
    g, res, rec = gpu_count(pairs, cuda_device)
    worker = os.path.join(os.path.dirname(__file__), "_dist_worker.py")
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                    "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), worker, str(tmp_path),
                    spec], check=True, timeout=600, capture_output=True)
    shards, xs = [], []
    for r in range(world):
        shards.append(np.load(tmp_path / f"rank{r}.npy"))
        xs.append(json.load(open(tmp_path / f"rank{r}.json"))["X"])
    assert all(x == [str(v) for v in res.X] for x in xs)
    assert np.array_equal(np.concatenate(shards), rec)


@pytest.mark.parametrize("exact", ["1", "0"])
def test_record_list_modes(cuda_device, monkeypatch, exact):
    """H-edge record list filled by exact reservations after phase 2
    (GL_TL_EXACT=1, the large-graph mode) or by C(k,2) up-front reservations
    (=0): bit-exact either way, including the big-k path (K_1200: k = 1199 >
    1088, records kept as SoA) and the warp / block classes (RMAT-13, BA)."""
    monkeypatch.setenv("GL_TL_EXACT", exact)
    for pairs in (gl.generate_rmat(13, 16, seed=21), gl.generate_ba(20000, 10, seed=4)):
        o = Oracle(pairs)
        X, orec = o.count(threads=THREADS, micro=True)
        g, res, rec = gpu_count(pairs, cuda_device)
        assert res.X == X
        assert np.array_equal(rec, orec.view(gl.MICRO_DTYPE))
    n = 1200
    g, res, rec = gpu_count([(a, b) for a in range(n) for b in range(a + 1, n)], cuda_device)
    assert res.X[7] == math.comb(n, 4) and (rec["x10"] == 0).all() and (rec["x7"] == math.comb(n - 2, 2)).all()
