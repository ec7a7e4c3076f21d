"""CPU: the C-ABI library itself -- exports, parser, generators, count algebra,
error behaviour.  No device compute is called here."""
import json
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

import paper_1608_05138_b200 as gl
from oracle import Oracle, global_from_unrestricted as or_global

HEADER = os.path.join(ROOT, "include", "graphlet_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gl_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(gl.LIB, n)]
    assert not missing, missing


def test_library_has_no_oracle_or_cpu_fallback():
    out = subprocess.run(["nm", "-D", "--defined-only", gl.lib_path()], capture_output=True, text=True).stdout
    assert " or_" not in out and "ref_" not in out
    deps = subprocess.run(["ldd", gl.lib_path()], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "graphlet_ref" not in deps
    # the kernels are real sm_100a SASS
    sass = subprocess.run(["cuobjdump", "--list-elf", gl.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in sass


def test_version():
    assert "sm_100a" in gl.version()


# ------------------------------------------------------------------ parser

def test_parser_matches_reference_vectors():
    vecs = json.load(open(os.path.join(GOLDEN, "parser.json")))
    for name, v in vecs.items():
        if v["pairs"] is None:
            with pytest.raises(gl.ParseError) as ei:
                gl.load_edge_list(v["text"])
            assert ei.value.line == v["err_line"], name
            assert str(ei.value) == v["err"], name
        else:
            got = gl.load_edge_list(v["text"])
            assert got.tolist() == v["pairs"], name


def test_parser_spec_examples_and_file(tmp_path):
    assert gl.load_edge_list("1 2\n2 3\n").tolist() == [[1, 2], [2, 3]]
    txt = "# c\n%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n1 2\n1 3\n"
    assert gl.load_edge_list(txt).tolist() == [[1, 2], [1, 3]]
    with pytest.raises(gl.ParseError) as ei:
        gl.load_edge_list("1 x\n")
    assert ei.value.line == 1
    assert gl.load_edge_list("").shape == (0, 2)
    p = tmp_path / "g.txt"
    p.write_text("5 6\n6 7\n")
    assert gl.load_edge_list_file(str(p)).tolist() == [[5, 6], [6, 7]]
    with pytest.raises(OSError):
        gl.load_edge_list_file(str(tmp_path / "missing.txt"))


# ------------------------------------------------------------------ generators

def test_generators_deterministic():
    a = gl.generate_rmat(10, 8, seed=3)
    assert a.shape == (8 << 10, 2) and np.array_equal(a, gl.generate_rmat(10, 8, seed=3))
    assert not np.array_equal(a, gl.generate_rmat(10, 8, seed=4))
    assert a.max() < (1 << 10)
    g = gl.generate_gnm(100, 1000, seed=1)
    assert g.shape == (1000, 2)
    canon = {(min(x, y), max(x, y)) for x, y in g.tolist()}
    assert len(canon) == 1000 and all(x != y for x, y in canon)
    assert np.array_equal(g, gl.generate_gnm(100, 1000, seed=1))
    with pytest.raises(ValueError):
        gl.generate_gnm(10, 46, seed=1)
    b = gl.generate_ba(500, 4, seed=1)
    assert b.shape[0] == 10 + (500 - 5) * 4
    assert Oracle(b).m == b.shape[0]  # BA never repeats an edge


def test_rmat_skew():
    """Fig. 1 qualitative: power-law degrees on the RMAT workload family."""
    o = Oracle(gl.generate_rmat(14, 16, seed=1))
    deg = o.degrees()
    assert deg.max() > 50 * np.median(deg)


# ------------------------------------------------------------------ algebra

def test_global_algebra_matches_oracle_and_rejects_corruption():
    pairs = gl.generate_ba(200, 3, seed=2)
    o = Oracle(pairs)
    X, rec = o.count(micro=True)
    from test_oracle import unrestricted_from_micro
    Cs = unrestricted_from_micro(rec, o.n, o.m)
    assert gl.global_from_unrestricted(Cs, o.n, o.m) == X == or_global(Cs, o.n, o.m)
    bad = list(Cs)
    bad[3] += 1
    with pytest.raises(gl.CountConsistencyError, match="X3"):
        gl.global_from_unrestricted(bad, o.n, o.m)
    bad = list(Cs)
    bad[10] += 2
    with pytest.raises(gl.CountConsistencyError, match="X10"):
        gl.global_from_unrestricted(bad, o.n, o.m)


def test_global_algebra_128bit():
    n = 2**32 - 2  # C(n,4) needs ~126 bits
    X = gl.global_from_unrestricted([0] * 17, n, 0)
    import math
    assert X[2] == math.comb(n, 2) and X[6] == math.comb(n, 3) and X[17] == math.comb(n, 4)


def test_graph_names():
    assert gl.graphlet_name(7) == "4-clique" and gl.graphlet_name(12) == "4-path"
    assert gl.graphlet_name(99) == "?"


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(gl.CudaError):
        gl.Graph.build([(1, 2), (2, 3)])


def test_cpp_api_mirror_host_calls(tmp_path):
    """include/graphlet_b200.hpp (C++ mirror of the reference API) compiles
    against the product library; its host-only calls behave like the reference."""
    exe = tmp_path / "cpp_api_check"
    libdir = os.path.dirname(gl.lib_path())
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp_api_check.cpp"), "-o", str(exe), "-L", libdir,
                    "-lgraphlet_b200", f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert out.strip() == "ok"


def test_cli_usage_and_errors(tmp_path):
    tool = os.path.join(os.path.dirname(gl.lib_path()), "graphlet_count")
    assert subprocess.run([tool], capture_output=True).returncode == 2
    assert subprocess.run([tool, "count", str(tmp_path / "missing.txt")], capture_output=True).returncode == 1
    bad = tmp_path / "bad.txt"
    bad.write_text("1 2\n3 x\n")
    r = subprocess.run([tool, "count", str(bad)], capture_output=True, text=True)
    assert r.returncode == 2 and "line 2" in r.stderr
