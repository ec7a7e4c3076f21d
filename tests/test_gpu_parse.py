"""GPU: load_edge_list (graph.cpp:47-85) on the device (csrc/parse.cu) against
the reference parser's vectors (tests/golden/parser.json, made by the
reference's own parser) and against the host scanner on fuzzed texts: same
pairs, or the same parse_error line number and message."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

gl = pytest.importorskip("paper_1608_05138_b200")


def outcome(fn, text):
    try:
        return ("ok", fn(text).tolist())
    except gl.ParseError as e:
        return ("err", e.line, str(e))


def test_device_parser_reference_vectors(cuda_device):
    vecs = json.load(open(os.path.join(GOLDEN, "parser.json")))
    for name, v in vecs.items():
        got = outcome(lambda t: gl.parse_edge_list_device(t, cuda_device), v["text"])
        if v["pairs"] is None:
            assert got == ("err", v["err_line"], v["err"]), name
        else:
            assert got == ("ok", v["pairs"]), name


def _fuzz_text(rng):
    lines = []
    for _ in range(int(rng.integers(0, 40))):
        k = int(rng.integers(0, 14))
        sep = lambda: "".join(rng.choice([" ", "\t", "\r"], size=int(rng.integers(1, 3))))  # noqa: E731
        if k == 0:
            lines.append("")
        elif k == 1:
            lines.append(sep() if rng.random() < 0.5 else "")
        elif k == 2:
            lines.append("# comment " + str(int(rng.integers(0, 99))))
        elif k == 3:
            lines.append(("  " if rng.random() < 0.3 else "") + "%%MatrixMarket matrix coordinate")
        elif k == 4:
            lines.append("% other comment")
        elif k == 5:  # malformed tokens
            lines.append(str(int(rng.integers(0, 9))) + sep() + rng.choice(["x", "-1", "+2", "1.5", "0x10", ""]))
        elif k == 6:  # wrong token counts
            lines.append(sep().join(str(int(x)) for x in rng.integers(0, 100, size=int(rng.choice([1, 3, 4])))))
        elif k == 7:  # u64 edge values (2^64 - 1 ok, 2^64 overflow)
            lines.append(f"{2**64 - 1}{sep()}{rng.choice(['0', str(2**64), '18446744073709551615'])}")
        elif k == 8:  # leading zeros, trailing separators
            lines.append(f"007{sep()}0{sep() if rng.random() < 0.5 else ''}")
        else:
            a, b = (int(x) for x in rng.integers(0, 10**12, size=2))
            lines.append((sep() if rng.random() < 0.2 else "") + f"{a}{sep()}{b}" + (sep() if rng.random() < 0.3 else ""))
    text = "\n".join(lines)
    if rng.random() < 0.5:
        text += "\n"
    return text


def test_device_parser_fuzz_vs_host(cuda_device):
    rng = np.random.default_rng(77)
    n_err = 0
    for i in range(400):
        text = _fuzz_text(rng)
        host = outcome(gl.load_edge_list, text)
        dev = outcome(lambda t: gl.parse_edge_list_device(t, cuda_device), text)
        assert dev == host, (i, text)
        n_err += host[0] == "err"
    assert 50 < n_err < 390  # both outcomes exercised


def test_build_text_equals_build_pairs(cuda_device):
    pairs = gl.generate_rmat(12, 16, seed=4)
    text = "# rmat-12\n" + "".join(f"{a}\t{b}\n" for a, b in pairs.tolist())
    g1 = gl.Graph.build_text(text, cuda_device)
    g2 = gl.Graph.build(pairs, cuda_device)
    assert g1.count().X == g2.count().X
    assert np.array_equal(g1.micro_records(), g2.micro_records())
    with pytest.raises(gl.ParseError) as ei:
        gl.Graph.build_text(text + "1 2 3\n", cuda_device)
    assert ei.value.line == len(pairs) + 2


@pytest.mark.slow
def test_device_parser_rmat20_text(cuda_device):
    """configs[1]'s 16.8M edges as text: the device parse returns the pairs exactly."""
    pairs = gl.generate_rmat(20, 16, seed=1)
    text = "\n".join(f"{a} {b}" for a, b in pairs.tolist()).encode()
    got = gl.parse_edge_list_device(text, cuda_device)
    assert np.array_equal(got, pairs)
