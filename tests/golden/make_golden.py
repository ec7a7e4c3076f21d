"""Regenerate tests/golden/*.json from the REFERENCE's own code.

Runs the reference sources compiled here (oracle/_ref/libgraphlet_ref.so,
built from /root/reference/proj/src by oracle/Makefile) on small graphs and
records the inputs, the global counts X1..X17 and the per-edge MicroRecords
(counts.cpp:122-136).  Run in the build container (where /root/reference
exists):  python tests/golden/make_golden.py
The fixtures are committed; tests never need /root/reference at run time.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import RefLib  # noqa: E402


def micro_digest(rec):
    return hashlib.sha256(np.ascontiguousarray(rec).tobytes()).hexdigest()


def er(n, p, seed):
    rng = np.random.default_rng(seed)
    return [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < p]


def ba(n, k, seed):
    rng = np.random.default_rng(seed)
    ends, out = [], []
    for a in range(k + 1):
        for b in range(a + 1, k + 1):
            out.append((a, b)); ends += [a, b]
    for v in range(k + 1, n):
        picked = set()
        while len(picked) < k:
            picked.add(ends[rng.integers(len(ends))])
        for w in sorted(picked):
            out.append((v, w)); ends += [v, w]
    return out


def rmat(scale, ef, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(ef << scale):
        r = c = 0
        for _ in range(scale):
            x = rng.random(); r <<= 1; c <<= 1
            if x < 0.57: pass
            elif x < 0.76: c |= 1
            elif x < 0.95: r |= 1
            else: r |= 1; c |= 1
        out.append((r, c))
    return out


CASES = {
    "k4": [(1, 2), (1, 3), (1, 4), (2, 3), (2, 4), (3, 4)],
    "c4": [(1, 2), (2, 3), (3, 4), (4, 1)],
    "star_k13": [(10, 1), (10, 2), (10, 3)],
    "diamond": [(1, 2), (1, 3), (1, 4), (2, 3), (2, 4)],
    "path_p4": [(1, 2), (2, 3), (3, 4)],
    "c5": [(1, 2), (2, 3), (3, 4), (4, 5), (5, 1)],
    "k5": [(a, b) for a in range(5) for b in range(a + 1, 5)],
    "single_edge": [(7, 9)],
    "loops_dups_gaps": [(1, 1), (1, 2), (2, 1), (1000000000000, 2), (5, 5), (2, 3), (3, 1000000000000),
                        (18446744073709551615, 3)],
    "only_self_loops": [(4, 4), (9, 9)],
    "empty": [],
    "er_25_p03": er(25, 0.3, 7),
    "er_40_p05": er(40, 0.5, 11),
    "ba_60_k4": ba(60, 4, 5),
    "ba_400_k6": ba(400, 6, 1),
    "rmat_s9_ef8": rmat(9, 8, 3),
}


def main():
    for name, pairs in CASES.items():
        arr = np.asarray(pairs, dtype=np.uint64).reshape(-1, 2)
        r = RefLib(arr)
        X, rec = r.count(threads=1, micro=True)
        v, u, vl, ul = r.orient()
        doc = {
            "generator": "tests/golden/make_golden.py (reference sources via oracle/_ref)",
            "pairs": [[int(a), int(b)] for a, b in arr],
            "n": r.n, "m": r.m,
            "X": [str(x) for x in X],
            "micro_sha256": micro_digest(rec),
            "edge_labels_sha256": hashlib.sha256(vl.tobytes() + ul.tobytes()).hexdigest(),
        }
        if r.m <= 300:
            doc["micro"] = [[int(x) for x in row] for row in rec.tolist()]
        if r.n <= 40:
            doc["brute_force"] = [str(x) for x in r.brute_force(cap=64)]
        with open(os.path.join(HERE, name + ".json"), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        print(name, r.n, r.m, X[7], X[10])
    # parser vectors from the reference parser (graph.cpp:47-85)
    texts = {
        "basic": "1 2\n2 3\n",
        "mm": "# c\n%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n1 2\n1 3\n",
        "bad_token": "1 x\n",
        "three_tokens": "1 2\n3 4 5\n",
        "crlf_tabs": "  1\t2\r\n\r\n# x\n% y\n3 4",
        "one_token": "\n\n7\n",
        "overflow": "18446744073709551616 1\n",
        "max": "18446744073709551615 0\n",
        "sign": "-1 2\n",
        "plus": "+1 2\n",
        "empty": "",
        "mm_short_banner": "%%Matrix\n1 2\n",
        "mm_then_comment": "%%MatrixMarket x\n% c\n5 5 5\n1 2\n",
    }
    out = {}
    for k, t in texts.items():
        pairs, line, err = RefLib.parse(t)
        out[k] = {"text": t, "pairs": None if pairs is None else pairs.tolist(), "err_line": line,
                  "err": err}
    with open(os.path.join(HERE, "parser.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
