"""Full parity on the GPU box: every micro record and X_1..X_17 vs the
oracle's reference pipeline (16 host threads; minutes of CPU time), for the
default cycle-kind choice and with the sparse-big choice forced both ways
(GL_SPARSE_BIG=all / off).
Usage: python scripts/parity_large.py [rmat:18 rmat:20:1 ba:500000:8 ...] (rmat:<scale>[:<seed>])
(default rmat:18 rmat:19); results are kept in profiles/*parity_large*.txt"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
import paper_1608_05138_b200 as gl  # noqa: E402
from oracle import Oracle  # noqa: E402

specs = sys.argv[1:] or ["rmat:18", "rmat:19"]
for spec in specs:
    kind, *args = spec.split(":")
    if kind == "rmat":
        sc = int(args[0])
        pairs = gl.generate_rmat(sc, 16, seed=int(args[1]) if len(args) > 1 else 100 + sc)
    else:
        n, k = int(args[0]), int(args[1])
        pairs = gl.generate_ba(n, k, seed=7)
    t = time.time()
    o = Oracle(pairs)
    X, orec = o.count(threads=16, micro=True)
    to = time.time() - t
    for mode in ("default", "all", "off"):
        if mode == "default":
            os.environ.pop("GL_SPARSE_BIG", None)
        else:
            os.environ["GL_SPARSE_BIG"] = mode
        g = gl.Graph.build(pairs, 0)
        res = g.count()
        rec = g.micro_records()
        print(spec, g.num_edges(), 'oracle s', round(to, 1), 'cycle kinds', mode, 'X equal', res.X == X,
              'micro equal', np.array_equal(rec, orec.view(gl.MICRO_DTYPE)), flush=True)
        del g
