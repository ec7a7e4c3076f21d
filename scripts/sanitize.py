"""Small counts for compute-sanitizer runs (scripts/sanitize.sh):
python scripts/sanitize.py [rmat:<scale> | ba:<n>:<k> | recut] ...
(plain integers are RMAT scales; GL_SPARSE_BIG=all forces the windowed hash)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1608_05138_b200 as gl  # noqa: E402

for spec in sys.argv[1:] or ["14", "16"]:
    if spec == "recut":
        from test_gpu_parity import recut_graph
        pairs = recut_graph()
    elif spec.startswith("ba:"):
        _, n, k = spec.split(":")
        pairs = gl.generate_ba(int(n), int(k), seed=3)
    else:
        pairs = gl.generate_rmat(int(spec.split(":")[-1]), 16, seed=1)
    g = gl.Graph.build(pairs)
    r = g.count()
    print(spec, g.num_edges(), g.max_degree(), r.X[7], r.X[10], flush=True)
