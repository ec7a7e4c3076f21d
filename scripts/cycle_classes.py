"""Print the cycle-pass top classes (GL_DEBUG) of a few graphs, and the
windowed-hash window/re-cut counts from the instrumented library:
GRAPHLET_B200_LIB=libgraphlet_b200_prof.so GL_SPARSE_BIG=all python scripts/cycle_classes.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GL_DEBUG"] = "1"
import paper_1608_05138_b200 as gl  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import recut_graph  # noqa: E402

cases = [("ba", 60000, 6, 3), ("ba", 200000, 4, 11), ("ba", 30000, 12, 5), ("recut", 0, 0, 1)]
for kind, n, k, seed in cases:
    g = gl.Graph.build(recut_graph(seed) if kind == "recut" else gl.generate_ba(n, k, seed=seed))
    buf = (C.c_ulonglong * 64)()
    prof = hasattr(gl.LIB, "gl_debug_cycle_profile") and "prof" in os.environ.get("GRAPHLET_B200_LIB", "")
    if prof:
        gl.LIB.gl_debug_cycle_profile(buf, 1)
    g.count()
    if prof:
        gl.LIB.gl_debug_cycle_profile(buf, 0)
        print(f"{kind}({n},{k},{seed}): windowed-hash windows {buf[30]} wedges {buf[31]} re-cuts {buf[29]}", flush=True)
