import sys
sys.path.insert(0, ".")
import paper_1608_05138_b200 as gl
for s in [int(x) for x in sys.argv[1:]] or [14, 16]:
    g = gl.Graph.build(gl.generate_rmat(s, 16, seed=1))
    r = g.count()
    print(s, g.num_edges(), g.max_degree(), r.X[7], r.X[10], r.ms, flush=True)
