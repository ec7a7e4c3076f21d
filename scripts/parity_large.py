"""Full parity at RMAT 18/19 on the GPU box (every micro record and X_1..X_17
vs the oracle's reference pipeline, 16 host threads; minutes of CPU time).
Usage: python scripts/parity_large.py  -- result kept in profiles/r1_parity_large.txt"""
import sys, time, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import paper_1608_05138_b200 as gl
from oracle import Oracle
for sc in [18, 19]:
    pairs = gl.generate_rmat(sc, 16, seed=100 + sc)
    t=time.time(); o = Oracle(pairs); X, orec = o.count(threads=16, micro=True); to=time.time()-t
    g = gl.Graph.build(pairs, 0); res = g.count(); rec = g.micro_records()
    print(sc, g.num_edges(), 'oracle s', round(to,1), 'X equal', res.X == X, 'micro equal', np.array_equal(rec, orec.view(gl.MICRO_DTYPE)), flush=True)
