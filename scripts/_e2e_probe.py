import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1608_05138_b200 as gl
hp = gl.generate_rmat(20, 16, seed=1)
pin = torch.from_numpy(hp.view(np.int64).reshape(-1)).pin_memory()
for it in range(4):
    g = gl.Graph.build_host_ptr(pin.data_ptr(), len(hp), 0)
    r1 = g.count(); r2 = g.count(); r3, *_ = g.count_edges(); r4, *_ = g.count_edges()
    print(it, "count1", [round(x,2) for x in r1.ms], "count2", [round(x,2) for x in r2.ms], "edges1", [round(x,2) for x in r3.ms], "edges2", [round(x,2) for x in r4.ms], flush=True)
    g.close()
