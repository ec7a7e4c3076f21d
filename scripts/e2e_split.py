"""Split the e2e step (bench.py's e2e loop: gl_graph_build from pinned host
pairs, gl_count_edges into pinned buffers, graph freed) into build / count +
copy-out / close wall times, and the count's own per-phase device times."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1608_05138_b200 as gl  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
hp = gl.generate_rmat(scale, 16, seed=1)
pin = torch.from_numpy(hp.view(np.int64).reshape(-1)).pin_memory()
count = len(hp)
m0 = None
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = gl.Graph.build_host_ptr(pin.data_ptr(), count, 0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    m = g.num_edges()
    if m0 is None:
        m0 = m
        pt = torch.empty(m, dtype=torch.int32).pin_memory()
        p7 = torch.empty(m, dtype=torch.int64).pin_memory()
        p10 = torch.empty(m, dtype=torch.int64).pin_memory()
    t1b = time.perf_counter()
    res, _, _, _ = g.count_edges(pt.numpy().view(np.uint32), p7.numpy().view(np.uint64), p10.numpy().view(np.uint64))
    t2 = time.perf_counter()
    g.close()
    t3 = time.perf_counter()
    print(f"it {it}: build {1e3*(t1-t0):.1f} count+copy {1e3*(t2-t1b):.1f} close {1e3*(t3-t2):.1f} ms; "
          f"device phases {[round(x, 2) for x in res.ms]} launches {res.launches}", flush=True)
