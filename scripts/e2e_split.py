"""Split the e2e step (bench.py's e2e loop) into build / count / D2H wall times."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1608_05138_b200 as gl
from paper_1608_05138_b200.dist import sharded_step

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
hp = gl.generate_rmat(scale, 16, seed=1)
pin = torch.from_numpy(hp.view(np.int64).reshape(-1)).pin_memory()
count = len(hp)
stream = torch.cuda.Stream()
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = gl.Graph.build_host_ptr(pin.data_ptr(), count, 0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    m = g.num_edges()
    p = torch.empty(2 * g.partials_len(1), dtype=torch.int64, device="cuda")
    X, _ = sharded_step(g, p, 0, 1, stream)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    pt = torch.empty(m, dtype=torch.int32).pin_memory()
    p7 = torch.empty(m, dtype=torch.int64).pin_memory()
    p10 = torch.empty(m, dtype=torch.int64).pin_memory()
    t2b = time.perf_counter()
    g.edge_counts(0, m, pt.numpy().view(np.uint32), p7.numpy().view(np.uint64), p10.numpy().view(np.uint64))
    t3 = time.perf_counter()
    g.close()
    del p
    t4 = time.perf_counter()
    print(f"it {it}: build {1e3*(t1-t0):.1f} count {1e3*(t2-t1):.1f} pin-alloc {1e3*(t2b-t2):.1f} d2h {1e3*(t3-t2b):.1f} close {1e3*(t4-t3):.1f} ms ms={g.last_timings() if hasattr(g,'last_timings') else ''}", flush=True)
