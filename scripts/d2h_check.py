import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1608_05138_b200 as gl
from paper_1608_05138_b200.dist import _tensor_from_ptr
g = gl.Graph.build(gl.generate_rmat(20, 16, seed=1), 0)
g.count()
m = g.num_edges()
pt = torch.empty(m, dtype=torch.int32).pin_memory(); p7 = torch.empty(m, dtype=torch.int64).pin_memory(); p10 = torch.empty(m, dtype=torch.int64).pin_memory()
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g.edge_counts(0, m, pt.numpy().view(np.uint32), p7.numpy().view(np.uint64), p10.numpy().view(np.uint64))
    t1 = time.perf_counter()
    tp, x7p, x10p = g.edge_counts_device()
    a = _tensor_from_ptr(tp, m, torch.int32, torch.device('cuda', 0)); b = _tensor_from_ptr(x7p, m, torch.int64, torch.device('cuda', 0)); c = _tensor_from_ptr(x10p, m, torch.int64, torch.device('cuda', 0))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    pt.copy_(a); p7.copy_(b); p10.copy_(c); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"gl_edge_counts {1e3*(t1-t0):.2f} ms   torch copies {1e3*(t3-t2):.2f} ms   bytes {m*20/1e6:.0f} MB")
