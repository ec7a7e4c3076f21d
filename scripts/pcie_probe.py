"""Host<->device copy bandwidth of the box (pinned host memory), for reading
the e2e numbers: python scripts/pcie_probe.py"""
import torch

for mb in (64, 256, 1024):
    n = mb << 20
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        print(f"{name} {mb:5d} MiB: {ms:7.2f} ms  {n / ms / 1e6:6.1f} GB/s", flush=True)
