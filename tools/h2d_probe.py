"""H2D / D2H bandwidth of pinned and pageable host buffers on the GPU box."""
import time
import torch

n = 528 * 1024 * 1024 // 8
dev = torch.device("cuda", 0)
d = torch.empty(n, dtype=torch.int64, device=dev)
for kind in ("pinned", "pageable"):
    h = torch.ones(n, dtype=torch.int64)
    if kind == "pinned":
        h = h.pin_memory()
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"{kind} H2D 528 MB: {ms:.2f} ms = {n * 8 / ms / 1e6:.1f} GB/s")
    # split into 4 chunks on 2 streams
    ss = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    s.record()
    for r in range(5):
        for i in range(4):
            with torch.cuda.stream(ss[i % 2]):
                d[i * n // 4:(i + 1) * n // 4].copy_(h[i * n // 4:(i + 1) * n // 4], non_blocking=True)
    for st in ss:
        torch.cuda.current_stream().wait_stream(st)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"{kind} H2D 4 chunks / 2 streams: {ms:.2f} ms = {n * 8 / ms / 1e6:.1f} GB/s")
