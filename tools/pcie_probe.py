"""Pinned host -> device copy bandwidth on this box (one 269 MB copy, and in
16 / 64 MB pieces on a side stream), to compare with the e2e step time."""
import torch

n = 269119488
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for piece in (n, 64 << 20, 16 << 20):
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record()
            for o in range(0, n, piece):
                d[o:o + piece].copy_(h[o:o + piece], non_blocking=True)
            b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = sorted(ts)[2]
    print(f"piece {piece >> 20} MB: {t:.3f} ms, {n / t / 1e6:.1f} GB/s")
