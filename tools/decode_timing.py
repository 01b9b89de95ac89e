"""Time K5 at M7B shapes: 99 steps as a CUDA graph (warm) and cold single launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

L, HQ, HKV, D, M, TAU, STEPS = 32, 32, 8, 128, 2960, 64, 99
g = torch.Generator(device="cuda").manual_seed(0)
q = (torch.randn((1, L, HQ, TAU, D), device="cuda", generator=g) * 2).to(torch.bfloat16)
k = torch.randn((1, L, HKV, M + STEPS, D), device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn((1, L, HKV, M + STEPS, D), device="cuda", generator=g).to(torch.bfloat16)
qd = torch.randn((1, L, HQ, STEPS, D), device="cuda", generator=g).to(torch.bfloat16)
ALPHA = float(os.environ.get("ALPHA", "0.1"))
eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), decode_steps=STEPS, alpha=ALPHA)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for rep in range(6):
    eng.compress(q, k, v)
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.decode(qd, k, v, graph=True)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
cold = []
eng.compress(q, k, v)
for s in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.decode_step(qd, k, v, s)
    b.record()
    torch.cuda.synchronize()
    cold.append(a.elapsed_time(b))
print(f"alpha={ALPHA} {os.environ.get('VLC_LIB_PATH', 'default')}: graph 99 steps {np.median(ts[2:]) * 1e3:.0f} us "
      f"({np.median(ts[2:]) * 1e3 / 99:.2f} us/step); cold launch {np.median(cold) * 1e3:.2f} us; "
      f"kept {eng.kept_counts.sum().item()} max_k {eng.kept_counts.max().item()} min_k {eng.kept_counts.min().item()}")
