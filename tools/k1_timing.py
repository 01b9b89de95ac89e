"""Time K1 (score_stats) alone at M7B shapes (cold L2 before each launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

L, HQ, HKV, D, M, TAU = 32, 32, 8, 128, 2960, 64
g = torch.Generator(device="cuda").manual_seed(0)
q = (torch.randn((1, L, HQ, TAU, D), device="cuda", generator=g) * 2).to(torch.bfloat16)
k = torch.randn((1, L, HKV, M, D), device="cuda", generator=g).to(torch.bfloat16)
eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for rep in range(12):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.score_stats(q, k)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
flops = 2 * D * HQ * (TAU * (M - TAU) + TAU * (TAU + 1) // 2) * L
t = float(np.median(ts[2:]))
print(f"{os.environ.get('VLC_LIB_PATH', 'default')}: K1 {t:.1f} us  {flops / t / 1e6:.0f} TFLOP/s "
      f"({flops / t / 1e6 / 1644.3:.3f} of measured bf16 peak)")
