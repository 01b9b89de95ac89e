"""K1 time at the bench workload (M7B shapes, the reference generator's recipe
drawn on the device), exact mode off and on, L2 flushed before each call:
VLC_LIB_PATH=exp_libs/x.so python tools/k1_quick.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402
from paper_2410_23317_b200.trace import GenSpec, device_synthetic  # noqa: E402

L, HQ, HKV, D, M, TAU = (int(x) for x in os.environ.get("K1_SHAPE", "32,32,8,128,2960,64").split(","))
spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M,
               post_vision_len=TAU, decode_len=1, seed=0)
qw, qd, k, v = device_synthetic(spec, 1, TAU)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flops = 2 * D * HQ * (TAU * (M - TAU) + TAU * (TAU + 1) // 2) * L
out = []
for exact in (False, True):
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), exact=exact)
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.score_stats(qw, k)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    t = float(np.median(ts[2:]))
    chk = (int(eng.below_head.sum().item()), float(eng.col_partial.double().sum().item()))
    out.append(f"exact={int(exact)} {t:6.1f} us ({flops / t / 1e6:.0f} TFLOP/s) below {chk[0]} mass {chk[1]:.6f}")
print(os.path.basename(os.environ.get("VLC_LIB_PATH", "in-tree")), " | ".join(out))
