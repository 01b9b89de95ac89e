"""K5 at the bench workload (M7B shapes, generator recipe drawn on the device):
99-step decode graph (L2 flushed before each replay) and a cold single step,
plus a checksum of the last step's output against the first library run
(gpurun_out/k5_ref.npy): VLC_LIB_PATH=exp_libs/x.so python tools/k5_quick.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402
from paper_2410_23317_b200.trace import GenSpec, device_synthetic  # noqa: E402

L, HQ, HKV, D, M, TAU, N = 32, 32, 8, 128, 2960, 64, 99
B = int(os.environ.get("BATCH", "1"))
spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M,
               post_vision_len=TAU, decode_len=N, seed=0)
qw, qd, k, v = device_synthetic(spec, B, TAU)
ALPHA = float(os.environ.get("ALPHA", "0.1"))
eng = VLCache(Shape(B, L, HQ, HKV, D, M, TAU), decode_steps=N, alpha=ALPHA)
eng.compress(qw, k, v)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps, cold=True):
    ts = []
    for _ in range(reps):
        if cold:
            flush.zero_()
            flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts[2:]))


g = timed(lambda: eng.decode(qd, k, v, graph=True), 7)
out = eng.out.float().cpu().numpy()
c50 = timed(lambda: eng.decode_step(qd, k, v, 50), 9)
ref = f"gpurun_out/k5_ref_{B}_{ALPHA}.npy"
if not os.path.exists(ref):
    np.save(ref, out)
err = float(np.abs(out - np.load(ref)).max())
print(f"{os.path.basename(os.environ.get('VLC_LIB_PATH', 'in-tree')):18s} B={B} a={ALPHA} graph {g / N:6.2f} us/step  "
      f"cold step50 {c50:6.2f} us  max|out-ref| {err:.2e}")
