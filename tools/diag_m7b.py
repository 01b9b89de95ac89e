"""Diagnostics at the bench workload (M7B, reference generator inputs): per-layer
kept counts and K1 / K5 timings, cold L2 (flush before each launch) and warm."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

c = bench.CFG
n_dec = c["n_out"] - 1
qw, qd, ks, vs = bench.synth_inputs(1, 0, c["tau"])
dev = lambda a: torch.from_numpy(a).to(torch.bfloat16).cuda()  # noqa: E731
d_qw, d_qd, d_k, d_v = dev(qw), dev(qd), dev(ks), dev(vs)
eng = VLCache(Shape(1, c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["prompt_len"], c["tau"]),
              alpha=c["alpha"], p=c["p"], recent_frac=c["recent"], decode_steps=n_dec)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10, cold=True):
    ts = []
    for _ in range(reps):
        if cold:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts[2:]))


k1 = timed(lambda: eng.score_stats(d_qw, d_k))
eng.compress(d_qw, d_k, d_v)
counts = eng.kept_counts.view(-1).cpu().numpy()
print("kept per layer:", counts.tolist())
print(f"sum {counts.sum()} mean {counts.mean():.1f} max {counts.max()} min {counts.min()}")
k5c = timed(lambda: eng.decode_step(d_qd, d_k, d_v, 50))
k5w = timed(lambda: eng.decode_step(d_qd, d_k, d_v, 50), cold=False)
g99 = timed(lambda: eng.decode(d_qd, d_k, d_v, graph=True), reps=6)
by = bench.decode_bytes_per_step(counts, 50)
print(f"K1 cold {k1:.1f} us ({bench.k1_flops(1) / k1 / 1e6:.0f} TFLOP/s)")
print(f"K5 step50 cold {k5c:.2f} us ({by / k5c / 1e3:.0f} GB/s), warm {k5w:.2f} us; graph99 {g99:.0f} us "
      f"({g99 / 99:.2f} us/step)")
