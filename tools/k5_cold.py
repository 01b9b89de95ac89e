"""K5 single-launch ("cold") timing variants at M7B after one compress: the
L2 flushed by a 512 MB write (bench.py's flush), by a write then a 512 MB
read (no dirty lines left to write back), and each launch captured with its
flush in a CUDA graph (no host launch gap)."""
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
eng.compress(d_qw, d_k, d_v)
counts = eng.kept_counts.view(1, c["layers"]).cpu().numpy().reshape(-1)
by = np.mean([bench.decode_bytes_per_step(counts, s) for s in range(n_dec)])
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
rd = torch.empty(512 << 20, dtype=torch.uint8, device="cuda").fill_(1)
acc = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()


def run(mode):
    per = []
    for s in range(n_dec):
        flush.zero_()
        if mode == "write+read":
            acc.add_(rd.view(torch.int64).sum())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.decode_step(d_qd, d_k, d_v, s)
        b.record(st)
        per.append((a, b))
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in per]) * 1e3


for mode in ("write", "write+read", "write", "write+read"):
    t = run(mode)
    print(f"{mode:11s} mean {t.mean():6.2f} us  median {np.median(t):6.2f}  min {t.min():6.2f}  "
          f"{by / (t.mean() / 1e6) / 1e9:7.0f} GB/s avg bytes {by / 1e6:.1f} MB", flush=True)
