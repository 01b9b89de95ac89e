"""Compress once, then replay the 99-step decode graph a few times (for ncu
--graph-profiling node --cache-control none: K5 launches as the bench runs
them).  BATCH=8 replicates the prompt into distinct buffers like bench.py's
HBM probe (k5_hbm_probe): the cache then exceeds L2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

c = bench.CFG
n_dec = c["n_out"] - 1
B = int(os.environ.get("BATCH", "1"))
qw, qd, ks, vs = bench.synth_inputs(1, 0, c["tau"])
dev = lambda a: torch.from_numpy(a).to(torch.bfloat16).cuda().expand(B, *a.shape[1:]).contiguous()  # noqa: E731
d_qw, d_qd, d_k, d_v = dev(qw), dev(qd), dev(ks), dev(vs)
eng = VLCache(Shape(B, c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["prompt_len"], c["tau"]),
              alpha=c["alpha"], p=c["p"], recent_frac=c["recent"], decode_steps=n_dec)
for rep in range(int(os.environ.get("REPS", "3"))):
    eng.compress(d_qw, d_k, d_v)
    eng.decode(d_qd, d_k, d_v, graph=True)
torch.cuda.synchronize()
print("ok")
