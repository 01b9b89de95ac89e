"""Compress once, then replay the 99-step decode graph a few times (for ncu
--graph-profiling node --cache-control none: warm-L2 K5 launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
for rep in range(int(os.environ.get("REPS", "3"))):
    eng.compress(d_qw, d_k, d_v)
    eng.decode(d_qd, d_k, d_v, graph=True)
torch.cuda.synchronize()
print("ok")
