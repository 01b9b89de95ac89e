"""Per-kernel device time of one bench step (compress + 99 decode steps) at M7B,
L2 flushed before the step (torch.profiler / CUPTI; not a bench number)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

c = bench.CFG
qw, qd, ks, vs = bench.synth_inputs(1, 0, c["tau"])
dev = lambda a: torch.from_numpy(a).to(torch.bfloat16).cuda()  # noqa: E731
d_qw, d_qd, d_k, d_v = dev(qw), dev(qd), dev(ks), dev(vs)
eng = VLCache(Shape(1, c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["prompt_len"], c["tau"]),
              alpha=c["alpha"], decode_steps=c["n_out"] - 1)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def step():
    eng.score_stats(d_qw, d_k)
    eng.allocate(); eng.select(); eng.gather(d_k, d_v)
    eng.decode(d_qd, d_k, d_v, graph=True)


for _ in range(3):
    flush.zero_(); step()
torch.cuda.synchronize()
flush.zero_()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
tot = 0.0
for evt in sorted(prof.key_averages(), key=lambda e: -e.device_time_total):
    if evt.device_time_total > 0:
        tot += evt.device_time_total
        print(f"{evt.key[:70]:70s} {evt.count:5d} {evt.device_time_total:9.1f} us")
print(f"total kernel time {tot:.1f} us")
