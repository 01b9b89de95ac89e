"""K1 with and without exact mode at the bench workload (reference generator
inputs) and with random Gaussian inputs: time, listed entries, overflow."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

c = bench.CFG
shape = Shape(1, c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["prompt_len"], c["tau"])
qw, qd, ks, vs = bench.synth_inputs(1, 0, c["tau"])
gen = (torch.from_numpy(qw).to(torch.bfloat16).cuda(), torch.from_numpy(ks).to(torch.bfloat16).cuda())
g = torch.Generator(device="cuda").manual_seed(0)
rnd = ((torch.randn(gen[0].shape, device="cuda", generator=g) * 2).to(torch.bfloat16),
       torch.randn(gen[1].shape, device="cuda", generator=g).to(torch.bfloat16))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name, (q, k) in (("generator", gen), ("randn", rnd)):
    for exact in (False, True):
        eng = VLCache(shape, exact=exact)
        ts = []
        for _ in range(8):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            eng.score_stats(q, k)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        extra = ""
        if exact:
            cnt = eng.exact_ws[:12].view(torch.int32).cpu().numpy()
            extra = f"  near-max listed {cnt[0]}, near-threshold listed {cnt[1]}, overflow {cnt[2]}"
        print(f"{name:9s} exact={exact!s:5s}: K1 {np.median(ts[2:]):.1f} us{extra}")

# per-kernel durations of one exact-mode call (CUPTI via torch.profiler)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

eng = VLCache(shape, exact=True)
eng.score_stats(*gen)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.score_stats(*gen)
    torch.cuda.synchronize()
for evt in prof.key_averages():
    if evt.device_time_total > 0:
        print(f"  {evt.key[:60]:60s} {evt.device_time_total:9.1f} us")
