"""One compress + a few decode steps at LLaVA-1.6-Mistral-7B shapes -- a short,
deterministic command for ncu captures.  Random bf16 inputs by default;
GEN=1: the bench's reference-generator inputs; EXACT=0: plain fp32 decisions.

  ncu --set full -k regex:decode_kernel -s 2 -c 1 -o prof python tools/profile_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

L, HQ, HKV, D, M, TAU, STEPS = 32, 32, 8, 128, 2960, 64, int(os.environ.get("STEPS", "4"))
B = int(os.environ.get("BATCH", "1"))
if os.environ.get("GEN") == "1":
    import bench

    dev = lambda a: torch.from_numpy(a).to(torch.bfloat16).cuda()  # noqa: E731
    q, qd, k, v = (dev(a) for a in bench.synth_inputs(B, 0, TAU))
else:
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.randn((B, L, HQ, TAU, D), device="cuda", generator=g) * 2).to(torch.bfloat16)
    k = torch.randn((B, L, HKV, M + STEPS, D), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((B, L, HKV, M + STEPS, D), device="cuda", generator=g).to(torch.bfloat16)
    qd = torch.randn((B, L, HQ, STEPS, D), device="cuda", generator=g).to(torch.bfloat16)
eng = VLCache(Shape(B, L, HQ, HKV, D, M, TAU), decode_steps=STEPS, exact=os.environ.get("EXACT", "1") == "1")
for rep in range(2):
    eng.compress(q, k, v)
    for s in range(STEPS):
        eng.decode_step(qd, k, v, s)
torch.cuda.synchronize()
print("ok", eng.kept_counts.sum().item())
