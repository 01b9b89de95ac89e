"""One prefill at M7B shapes (random bf16) -- a short command for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_23317_b200.prefill import prefill  # noqa: E402

L = int(os.environ.get("LAYERS", "4"))
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((1, L, 32, 2960, 128), device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn((1, L, 8, 2960, 128), device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn((1, L, 8, 2960, 128), device="cuda", generator=g).to(torch.bfloat16)
for _ in range(2):
    prefill(q, k, v, 2960)
torch.cuda.synchronize()
print("ok")
