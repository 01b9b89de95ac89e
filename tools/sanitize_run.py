"""A short run of every kernel of the path for compute-sanitizer (tools/sanitize.sh):
TOY shapes, exact and plain K1, K2-K4, 3 decode steps eager then as a graph
(programmatic dependent launch chain), the prefill and the float32 seam."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_23317_b200 import _kernels  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402
from paper_2410_23317_b200.prefill import prefill  # noqa: E402
from paper_2410_23317_b200.trace import GenSpec, device_synthetic  # noqa: E402

# SAN_L / SAN_HKV: enough (layer, KV head) slots (>= the SM count) to take K5's
# early-release path as well
L, HKV = int(os.environ.get("SAN_L", "2")), int(os.environ.get("SAN_HKV", "2"))
HQ, D, M, TAU, N = 4 * HKV, 128, 624, 32, int(os.environ.get("SAN_N", "3"))   # SAN_N > 16: K5's periodic late release
spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M, post_vision_len=TAU,
               decode_len=N, seed=0)
qw, qd, k, v = device_synthetic(spec, 1, TAU)
for exact in (True, False):
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), decode_steps=N, exact=exact)
    eng.compress(qw, k, v)
    eng.decode(qd, k, v, graph=False)
    eng.decode(qd, k, v, graph=True)
    torch.cuda.synchronize()
    eng.check()
g = torch.Generator(device="cuda").manual_seed(1)
qp = torch.randn((1, L, HQ, M, D), device="cuda", generator=g).to(torch.bfloat16)
out, rmax, rsum = prefill(qp, k, v, M)
rng = np.random.default_rng(0)
_kernels.stats_tiled(rng.standard_normal((40, 64)).astype(np.float32),
                     rng.standard_normal((128, 64)).astype(np.float32), 88, 0.01, 33)
_kernels.decode_step(rng.standard_normal((4, 64)).astype(np.float32),
                     rng.standard_normal((100, 64)).astype(np.float32),
                     rng.standard_normal((100, 64)).astype(np.float32))
torch.cuda.synchronize()
print("sanitize run ok")
