"""One exact-mode and one plain K1 call at M7B on generator inputs (after two
warm-ups each), for `ncu --metrics gpu__time_duration.sum` launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402
from paper_2410_23317_b200.trace import GenSpec, device_synthetic  # noqa: E402

L, HQ, HKV, D, M, TAU = (int(x) for x in os.environ.get("K1_SHAPE", "32,32,8,128,2960,64").split(","))
spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M,
               post_vision_len=TAU, decode_len=1, seed=0)
qw, qd, k, v = device_synthetic(spec, 1, TAU)
torch.cuda.synchronize()
for exact in (True, False):
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), exact=exact)
    for _ in range(3):
        eng.score_stats(qw, k)
    torch.cuda.synchronize()
