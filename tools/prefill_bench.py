"""f2 measurement: causal prefill at LLaVA-1.6-Mistral-7B shapes (L32 Hq32 Hkv8 d128,
m = 2960) on the B200 (vlc_prefill, events, L2 flushed), tensor-core flops vs the
measured bf16 peak, and the reference's float32 numpy prefill (bench.py:196-234,
restated in oracle/) on one layer of the host, extrapolated."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_23317_b200.prefill import prefill  # noqa: E402

B, L, HQ, HKV, D, M = 1, 32, 32, 8, 128, 2960
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((B, L, HQ, M, D), device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn((B, L, HKV, M, D), device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn((B, L, HKV, M, D), device="cuda", generator=g).to(torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(8):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    prefill(q, k, v, M)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts[2:]))
causal = M * (M + 1) // 2
flops = 4 * D * causal * HQ * L * B            # QK^T + PV, the attention's own work
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
tc = peak.get("bf16_tflops")
line = {"prefill_ms": ms, "attention_tflops": flops / ms / 1e9, "flops": flops,
        "note": "one pass (online softmax, lazy O rescale in TMEM): QK^T and PV once per tile"}
if tc:
    line["frac_of_bf16_peak"] = flops / ms / 1e9 / tc
# row f2's fusion at the bench workload (generator inputs): prefill + K1 column pass
# on the prefill's statistics + K2-K4, vs prefill followed by the two-pass compress
import bench  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

c = bench.CFG
qa, _, ka, va = bench.synth_inputs(1, 0, M)
dev = lambda x: torch.from_numpy(x).to(torch.bfloat16).cuda()  # noqa: E731
qa, ka, va = dev(qa), dev(ka), dev(va)
shape = Shape(1, L, HQ, HKV, D, M, c["tau"])
eng = VLCache(shape, alpha=c["alpha"], decode_steps=c["n_out"] - 1)
qwin = qa[:, :, :, M - c["tau"]:].contiguous()


def timed(fn, reps=6):
    out = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out[1:]))


line["fused_prefill_compress_ms"] = timed(lambda: eng.prefill_compress(qa, ka, va))
line["prefill_then_compress_ms"] = timed(lambda: (prefill(qa, ka, va, M, stats=False), eng.compress(qwin, ka, va)))
# CPU: the reference algorithm (float32 numpy, tile 128) on one layer
if os.environ.get("CPU", "1") == "1":
    from oracle import oracle as O

    qh, kh, vh = (t[0, 0].float().cpu().numpy() for t in (q, k, v))
    t0 = time.perf_counter()
    O.prefill_layer(qh, kh, vh, M, 128)
    line["cpu_ms_per_prompt_extrapolated"] = (time.perf_counter() - t0) * 1e3 * L
    line["cpu_sample"] = "1 of 32 layers, numpy float32 (host BLAS threads), x32"
print(json.dumps(line))
