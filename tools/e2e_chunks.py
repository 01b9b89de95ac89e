"""e2e step time of VLCache.run_from_host for different pipeline depths (chunks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

c = bench.CFG
m, n_dec = c["prompt_len"], c["n_out"] - 1
qw, qd, ks, vs = bench.synth_inputs(1, 0, c["tau"])
hp = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).pin_memory()  # noqa: E731
e = (hp(qw), hp(ks[:, :, :, :m]), hp(vs[:, :, :, :m]), hp(qd), hp(ks[:, :, :, m:m + n_dec]), hp(vs[:, :, :, m:m + n_dec]))
eng = VLCache(Shape(1, c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], m, c["tau"]), alpha=c["alpha"],
              decode_steps=n_dec)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
CASES = os.environ.get("E2E_CASES")   # "chunks,dec_chunks,early;..." (default: the dec_early sweep)
grid = ([tuple(int(x) for x in c.split(",")) for c in CASES.split(";")] if CASES
        else [(4, 8, e_) for e_ in (0, 1, 2, 3, 8)] * 2)
for chunks, dec_chunks, early in grid:
    ts = []
    for i in range(8):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.run_from_host(*e, chunks=chunks, dec_chunks=dec_chunks, dec_early=early)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.mean(ts[3:]))
    print(f"chunks {chunks} dec_chunks {dec_chunks} early {early}: {t:.3f} ms/step, {n_dec / t * 1e3:.0f} tok/s")
