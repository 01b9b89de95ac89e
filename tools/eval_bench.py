"""Row f4 measurement: the evaluation report (hit rates of a policy + modality
contribution / coverage) on a VLM-shaped trace, B200 path vs the CPU oracle
restatement of the reference's numpy + compiled-kernel path on the host cores.

  python tools/eval_bench.py [layers] [decode_rows]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_23317_b200 as V  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2410_23317_b200.trace import AttentionTrace, GenSpec, generate_trace, round_to_bf16  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
NDEC = int(sys.argv[2]) if len(sys.argv) > 2 else 8
spec = GenSpec(num_layers=L, num_query_heads=32, num_kv_heads=8, head_dim=128, prompt_len=2960,
               post_vision_len=64, decode_len=NDEC, seed=0)
tr, _ = generate_trace(spec)
tr = AttentionTrace(header=tr.header, layout=tr.layout, queries=[round_to_bf16(x) for x in tr.queries],
                    keys=[round_to_bf16(x) for x in tr.keys])
h = tr.header
m, seq, k = h.prompt_len, h.seq_len, 296
pol = {"vlcache": V.PostVision()}

V.build_report(tr, pol, k=k)   # warm-up (library load, graph of allocations)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = V.build_report(tr, pol, k=k)
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t0

# CPU: the same report through the oracle (reference kernels restated in C, numpy above)
t0 = time.perf_counter()
win = V.EvalWindow.for_header(h)
cpu_rows = []
for l in range(L):
    for q in range(h.num_query_heads):
        kv = tr.kv_head_for(q)
        scores = O.stats_tiled(tr.queries[l][q, m - 64:m], tr.keys[l][kv, :m], m - 64, 0.01, 128)[2][:m]
        orow = O.causal_probs(tr.queries[l][q, m:m + 1], tr.keys[l][kv, :m], m, m)
        cpu_rows.append(O.hit_rate(scores, orow, k, k))
cpu_mod = []
for l in range(L):
    for mod in V.MODALITIES:
        c, v = [], []
        for q in range(h.num_query_heads):
            probs = O.causal_probs(tr.queries[l][q, m:seq], tr.keys[l][tr.kv_head_for(q), :seq], m, seq)
            c.append(O.filtered_share(probs, m, tr.layout.indices(mod), 0.01))
            v.append(O.topk_share(probs, m, tr.layout.indices(mod), win.top_k))
        cpu_mod.append((float(np.mean(c)), float(np.mean(v))))
t_cpu = time.perf_counter() - t0

same_hits = [r["hit_rate"] for r in rep.hit_rate_rows] == cpu_rows
mod_ok = all(abs(r["contribution"] - c) <= 1e-6 * max(1.0, abs(c)) and r["coverage"] == v
             for r, (c, v) in zip(rep.modality_rows, cpu_mod))
print(f"eval report L{L} Hq32 Hkv8 d128 m{m} decode_rows{NDEC} k{k}: GPU {t_gpu * 1e3:.1f} ms, "
      f"CPU oracle {t_cpu * 1e3:.1f} ms (1 thread), x{t_cpu / t_gpu:.1f}; hit rates identical: {same_hits}; "
      f"modality rows agree: {mod_ok}")
