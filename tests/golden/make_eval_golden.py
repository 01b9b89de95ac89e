"""Golden vectors of the reference's evaluation path.

Run here (where /root/reference is mounted):  python tests/golden/make_eval_golden.py
Builds and imports the reference exactly as make_golden.py does and records
oracle_scores, dense_attention_rows, contribution, coverage, cache_hit_rate and
build_report on bf16-rounded generator traces (the "bf16-in" convention: the
same values feed K1 on the B200, so policy scores agree too).  Writes
tests/golden/eval_golden.npz + eval_report.json; the GPU box never reads
/root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import bf16_round, load_reference  # noqa: E402

# reference tests/conftest.py:7-21 (make_spec defaults) plus trace_mid and a VLM-shaped case
CASES = {
    "small": dict(num_layers=2, num_query_heads=4, num_kv_heads=2, head_dim=32, prompt_len=96,
                  post_vision_len=12, decode_len=4, seed=11, heavy_fraction=0.05, noise_scale=0.1),
    "mid": dict(num_layers=3, num_query_heads=4, num_kv_heads=2, head_dim=32, prompt_len=192,
                post_vision_len=24, decode_len=6, seed=7, heavy_fraction=0.05, noise_scale=0.1),
    "vlm": dict(num_layers=2, num_query_heads=8, num_kv_heads=2, head_dim=64, prompt_len=624,
                post_vision_len=32, decode_len=8, seed=3),
}
KS = (5, 10, 20)


def rounded_trace(vl, spec):
    tr, _ = vl.generate_trace(vl.GenSpec(**spec))
    return vl.AttentionTrace(header=tr.header, layout=tr.layout,
                             queries=[bf16_round(x) for x in tr.queries],
                             keys=[bf16_round(x) for x in tr.keys])


def main():
    vl = load_reference()
    out, reports = {}, {}
    for name, spec in CASES.items():
        tr = rounded_trace(vl, spec)
        h = tr.header
        m, L, H = h.prompt_len, h.num_layers, h.num_query_heads
        out[f"{name}/oracle"] = np.array([[[vl.oracle_scores(tr, l, q, o) for o in range(h.decode_len)]
                                           for q in range(H)] for l in range(L)])
        w_pv = vl.QueryWindow(m - h.post_vision_len, m)
        w_dec = vl.QueryWindow(m, h.seq_len)
        out[f"{name}/dense_pv"] = np.array([vl.dense_attention_rows(tr, l, 1, w_pv) for l in range(L)])
        out[f"{name}/dense_dec"] = np.array([vl.dense_attention_rows(tr, l, H - 1, w_dec) for l in range(L)])
        win = vl.EvalWindow.for_header(h)
        win3 = vl.EvalWindow.for_header(h, alpha_eval=0.3)
        for mod in ("vision", "language"):
            out[f"{name}/contribution/{mod}"] = np.array(
                [[vl.contribution(tr, l, q, win, mod) for q in range(H)] for l in range(L)])
            out[f"{name}/contribution05/{mod}"] = np.array(
                [[vl.contribution(tr, l, q, win, mod, p=0.05) for q in range(H)] for l in range(L)])
            out[f"{name}/coverage/{mod}"] = np.array(
                [[vl.coverage(tr, l, q, win, mod) for q in range(H)] for l in range(L)])
            out[f"{name}/coverage03/{mod}"] = np.array(
                [[vl.coverage(tr, l, q, win3, mod) for q in range(H)] for l in range(L)])
        pols = {"post_vision": vl.PostVision(), "h2o": vl.AccumulatedAttention(),
                "streaming": vl.StreamingInitRecent(n_init=4, n_recent=16)}
        for pname, pol in pols.items():
            for k in KS:
                out[f"{name}/hit/{pname}/{k}"] = np.array(
                    [[vl.cache_hit_rate(tr, l, q, pol, k) for q in range(H)] for l in range(L)])
            rows = min(3, h.decode_len)
            out[f"{name}/hit_rows/{pname}"] = np.array(
                [[vl.cache_hit_rate(tr, l, q, pol, 10, oracle_k=20, num_decode_rows=rows) for q in range(H)]
                 for l in range(L)])
        reports[name] = vl.build_report(tr, {"vlcache": vl.PostVision(), "h2o": vl.AccumulatedAttention()},
                                        k=10).to_dict()
    np.savez_compressed(os.path.join(HERE, "eval_golden.npz"), **out)
    with open(os.path.join(HERE, "eval_report.json"), "w") as f:
        json.dump(reports, f, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
