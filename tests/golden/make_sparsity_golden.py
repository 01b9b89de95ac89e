"""Golden vectors of the reference's O(m^2) analysis sparsities (SURVEY.md
section 8 row f4): prefill_sparsity (every prompt row, sparsity.py:83-85) and
decoding_sparsity (the decoding rows, sparsity.py:98-103), plus
post_vision_sparsity, on bf16-rounded generator traces ("bf16-in", the values
K1 consumes on the B200).

Run here (where /root/reference is mounted):  python tests/golden/make_sparsity_golden.py
Writes tests/golden/sparsity_golden.npz; the GPU box never reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_eval_golden import rounded_trace  # noqa: E402
from make_golden import load_reference  # noqa: E402

CASES = {
    "small": dict(num_layers=2, num_query_heads=4, num_kv_heads=2, head_dim=32, prompt_len=96,
                  post_vision_len=12, decode_len=4, seed=11, heavy_fraction=0.05, noise_scale=0.1),
    "mid": dict(num_layers=3, num_query_heads=4, num_kv_heads=2, head_dim=32, prompt_len=192,
                post_vision_len=24, decode_len=6, seed=7, heavy_fraction=0.05, noise_scale=0.1),
    "vlm": dict(num_layers=2, num_query_heads=8, num_kv_heads=2, head_dim=64, prompt_len=624,
                post_vision_len=32, decode_len=8, seed=3),
    "m7b_slice": dict(num_layers=2, num_query_heads=32, num_kv_heads=8, head_dim=128, prompt_len=1200,
                      post_vision_len=64, decode_len=16, seed=5),
}


def main():
    vl = load_reference()
    out = {}
    for name, spec in CASES.items():
        tr = rounded_trace(vl, spec)
        for fn in ("prefill_sparsity", "decoding_sparsity", "post_vision_sparsity"):
            ls = getattr(vl, fn)(tr, vl.SparsityConfig())
            out[f"{name}_{fn}_gamma"] = ls.gamma
            out[f"{name}_{fn}_means"] = ls.layer_means()
        for k, v in spec.items():
            out[f"{name}_spec_{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "sparsity_golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
