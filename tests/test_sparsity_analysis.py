"""Row f4's O(m^2) analysis sparsities against the reference's own outputs
(tests/golden/sparsity_golden.npz, made by tests/golden/make_sparsity_golden.py
from the reference's prefill_sparsity / decoding_sparsity / post_vision_sparsity,
sparsity.py:83-103, on bf16-rounded generator traces).

CPU: the oracle restatement (per-(layer, head) stats, gamma = sum below / sum
causal, reference sparsity.py:69-80) reproduces the golden gamma bit for bit.
GPU: the package's functions (K1 over every head in one launch, exact mode)
give the same gamma and head means bit for bit -- including the prefill window,
every prompt row as a query (many 128-row blocks per slot)."""

import os

import numpy as np
import pytest

from paper_2410_23317_b200.trace import AttentionTrace, GenSpec, generate_trace, round_to_bf16

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sparsity_golden.npz")
FNS = ("prefill_sparsity", "decoding_sparsity", "post_vision_sparsity")


def _golden():
    return np.load(GOLDEN)


def _cases(g):
    return sorted({k.split("_spec_")[0] for k in g.files if "_spec_" in k})


def _trace(g, name):
    keys = [k for k in g.files if k.startswith(name + "_spec_")]
    spec = {k.split("_spec_")[1]: g[k].item() for k in keys}
    tr, _ = generate_trace(GenSpec(**spec))
    return AttentionTrace(header=tr.header, layout=tr.layout, queries=[round_to_bf16(x) for x in tr.queries],
                          keys=[round_to_bf16(x) for x in tr.keys])


def _window(fn, h):
    m, t = h.prompt_len, h.seq_len
    return {"prefill_sparsity": (0, m), "decoding_sparsity": (m, t),
            "post_vision_sparsity": (m - h.post_vision_len, m)}[fn]


@pytest.mark.parametrize("name", ["small", "mid"])
def test_oracle_matches_reference_sparsity_golden(name):
    from oracle import oracle as O

    g = _golden()
    tr = _trace(g, name)
    h = tr.header
    for fn in FNS:
        lo, hi = _window(fn, h)
        gamma = np.empty((h.num_layers, h.num_query_heads))
        for l in range(h.num_layers):
            for q in range(h.num_query_heads):
                st = O.stats_tiled(tr.queries[l][q, lo:hi], tr.keys[l][q // h.group_size, :hi], lo, 0.01, 128)
                gamma[l, q] = st[3].sum() / st[4].sum()
        np.testing.assert_array_equal(gamma, g[f"{name}_{fn}_gamma"], err_msg=fn)
        np.testing.assert_array_equal(gamma.mean(axis=1), g[f"{name}_{fn}_means"], err_msg=fn)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["small", "mid", "vlm", "m7b_slice"])
def test_device_sparsities_match_reference(name):
    import paper_2410_23317_b200 as vl

    g = _golden()
    tr = _trace(g, name)
    for fn in FNS:
        ls = getattr(vl, fn)(tr, vl.SparsityConfig())
        np.testing.assert_array_equal(ls.gamma, g[f"{name}_{fn}_gamma"], err_msg=fn)
        np.testing.assert_array_equal(ls.layer_means(), g[f"{name}_{fn}_means"], err_msg=fn)
