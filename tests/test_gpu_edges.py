"""Edge cases of the sm_100a path against the CPU oracle (bf16-in protocol).

Windows that straddle 32-row groups and heads, single-row windows, prefill-
sized windows (many 128-row blocks), extreme budgets and reserve fractions,
very long score rows (the global-scratch radix select) and empty/size-one
decode caches -- the shapes the reference's own tests exercise
(test_kernels.py CASES, test_scoring.py ties, test_budget.py clips).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2410_23317_b200 import _kernels  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402
from paper_2410_23317_b200.trace import GenSpec  # noqa: E402
from test_gpu_parity import bf16, check_kept_sets, make_inputs  # noqa: E402


@pytest.mark.parametrize("layers,hq,hkv,d,m,tau,alpha,recent", [
    (2, 8, 2, 64, 300, 12, 0.1, 0.1),      # 48-row slots: heads straddle 32-row groups
    (2, 8, 8, 64, 200, 1, 0.1, 0.1),       # single-row windows
    (1, 4, 2, 64, 260, 260, 0.1, 0.1),     # prefill window: 520 rows, 5 row blocks
    (3, 4, 4, 128, 400, 40, 1.0, 0.1),     # alpha = 1 (clipped budgets)
    (3, 4, 4, 128, 400, 40, 0.01, 0.1),    # tiny budgets, reserve dominates
    (2, 4, 2, 128, 400, 40, 0.1, 0.0),     # no recent reserve
    (2, 4, 2, 128, 400, 40, 0.1, 1.0),     # reserve = the whole budget
])
def test_engine_edges(layers, hq, hkv, d, m, tau, alpha, recent):
    spec = GenSpec(num_layers=layers, num_query_heads=hq, num_kv_heads=hkv, head_dim=d, prompt_len=m,
                   post_vision_len=tau, decode_len=3, seed=21)
    host, dv = make_inputs(spec, tau)
    g = hq // hkv
    eng = VLCache(Shape(1, layers, hq, hkv, d, m, tau), alpha=alpha, recent_frac=recent, decode_steps=3,
                  keep_scores=True)
    eng.compress(dv["q_win"], dv["keys"], dv["values"])
    ref = O.compression_pass(host[0]["q_win"], host[0]["keys"], m, g, alpha=alpha, recent_frac=recent)
    ref_below = np.array([[ref["stats"][(l, h)][3].sum() for h in range(hq)] for l in range(layers)])
    np.testing.assert_array_equal(eng.below_head.view(layers, hq).cpu().numpy(), ref_below)
    np.testing.assert_array_equal(eng.kept_counts.cpu().numpy(), ref["kept_counts"])
    np.testing.assert_allclose(eng.scores.view(layers, hkv, m).cpu().numpy(), ref["scores"], rtol=1e-5,
                               atol=1e-12)
    kept = eng.kept_sets()[0]
    check_kept_sets(kept, ref["kept"], ref["scores"], ref["kept_counts"])
    outs = []
    eng.decode(dv["q_dec"], dv["keys"], dv["values"], outputs=outs)
    ref_out = O.decode_sequence(host[0]["q_dec"], host[0]["keys"], host[0]["values"], kept, m, g, 3)
    for s in range(3):
        np.testing.assert_allclose(outs[s].view(layers, hq, d).cpu().numpy(),
                                   np.stack([ref_out[s][l] for l in range(layers)]), rtol=1e-4, atol=1e-5)


def test_long_score_rows_use_global_scratch():
    """n > 24576 scores take the global-memory radix path; ties included."""
    import paper_2410_23317_b200 as vl

    rng = np.random.default_rng(3)
    for n, k in ((30000, 3000), (40000, 17)):
        s = np.round(rng.standard_normal(n) * 4) / 4          # many ties
        for frac in (0.0, 0.1):
            np.testing.assert_array_equal(vl.evict(s, k, vl.EvictionConfig(frac)), O.evict(s, k, frac))


def test_negative_and_signed_zero_scores():
    import paper_2410_23317_b200 as vl

    s = np.array([-1.0, -0.0, 0.0, -2.5, 3.0, -0.0, 1e-300, -1e-300])
    for k in range(1, s.size + 1):
        np.testing.assert_array_equal(vl.top_k_indices(s, k), O.top_k(s, k))


def test_stats_window_smaller_than_tau_matches_oracle():
    """A stats window of the last 50 rows when tau = 64 (reference
    measure_gamma_mean(window_rows=50)): rows [m-50, m) over keys [0, m)."""
    spec = GenSpec(num_layers=2, num_query_heads=8, num_kv_heads=2, head_dim=128, prompt_len=700,
                   post_vision_len=64, decode_len=1, seed=4)
    host, dv = make_inputs(spec, 50)
    eng = VLCache(Shape(1, 2, 8, 2, 128, 700, 50), keep_scores=True)
    eng.compress(dv["q_win"], dv["keys"])
    ref = O.compression_pass(host[0]["q_win"], host[0]["keys"], 700, 4)
    np.testing.assert_array_equal(eng.kept_counts.cpu().numpy(), ref["kept_counts"])
    check_kept_sets(eng.kept_sets()[0], ref["kept"], ref["scores"], ref["kept_counts"])


@pytest.mark.parametrize("w,n,qb", [(1, 1, 0), (3, 3, 0), (130, 300, 170), (257, 257, 0)])
def test_stats_tiny_and_ragged(w, n, qb):
    rng = np.random.default_rng(w * 7 + n)
    q, k = bf16(rng.standard_normal((w, 64))), bf16(rng.standard_normal((n, 64)))
    got = _kernels.stats_tiled(q, k, qb, 0.01, 128)
    ref = O.stats_tiled(q, k, qb, 0.01, 128)
    np.testing.assert_allclose(got[0], ref[0], rtol=1e-6)
    np.testing.assert_allclose(got[2], ref[2], rtol=1e-5, atol=1e-12)
    np.testing.assert_array_equal(got[3], ref[3])
    np.testing.assert_array_equal(got[4], ref[4])
