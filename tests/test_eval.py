"""Row f4 (analysis / evaluation): the oracle restatement and the B200 path
against golden vectors produced by the reference's own evaluate.py
(tests/golden/make_eval_golden.py, bf16-rounded generator traces).

CPU tests pin oracle/'s restatement; GPU tests run the package functions
(vlc_attention_rows + K3 + K1) and compare with the same vectors.  Logits are
float32 roundings of float64 dots of fp32 rows on both sides, so probabilities
and the mass ratios agree to a float32 exp rounding (the device's correctly
rounded exp vs numpy's SIMD expf; rtol 1e-6); set-valued metrics (coverage, hit
rates) must match exactly.
"""

import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2410_23317_b200.trace import AttentionTrace, GenSpec, generate_trace, round_to_bf16

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {
    "small": dict(num_layers=2, num_query_heads=4, num_kv_heads=2, head_dim=32, prompt_len=96,
                  post_vision_len=12, decode_len=4, seed=11, heavy_fraction=0.05, noise_scale=0.1),
    "mid": dict(num_layers=3, num_query_heads=4, num_kv_heads=2, head_dim=32, prompt_len=192,
                post_vision_len=24, decode_len=6, seed=7, heavy_fraction=0.05, noise_scale=0.1),
    "vlm": dict(num_layers=2, num_query_heads=8, num_kv_heads=2, head_dim=64, prompt_len=624,
                post_vision_len=32, decode_len=8, seed=3),
}
KS = (5, 10, 20)
_TRACES = {}


@pytest.fixture(scope="module")
def eg():
    return np.load(os.path.join(HERE, "golden", "eval_golden.npz"))


def trace(name):
    if name not in _TRACES:
        tr, _ = generate_trace(GenSpec(**CASES[name]))
        _TRACES[name] = AttentionTrace(header=tr.header, layout=tr.layout,
                                       queries=[round_to_bf16(x) for x in tr.queries],
                                       keys=[round_to_bf16(x) for x in tr.keys])
    return _TRACES[name]


def _oracle_policy_scores(tr, layer, head, pname):
    h = tr.header
    m = h.prompt_len
    if pname == "streaming":   # reference scoring.py:175-179 (n_init=4, n_recent=16)
        s = np.zeros(m)
        s[m - 16:] = 1.0
        s[:4] = 2.0
        return s
    start, end = (m - h.post_vision_len, m) if pname == "post_vision" else (0, m)
    q = tr.queries[layer][head, start:end]
    k = tr.keys[layer][tr.kv_head_for(head), :end]
    return O.stats_tiled(q, k, start, 0.01, 128)[2][:m]


# ---------------------------------------------------------------- CPU: oracle pinned
@pytest.mark.parametrize("name", list(CASES))
def test_oracle_rows_match_reference(eg, name):
    tr = trace(name)
    h = tr.header
    m = h.prompt_len
    for l in range(h.num_layers):
        for q in range(h.num_query_heads):
            kv = tr.kv_head_for(q)
            rows = O.causal_probs(tr.queries[l][q, m:h.seq_len], tr.keys[l][kv, :m], m, m)
            np.testing.assert_allclose(rows, eg[f"{name}/oracle"][l, q], rtol=1e-14, atol=0)
        pv = O.causal_probs(tr.queries[l][1, m - h.post_vision_len:m], tr.keys[l][tr.kv_head_for(1), :m],
                            m - h.post_vision_len, m)
        np.testing.assert_allclose(pv, eg[f"{name}/dense_pv"][l], rtol=1e-14, atol=0)


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_contribution_coverage_match_reference(eg, name):
    tr = trace(name)
    h = tr.header
    m, seq = h.prompt_len, h.seq_len
    for l in range(h.num_layers):
        for q in range(h.num_query_heads):
            probs = O.causal_probs(tr.queries[l][q, m:seq], tr.keys[l][tr.kv_head_for(q), :seq], m, seq)
            for mod in ("vision", "language"):
                idx = tr.layout.indices(mod)
                for key, p in (("contribution", 0.01), ("contribution05", 0.05)):
                    want = eg[f"{name}/{key}/{mod}"][l, q]
                    got = O.filtered_share(probs, m, idx, p) if idx.size else 0.0
                    assert got == pytest.approx(want, abs=1e-12)
                for key, a in (("coverage", 0.1), ("coverage03", 0.3)):
                    assert O.topk_share(probs, m, idx, int(np.floor(a * seq))) == eg[f"{name}/{key}/{mod}"][l, q]


@pytest.mark.parametrize("name", ["small", "mid"])
def test_oracle_hit_rates_match_reference(eg, name):
    tr = trace(name)
    h = tr.header
    m = h.prompt_len
    for pname in ("post_vision", "h2o", "streaming"):
        for l in range(h.num_layers):
            for q in range(h.num_query_heads):
                scores = _oracle_policy_scores(tr, l, q, pname)
                orows = eg[f"{name}/oracle"][l, q]
                for k in KS:
                    assert O.hit_rate(scores, orows[:1], k, k) == eg[f"{name}/hit/{pname}/{k}"][l, q]
                rows = min(3, h.decode_len)
                assert O.hit_rate(scores, orows[:rows], 10, 20) == pytest.approx(
                    eg[f"{name}/hit_rows/{pname}"][l, q], abs=1e-15)


def test_eval_window_validation():
    from paper_2410_23317_b200 import EvalWindow, ValidationError

    with pytest.raises(ValidationError, match="first_decode_index"):
        EvalWindow(10, 10)
    with pytest.raises(ValidationError, match="alpha_eval"):
        EvalWindow(0, 10, alpha_eval=1.0)
    assert EvalWindow(5, 101, 0.1).top_k == 10


# ---------------------------------------------------------------- GPU: the B200 path
@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_oracle_scores_and_dense_rows(eg, name):
    import paper_2410_23317_b200 as V

    tr = trace(name)
    h = tr.header
    m = h.prompt_len
    for l in range(h.num_layers):
        for q in range(h.num_query_heads):
            for o in range(h.decode_len):
                np.testing.assert_allclose(V.oracle_scores(tr, l, q, o), eg[f"{name}/oracle"][l, q, o],
                                           rtol=1e-6, atol=1e-300)
        pv = V.dense_attention_rows(tr, l, 1, V.QueryWindow(m - h.post_vision_len, m))
        np.testing.assert_allclose(pv, eg[f"{name}/dense_pv"][l], rtol=1e-6, atol=1e-300)
        dec = V.dense_attention_rows(tr, l, h.num_query_heads - 1, V.QueryWindow(m, h.seq_len))
        np.testing.assert_allclose(dec, eg[f"{name}/dense_dec"][l], rtol=1e-6, atol=1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_contribution_coverage(eg, name):
    import paper_2410_23317_b200 as V

    tr = trace(name)
    h = tr.header
    win, win3 = V.EvalWindow.for_header(h), V.EvalWindow.for_header(h, alpha_eval=0.3)
    for l in range(h.num_layers):
        for q in range(h.num_query_heads):
            for mod in ("vision", "language"):
                # float32 exp of the device vs numpy's SIMD expf: <= 1 ulp per entry
                assert V.contribution(tr, l, q, win, mod) == pytest.approx(
                    eg[f"{name}/contribution/{mod}"][l, q], rel=1e-6, abs=1e-12)
                assert V.contribution(tr, l, q, win, mod, p=0.05) == pytest.approx(
                    eg[f"{name}/contribution05/{mod}"][l, q], rel=1e-6, abs=1e-12)
                assert V.coverage(tr, l, q, win, mod) == eg[f"{name}/coverage/{mod}"][l, q]
                assert V.coverage(tr, l, q, win3, mod) == eg[f"{name}/coverage03/{mod}"][l, q]


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_hit_rates(eg, name):
    import paper_2410_23317_b200 as V

    tr = trace(name)
    h = tr.header
    pols = {"post_vision": V.PostVision(), "h2o": V.AccumulatedAttention(),
            "streaming": V.StreamingInitRecent(n_init=4, n_recent=16)}
    for pname, pol in pols.items():
        for l in range(h.num_layers):
            for q in range(h.num_query_heads):
                for k in KS:
                    assert V.cache_hit_rate(tr, l, q, pol, k) == eg[f"{name}/hit/{pname}/{k}"][l, q], (pname, l, q, k)
                rows = min(3, h.decode_len)
                assert V.cache_hit_rate(tr, l, q, pol, 10, oracle_k=20, num_decode_rows=rows) == pytest.approx(
                    eg[f"{name}/hit_rows/{pname}"][l, q], abs=1e-15)
    # the oracle itself as the policy is a perfect score (reference test_evaluate.py:95-100)
    assert V.cache_hit_rate(tr, 0, 0, V.oracle_scores(tr, 0, 0), 10) == 1.0


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_build_report(name):
    import paper_2410_23317_b200 as V

    want = json.load(open(os.path.join(HERE, "golden", "eval_report.json")))[name]
    got = V.build_report(trace(name), {"vlcache": V.PostVision(), "h2o": V.AccumulatedAttention()}, k=10).to_dict()
    got = json.loads(json.dumps(got))
    assert got["curve_stats"] == want["curve_stats"]
    assert got["hit_rates"] == want["hit_rates"]
    assert len(got["modality"]) == len(want["modality"])
    for a, b in zip(got["modality"], want["modality"]):
        assert (a["layer"], a["modality"]) == (b["layer"], b["modality"])
        assert a["coverage"] == b["coverage"]
        assert a["contribution"] == pytest.approx(b["contribution"], rel=1e-6, abs=1e-12)


@pytest.mark.gpu
def test_gpu_eval_edges():
    """reference test_evaluate.py:187-205: empty modality, fully filtered prompt."""
    import paper_2410_23317_b200 as V

    tr, _ = generate_trace(GenSpec(**{**CASES["small"], "prompt_len": 48, "post_vision_len": 48, "seed": 2}))
    assert tr.layout.indices("vision").size == 0
    win = V.EvalWindow.for_header(tr.header)
    assert V.contribution(tr, 0, 0, win, "vision") == 0.0
    assert V.contribution(tr, 0, 0, win, "language") == pytest.approx(1.0, abs=1e-12)
    assert V.coverage(tr, 0, 0, win, "vision") + V.coverage(tr, 0, 0, win, "language") == 1.0
    # one decode key dwarfs both prompt keys: every prompt column is filtered out
    from paper_2410_23317_b200.trace import ModalityLayout, TraceHeader

    q = np.array([[[1.0], [1.0], [30.0]]], dtype=np.float32)
    k = np.array([[[0.1], [0.1], [30.0]]], dtype=np.float32)
    hdr = TraceHeader(num_layers=1, num_query_heads=1, num_kv_heads=1, head_dim=1, prompt_len=2,
                      post_vision_len=1, decode_len=1, seed=0)
    t = AttentionTrace(header=hdr, layout=ModalityLayout((0, 0), (0, 1), (1, 1)), queries=[q], keys=[k])
    win = V.EvalWindow.for_header(hdr)
    assert V.contribution(t, 0, 0, win, "language") == 0.0
    assert V.contribution(t, 0, 0, win, "vision") == 0.0
    with pytest.raises(V.ValidationError, match="alpha_eval"):
        V.coverage(trace("small"), 0, 0, V.EvalWindow.for_header(trace("small").header, alpha_eval=0.001), "vision")


@pytest.mark.gpu
@pytest.mark.parametrize("tau,group", [(64, 4), (128, 2), (192, 1)])
def test_gpu_batched_head_scores_bit_identical(tau, group):
    """build_report's one-launch policy scores equal one-head K1 launches bit for
    bit (each 64-row half of a 128-row block is one head's rows, in a one-head
    call's order).  head_scores itself runs the reference's float32 contract
    (the seam, float64 dots), so against it the scores agree to fp32 rounding
    and the hit rates up to near-ties at the top-k boundary."""
    import paper_2410_23317_b200 as V
    from paper_2410_23317_b200 import _kernels
    from paper_2410_23317_b200.evaluate import _all_head_scores

    spec = dict(num_layers=2, num_query_heads=8, num_kv_heads=8 // group, head_dim=64, prompt_len=700,
                post_vision_len=tau, decode_len=2, seed=5)
    tr, _ = generate_trace(GenSpec(**spec))
    tr = AttentionTrace(header=tr.header, layout=tr.layout, queries=[round_to_bf16(x) for x in tr.queries],
                        keys=[round_to_bf16(x) for x in tr.keys])
    got = _all_head_scores(tr, V.PostVision(), V.ScoringConfig())
    win = V.policy_window(V.PostVision(), tr.header)
    m = tr.header.prompt_len
    for l in range(2):
        for q in range(8):
            qr = tr.query_rows(l, q, win.start, win.end)
            kr = tr.key_rows(l, q, win.end)
            one = _kernels.stats_tiled_tc(qr, kr, win.start, V.ScoringConfig().p)[2][:m]
            np.testing.assert_array_equal(got[l, q], one)
            np.testing.assert_allclose(got[l, q], V.head_scores(tr, l, q, V.PostVision()), rtol=1e-5, atol=1e-12)
    rep = V.build_report(tr, {"pv": V.PostVision()}, k=50).to_dict()
    for row in rep["hit_rates"]:
        ref = V.cache_hit_rate(tr, row["layer"], row["head"], V.PostVision(), 50)
        assert abs(row["hit_rate"] - ref) <= 1 / 50 + 1e-12


def _eval_fuzz(n=8, seed=99):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        hkv = int(rng.choice([1, 2, 4]))
        m = int(rng.integers(40, 500))
        out.append(dict(num_layers=1, num_query_heads=hkv * int(rng.choice([1, 2, 4])), num_kv_heads=hkv,
                        head_dim=int(rng.choice([16, 32, 48, 64])), prompt_len=m,
                        post_vision_len=int(rng.integers(0, m // 2)), decode_len=int(rng.integers(1, 6)),
                        seed=int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("spec", _eval_fuzz())
def test_gpu_eval_fuzz(spec):
    """Random shapes (odd head dims, MHA/GQA, short prompts, tau = 0) against the
    oracle restatement: contribution within float32-exp rounding, coverage and
    hit rates within one position of a near-tie per row."""
    import paper_2410_23317_b200 as V

    tr, _ = generate_trace(GenSpec(**spec))
    h = tr.header
    m, seq = h.prompt_len, h.seq_len
    win = V.EvalWindow.for_header(h, alpha_eval=0.2)
    k = max(1, m // 10)
    for q in range(h.num_query_heads):
        kv = tr.kv_head_for(q)
        probs = O.causal_probs(tr.queries[0][q, m:seq], tr.keys[0][kv, :seq], m, seq)
        for mod in ("vision", "language"):
            idx = tr.layout.indices(mod)
            want = O.filtered_share(probs, m, idx, 0.01) if idx.size else 0.0
            assert V.contribution(tr, 0, q, win, mod) == pytest.approx(want, rel=1e-6, abs=1e-12)
            if win.top_k <= m:
                cov = V.coverage(tr, 0, q, win, mod)
                assert abs(cov - O.topk_share(probs, m, idx, win.top_k)) <= 1.0 / win.top_k + 1e-12
        orow = O.causal_probs(tr.queries[0][q, m:m + 1], tr.keys[0][kv, :m], m, m)
        np.testing.assert_allclose(V.oracle_scores(tr, 0, q), orow[0], rtol=1e-6, atol=1e-300)
        hr = V.cache_hit_rate(tr, 0, q, orow[0], k)
        assert hr >= 1.0 - 1.0 / k
