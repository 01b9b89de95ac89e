"""Parity of the sm_100a path against the CPU oracle (bf16-in protocol).

Both sides consume identical bf16-representable inputs.  Tolerances (SURVEY.md
§8c, from the reference's own tests):
  causal counts exact; below counts exact expected, |d| <= 2 per column and
  <= 8 per head-call allowed (test_kernels.py:83-85); row_max rtol 1e-6;
  row_sum / col_score rtol 1e-5, atol 1e-12; gamma, beta, k_l bit-exact given
  equal counts; kept sets bit-exact except indices whose oracle scores tie
  within 1e-6 * max score with the selection boundary; decode outputs rtol
  1e-4 / atol 1e-5 (test_kernels.py:108).
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import TOY  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2410_23317_b200 import _kernels  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402
from paper_2410_23317_b200.trace import GenSpec, iter_layers, round_to_bf16, synthesize_values  # noqa: E402

STATS_CASES = [
    (0, 96, 96, 32, 0), (1, 96, 96, 32, 0), (2, 40, 128, 64, 88), (3, 4, 256, 32, 252),
    (4, 1, 64, 16, 63), (5, 200, 200, 48, 0), (6, 64, 700, 128, 636), (7, 32, 624, 64, 592),
    (8, 256, 2960, 128, 2704), (9, 64, 2960, 128, 2896),
]


def bf16(x):
    return round_to_bf16(np.asarray(x, dtype=np.float32))


def assert_counts_close(got, ref, per_col=2, total=8):
    d = np.abs(got.astype(np.int64) - ref.astype(np.int64))
    assert d.max(initial=0) <= per_col and d.sum() <= total, (d.max(initial=0), d.sum())


@pytest.mark.parametrize("seed,w,n,d,qb", STATS_CASES)
def test_score_stats_matches_oracle(seed, w, n, d, qb):
    rng = np.random.default_rng(seed)
    q = bf16(rng.standard_normal((w, d)) * (2.0 if seed >= 8 else 1.0))
    k = bf16(rng.standard_normal((n, d)))
    got = _kernels.stats_tiled_tc(q, k, qb, 0.01, 128)
    ref = O.stats_tiled(q, k, qb, 0.01, 128)
    np.testing.assert_allclose(got[0], ref[0], rtol=1e-6, atol=0)
    np.testing.assert_allclose(got[1], ref[1], rtol=1e-5, atol=0)
    np.testing.assert_allclose(got[2], ref[2], rtol=1e-5, atol=1e-12)
    np.testing.assert_array_equal(got[4], ref[4])
    np.testing.assert_array_equal(got[3], ref[3])        # exact mode: every below decision
    assert got[2].sum() == pytest.approx(w, rel=1e-6)   # each row contributes mass 1


def test_p_extremes():
    """reference test_kernels.py:87-93, exact: p -> 0 nothing below; p = 1
    everything but the entries equal to their row max in float32 -- exact
    logit ties, decided from float64 dots by K1's exact mode."""
    rng = np.random.default_rng(7)
    q, k = bf16(rng.standard_normal((64, 32))), bf16(rng.standard_normal((64, 32)))
    got = _kernels.stats_tiled_tc(q, k, 0, 1e-300, 32)
    ref = O.stats_tiled(q, k, 0, 1e-300, 32)
    np.testing.assert_array_equal(got[3], ref[3])
    got = _kernels.stats_tiled_tc(q, k, 0, 1.0, 32)
    ref = O.stats_tiled(q, k, 0, 1.0, 32)
    np.testing.assert_array_equal(got[3], ref[3])


@pytest.mark.parametrize("seed,g,n,d", [(0, 2, 128, 32), (1, 4, 512, 64), (2, 1, 33, 16),
                                        (3, 4, 300, 128), (4, 7, 1000, 128), (5, 8, 1, 64)])
def test_decode_step_matches_oracle(seed, g, n, d):
    rng = np.random.default_rng(seed)
    q, k, v = (bf16(rng.standard_normal(s)) for s in ((g, d), (n, d), (n, d)))
    np.testing.assert_allclose(_kernels.decode_step(q, k, v), O.decode_step(q, k, v), rtol=1e-4, atol=1e-5)


def test_decode_uniform_weights_known_answer():
    d = 8
    q = np.zeros((1, d), np.float32)
    keys = np.arange(3 * d, dtype=np.float32).reshape(3, d)
    values = np.stack([np.full(d, 3.0), np.full(d, 6.0), np.full(d, 9.0)]).astype(np.float32)
    np.testing.assert_allclose(_kernels.decode_step(q, keys, values), np.full((1, d), 6.0), rtol=1e-6)


# ------------------------------------------------------------------ batched path
def make_inputs(spec: GenSpec, w: int, batch: int = 1):
    """bf16-rounded inputs; prompt b uses seed + b. Host arrays for the oracle
    and device tensors [B, L, H, ., d] for the engine."""
    host = []
    for b in range(batch):
        sp = GenSpec(**{**spec.__dict__, "seed": spec.seed + b})
        keys, q_win, q_dec = [], [], []
        for k, q in iter_layers(sp, keep_prompt_rows=w):
            keys.append(bf16(k))
            q = bf16(q)
            q_win.append(np.ascontiguousarray(q[:, :w]))
            q_dec.append(np.ascontiguousarray(q[:, w:]))
        values = [bf16(v) for v in synthesize_values(sp)]
        host.append(dict(keys=keys, q_win=q_win, q_dec=q_dec, values=values))

    def dev(name):
        a = np.stack([np.stack(h[name]) for h in host])
        return torch.from_numpy(a).cuda().to(torch.bfloat16).contiguous()

    return host, {n: dev(n) for n in ("keys", "q_win", "q_dec", "values")}


def check_kept_sets(got, ref, scores, counts):
    """Bit-exact, except symmetric-difference indices whose oracle scores tie
    within 1e-6 * max with the boundary score."""
    mism = 0
    for l in range(len(ref)):
        for kv in range(len(ref[l])):
            a, b = np.asarray(got[l][kv]), np.asarray(ref[l][kv])
            assert a.size == b.size == counts[l]
            assert np.all(np.diff(a) > 0)
            if np.array_equal(a, b):
                continue
            sc = scores[l, kv]
            diff = np.setxor1d(a, b)
            bound = np.min(sc[b[b < sc.size - math.ceil(0.1 * counts[l])]]) if b.size else 0.0
            assert np.all(np.abs(sc[diff] - bound) <= 1e-6 * sc.max()), (l, kv, diff)
            mism += 1
    return mism


@pytest.mark.parametrize("hkv,layers,m,tau,d,hq", [
    (8, 4, 624, 32, 64, 8),      # TOY
    (2, 4, 624, 32, 64, 8),      # TOY, GQA 4
    (8, 3, 2960, 64, 128, 32),   # M7B shapes, 3 of 32 layers
    (8, 2, 1200, 64, 128, 56),   # Y34B-style G=7
])
def test_engine_compress_and_decode_match_oracle(hkv, layers, m, tau, d, hq):
    run_parity_case(hkv, layers, m, tau, d, hq)


def _fuzz_cases(n=24, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        hkv = int(rng.choice([1, 2, 4, 8]))
        g = int(rng.choice([1, 2, 3, 4, 7, 8]))
        m = int(rng.integers(64, 1500))
        out.append((hkv, int(rng.integers(1, 4)), m, int(rng.integers(1, min(m, 160) + 1)),
                    int(rng.choice([64, 128])), hkv * g, float(rng.uniform(0.02, 0.5)), int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("hkv,layers,m,tau,d,hq,alpha,seed", _fuzz_cases())
def test_engine_fuzz_matches_oracle(hkv, layers, m, tau, d, hq, alpha, seed):
    """Random shapes, windows, budgets and seeds through the whole path."""
    run_parity_case(hkv, layers, m, tau, d, hq, alpha=alpha, seed=seed, n_dec=4)


def run_parity_case(hkv, layers, m, tau, d, hq, alpha=0.1, seed=0, n_dec=6):
    spec = GenSpec(num_layers=layers, num_query_heads=hq, num_kv_heads=hkv, head_dim=d, prompt_len=m,
                   post_vision_len=tau, decode_len=n_dec, seed=seed)
    host, dv = make_inputs(spec, tau)
    g = hq // hkv
    eng = VLCache(Shape(B=1, L=layers, Hq=hq, Hkv=hkv, d=d, m=m, w=tau), alpha=alpha, decode_steps=n_dec,
                  keep_scores=True)
    eng.compress(dv["q_win"], dv["keys"], dv["values"])
    torch.cuda.synchronize()
    ref = O.compression_pass(host[0]["q_win"], host[0]["keys"], m, g, tile=128, alpha=alpha)
    below = eng.below_head.view(layers, hq).cpu().numpy()
    ref_below = np.array([[ref["stats"][(l, h)][3].sum() for h in range(hq)] for l in range(layers)])
    np.testing.assert_array_equal(below, ref_below)
    np.testing.assert_array_equal(eng.gamma.view(layers, hq).cpu().numpy(), ref["gamma"])
    np.testing.assert_array_equal(eng.gamma_mean.cpu().numpy(), ref["gamma_mean"])
    np.testing.assert_array_equal(eng.beta_pre.cpu().numpy(), ref["beta_pre"])
    np.testing.assert_array_equal(eng.kept_counts.cpu().numpy(), ref["kept_counts"])
    scores = eng.scores.view(layers, hkv, m).cpu().numpy()
    np.testing.assert_allclose(scores, ref["scores"], rtol=1e-5, atol=1e-12)
    kept = eng.kept_sets()[0]
    check_kept_sets(kept, ref["kept"], ref["scores"], ref["kept_counts"])
    rm = eng.row_max.view(layers, hkv, g, tau).reshape(layers, hq, tau).cpu().numpy()
    ref_rm = np.array([[ref["stats"][(l, h)][0] for h in range(hq)] for l in range(layers)])
    np.testing.assert_allclose(rm, ref_rm, rtol=1e-6)
    # gather: the cache rows are the kept K/V rows, bit for bit
    koff = eng.cache_off.cpu().numpy()
    kc = eng.k_cache.view(-1, d).cpu().float().numpy()
    vc = eng.v_cache.view(-1, d).cpu().float().numpy()
    for l in range(layers):
        for kv in range(hkv):
            s = l * hkv + kv
            idx = kept[l][kv]
            np.testing.assert_array_equal(kc[koff[s]:koff[s] + idx.size], host[0]["keys"][l][kv, idx])
            np.testing.assert_array_equal(vc[koff[s]:koff[s] + idx.size], host[0]["values"][l][kv, idx])
    # decode over the device's kept sets, eager then graph, against the oracle loop
    outs = []
    eng.decode(dv["q_dec"], dv["keys"], dv["values"], outputs=outs)
    ref_out = O.decode_sequence(host[0]["q_dec"], host[0]["keys"], host[0]["values"], kept, m, g, n_dec)
    for s in range(n_dec):
        got = outs[s].view(layers, hq, d).cpu().numpy()
        exp = np.stack([ref_out[s][l] for l in range(layers)])
        np.testing.assert_allclose(got, exp, rtol=1e-4, atol=1e-5)
    eng.compress(dv["q_win"], dv["keys"], dv["values"])   # reset the appended rows
    last = eng.decode(dv["q_dec"], dv["keys"], dv["values"], graph=True)
    np.testing.assert_array_equal(last.cpu().numpy(), outs[-1].cpu().numpy())


def test_batched_prompts_are_independent():
    spec = GenSpec(num_layers=2, num_query_heads=8, num_kv_heads=2, head_dim=64, prompt_len=400,
                   post_vision_len=32, decode_len=2, seed=5)
    host, dv = make_inputs(spec, 32, batch=3)
    eng = VLCache(Shape(B=3, L=2, Hq=8, Hkv=2, d=64, m=400, w=32), decode_steps=2)
    eng.compress(dv["q_win"], dv["keys"], dv["values"])
    kept = eng.kept_sets()
    counts = eng.kept_counts.view(3, 2).cpu().numpy()
    for b in range(3):
        ref = O.compression_pass(host[b]["q_win"], host[b]["keys"], 400, 4, tile=128)
        np.testing.assert_array_equal(counts[b], ref["kept_counts"])
        check_kept_sets(kept[b], ref["kept"], ref["scores"], ref["kept_counts"])


def test_full_m7b_properties():
    """Full LLaVA-1.6-Mistral-7B shapes: size-independent invariants."""
    L, HQ, HKV, D, M, TAU = 32, 32, 8, 128, 2960, 64
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.randn((1, L, HQ, TAU, D), device="cuda", generator=g) * 2).to(torch.bfloat16)
    k = torch.randn((1, L, HKV, M + 4, D), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((1, L, HKV, M + 4, D), device="cuda", generator=g).to(torch.bfloat16)
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), decode_steps=4, keep_scores=True)
    eng.compress(q, k, v)
    counts = eng.kept_counts.cpu().numpy()
    kept = eng.kept_sets()[0]
    assert eng.kept_off[-1].item() == HKV * counts.sum()
    assert np.all((counts >= 1) & (counts <= M))
    gm = eng.gamma_mean.cpu().numpy()
    assert np.all((gm >= 0) & (gm <= 1))
    pre = eng.beta_pre.cpu().numpy()
    assert abs(pre.sum() - 0.1 * L) <= 1e-9
    sc = eng.scores.view(L, HKV, M).cpu().numpy()
    # every row contributes softmax mass 1: sum of a slot's scores = tau
    np.testing.assert_allclose(sc.sum(-1), TAU, rtol=1e-5)
    for l in range(L):
        reserve = min(math.ceil(0.1 * counts[l]), counts[l])
        for kv in range(HKV):
            idx = kept[l][kv]
            assert idx.size == counts[l] and np.all(np.diff(idx) > 0)
            assert np.all(np.isin(np.arange(M - reserve, M), idx))
            rest = np.setdiff1d(np.arange(M - reserve), idx)
            chosen = np.setdiff1d(idx, np.arange(M - reserve, M))
            if chosen.size and rest.size:
                assert sc[l, kv, chosen].min() >= sc[l, kv, rest].max()


def test_reference_api_on_toy_trace(golden):
    """The reference-shaped API (library path) on the bf16 TOY trace."""
    import paper_2410_23317_b200 as vl
    from paper_2410_23317_b200.trace import AttentionTrace, generate_trace

    spec = GenSpec(**{**TOY, "num_kv_heads": 2})
    tr, _ = generate_trace(spec)
    tr = AttentionTrace(tr.header, tr.layout, [bf16(x) for x in tr.queries], [bf16(x) for x in tr.keys])
    sp = vl.post_vision_sparsity(tr)
    np.testing.assert_array_equal(sp.gamma, golden["toy2_gamma"])
    gm = vl.measure_gamma_mean(tr)
    np.testing.assert_array_equal(gm, golden["toy2_gamma_mean"])
    alloc = vl.allocate_sparsity_aware(gm, 0.1, tr.header.prompt_len)
    np.testing.assert_array_equal(alloc.beta_preclip, golden["toy2_beta_pre"])
    np.testing.assert_array_equal(alloc.kept_counts, golden["toy2_kept_counts"])
    res = vl.compress_cache(tr, alloc, vl.PostVision())
    got = [[ks.kept for ks in row] for row in res.kept_sets]
    check_kept_sets(got, golden["toy2_kept"], golden["toy2_scores"], alloc.kept_counts)
    np.testing.assert_allclose(vl.score_tokens(tr, 1, 1, vl.PostVision()), golden["toy2_scores"][1, 1],
                               rtol=1e-5, atol=1e-12)


def test_allocate_api_bit_exact(golden):
    import paper_2410_23317_b200 as vl

    for g, (alpha, m), pre, beta, kept in list(zip(golden["alloc_gamma"], golden["alloc_alpha_m"],
                                                    golden["alloc_pre"], golden["alloc_beta"],
                                                    golden["alloc_kept"]))[:60]:
        a = vl.allocate_sparsity_aware(g, float(alpha), int(m))
        np.testing.assert_array_equal(a.beta_preclip, pre)
        np.testing.assert_array_equal(a.beta, beta)
        np.testing.assert_array_equal(a.kept_counts, kept)
    with pytest.raises(vl.DegenerateSparsityError):
        vl.allocate_sparsity_aware([1.0, 1.0], 0.1, 100)


def test_evict_api_matches_reference_including_ties(golden):
    import paper_2410_23317_b200 as vl

    for s, (k, frac), kept in list(zip(golden["evict_scores"], golden["evict_args"],
                                       golden["evict_kept"]))[:80]:
        got = vl.evict(s, int(k), vl.EvictionConfig(recent_window_frac=float(frac)))
        np.testing.assert_array_equal(got, kept)
    assert vl.top_k_indices(np.array([3.0, 1.0, 3.0, 2.0]), 1).tolist() == [2]
    assert vl.top_k_indices(np.array([3.0, 1.0, 3.0, 2.0]), 2).tolist() == [0, 2]
    assert vl.top_k_indices(np.zeros(5), 3).tolist() == [2, 3, 4]
    assert vl.top_k_indices(np.array([-0.0, 0.0, -1.0]), 1).tolist() == [1]


def test_fixed_budgets_through_compress_cache(golden):
    """Uniform / pyramid budgets (reference budget.py:114-147) drive K3 through
    the library path; kept sets against the oracle's evict on the reference's
    own TOY scores."""
    import paper_2410_23317_b200 as vl
    from paper_2410_23317_b200.trace import AttentionTrace, generate_trace

    spec = GenSpec(**{**TOY, "num_kv_heads": 2})
    tr, _ = generate_trace(spec)
    tr = AttentionTrace(tr.header, tr.layout, [bf16(x) for x in tr.queries], [bf16(x) for x in tr.keys])
    m, L = tr.header.prompt_len, tr.header.num_layers
    scores = golden["toy2_scores"]
    for alloc in (vl.allocate_uniform(0.1, L, m), vl.allocate_pyramid(0.1, L, m, decay_ratio=0.5),
                  vl.allocate_pyramid(0.05, L, m, decay_ratio=0.2)):
        res = vl.compress_cache(tr, alloc, vl.PostVision())
        got = [[ks.kept for ks in row] for row in res.kept_sets]
        ref = [[O.evict(scores[l, kv], int(alloc.kept_counts[l])) for kv in range(scores.shape[1])]
               for l in range(L)]
        check_kept_sets(got, ref, scores, alloc.kept_counts)


@pytest.mark.parametrize("seed,w,n,d,qb,tile", [
    (0, 96, 96, 32, 0, 32), (1, 96, 96, 32, 0, 17), (2, 40, 128, 64, 88, 33), (3, 4, 256, 32, 252, 64),
    (4, 1, 64, 16, 63, 4096), (5, 200, 200, 48, 0, 128), (6, 64, 2960, 128, 2896, 256),
])
def test_seam_f32_matches_reference_arithmetic(seed, w, n, d, qb, tile):
    """The kernel seam (vlcache._kernels drop-in) on float32 inputs -- the
    reference's own test_kernels.py CASES: the device restates _core.pyx's
    arithmetic per operation, so the statistics equal the C restatement (itself
    bit-identical to the compiled reference) up to glibc expf's rare 1-ulp
    departures from correct rounding (the device rounds exp(double) once)."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((w, d)).astype(np.float32)
    k = rng.standard_normal((n, d)).astype(np.float32)
    got = _kernels.stats_tiled(q, k, qb, 0.01, tile)
    ref = O.stats_tiled(q, k, qb, 0.01, tile)
    np.testing.assert_array_equal(got[0], ref[0])                       # row max: same float32 logits
    np.testing.assert_allclose(got[1], ref[1], rtol=1e-7, atol=0)
    np.testing.assert_allclose(got[2], ref[2], rtol=1e-7, atol=1e-300)
    np.testing.assert_array_equal(got[3], ref[3])
    np.testing.assert_array_equal(got[4], ref[4])
    for g_, n_ in ((1, 33), (4, 512), (7, 3000)):
        qq = rng.standard_normal((g_, d)).astype(np.float32)
        kk = rng.standard_normal((n_, d)).astype(np.float32)
        vv = rng.standard_normal((n_, d)).astype(np.float32)
        np.testing.assert_allclose(_kernels.decode_step(qq, kk, vv), O.decode_step(qq, kk, vv), rtol=1e-6,
                                   atol=1e-7)
