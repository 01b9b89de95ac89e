"""Edge cases of the sm_100a path against the CPU oracle (bf16-in protocol).

Windows that straddle 64-row halves and heads, single-row windows, prefill-
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
    (2, 8, 2, 64, 300, 12, 0.1, 0.1),      # 48-row slots: heads straddle 64-row halves
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


def test_register_path_tie_runs_and_ragged_sizes():
    """n <= 3072 keeps keys in registers: runs of > 32 equal scores at the
    k-th position (the uniform-bucket exit), sizes off the 512-thread grid,
    k = 1 / n, and a reserve covering the whole budget (no key chosen by score)."""
    import paper_2410_23317_b200 as vl

    rng = np.random.default_rng(5)
    for n in (1, 31, 512, 513, 1999, 2960, 3072):
        for vals in (3, 40, 0):
            s = rng.integers(0, vals, n).astype(np.float64) if vals else rng.standard_normal(n)
            for k in sorted({1, n // 3, n // 2, n - 1, n} - {0}):   # the API rejects k = 0
                for frac in (0.0, 0.1, 1.0):
                    np.testing.assert_array_equal(vl.evict(s, k, vl.EvictionConfig(frac)), O.evict(s, k, frac),
                                                  err_msg=f"n={n} vals={vals} k={k} frac={frac}")


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
    got = _kernels.stats_tiled_tc(q, k, qb, 0.01, 128)
    ref = O.stats_tiled(q, k, qb, 0.01, 128)
    np.testing.assert_allclose(got[0], ref[0], rtol=1e-6)
    np.testing.assert_allclose(got[2], ref[2], rtol=1e-5, atol=1e-12)
    np.testing.assert_array_equal(got[3], ref[3])
    np.testing.assert_array_equal(got[4], ref[4])


def test_full_m7b_generator_trace_matches_oracle():
    """BASELINE configs[1] in full: LLaVA-1.6-Mistral-7B shapes, 32 layers,
    generator trace (bf16-in) -- counts, budgets, kept sets and 4 decode steps
    against the oracle (threaded over (layer, head) like the reference allows)."""
    import os

    L, HQ, HKV, D, M, TAU, N = 32, 32, 8, 128, 2960, 64, 4
    spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M,
                   post_vision_len=TAU, decode_len=N, seed=0)
    host, dv = make_inputs(spec, TAU)
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), decode_steps=N, keep_scores=True)
    eng.compress(dv["q_win"], dv["keys"], dv["values"])
    threads = len(os.sched_getaffinity(0))
    ref = O.compression_pass(host[0]["q_win"], host[0]["keys"], M, HQ // HKV, threads=threads)
    ref_below = np.array([[ref["stats"][(l, h)][3].sum() for h in range(HQ)] for l in range(L)])
    np.testing.assert_array_equal(eng.below_head.view(L, HQ).cpu().numpy(), ref_below)
    np.testing.assert_array_equal(eng.gamma_mean.cpu().numpy(), ref["gamma_mean"])
    np.testing.assert_array_equal(eng.kept_counts.cpu().numpy(), ref["kept_counts"])
    kept = eng.kept_sets()[0]
    check_kept_sets(kept, ref["kept"], ref["scores"], ref["kept_counts"])
    outs = []
    eng.decode(dv["q_dec"], dv["keys"], dv["values"], outputs=outs)
    ref_out = O.decode_sequence(host[0]["q_dec"], host[0]["keys"], host[0]["values"], kept, M, HQ // HKV, N,
                                layers=[0, 13, 31])
    for s in range(N):
        got = outs[s].view(L, HQ, D).cpu().numpy()
        for l in (0, 13, 31):
            np.testing.assert_allclose(got[l], ref_out[s][l], rtol=1e-4, atol=1e-5)


def test_head_sharded_budgets_equal_unsharded():
    """KV-head sharding (parallel.HeadShard): each 'rank' runs K1 on its KV
    heads only; the zero-padded int64 counts summed over ranks (what the NCCL
    all-reduce does) give bit-identical budgets and kept sets to one device."""
    from paper_2410_23317_b200.parallel import HeadShard

    L, HQ, HKV, D, M, TAU, WORLD = 2, 56, 8, 128, 1500, 64, 4
    spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M,
                   post_vision_len=TAU, decode_len=1, seed=9)
    host, dv = make_inputs(spec, TAU)
    full = VLCache(Shape(1, L, HQ, HKV, D, M, TAU))
    full.compress(dv["q_win"], dv["keys"])
    counts = torch.zeros((1, L, HQ), dtype=torch.int64, device="cuda")
    locals_ = []
    for r in range(WORLD):
        sh = HeadShard(r, WORLD, HKV, HQ // HKV)
        (klo, khi), (qlo, qhi) = sh.kv_range, sh.q_range
        eng = VLCache(Shape(1, L, qhi - qlo, khi - klo, D, M, TAU), head_shard=sh)
        eng.score_stats(dv["q_win"][:, :, qlo:qhi].contiguous(), dv["keys"][:, :, klo:khi].contiguous())
        counts[:, :, qlo:qhi] += eng.below_head.view(1, L, qhi - qlo)
        locals_.append((eng, klo, khi, qlo, qhi))
    np.testing.assert_array_equal(counts.view(-1).cpu().numpy(), full.below_head.cpu().numpy())
    for eng, klo, khi, qlo, qhi in locals_:
        eng.below_alloc = counts.reshape(-1)
        eng.allocate()
        eng.select()
        np.testing.assert_array_equal(eng.kept_counts.cpu().numpy(), full.kept_counts.cpu().numpy())
        np.testing.assert_array_equal(eng.gamma_mean.cpu().numpy(), full.gamma_mean.cpu().numpy())
        mine, ref = eng.kept_sets()[0], full.kept_sets()[0]
        for l in range(L):
            for kv in range(khi - klo):
                np.testing.assert_array_equal(mine[l][kv], ref[l][klo + kv])


@pytest.mark.parametrize("alpha", [0.01, 0.2, 1.0])
def test_sweep_16k_context_properties(alpha):
    """SWEEP shapes (16,384-token prompt) on 2 layers: budgets against the
    oracle allocation of the device's own gamma' and against the oracle's own
    stats pass (counts, k_l, kept indices), sorted kept sets with the recent
    reserve, and decode against the oracle on one layer."""
    import math

    L, HQ, HKV, D, M, TAU = 2, 32, 8, 128, 16384, 64
    spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M,
                   post_vision_len=TAU, decode_len=2, seed=2)
    host, dv = make_inputs(spec, TAU)
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), alpha=alpha, decode_steps=2, keep_scores=True)
    eng.compress(dv["q_win"], dv["keys"], dv["values"])
    gm = eng.gamma_mean.cpu().numpy()
    _, _, kc = O.allocate_sparsity_aware(gm, alpha, M)
    counts = eng.kept_counts.cpu().numpy()
    np.testing.assert_array_equal(counts, kc)
    # and against the oracle's own stats pass: counts, budgets and kept indices
    import os

    ref = O.compression_pass(host[0]["q_win"], host[0]["keys"], M, HQ // HKV, alpha=alpha,
                             threads=len(os.sched_getaffinity(0)))
    ref_below = np.array([[ref["stats"][(l, h)][3].sum() for h in range(HQ)] for l in range(L)])
    np.testing.assert_array_equal(eng.below_head.view(L, HQ).cpu().numpy(), ref_below)
    np.testing.assert_array_equal(counts, ref["kept_counts"])
    check_kept_sets(eng.kept_sets()[0], ref["kept"], ref["scores"], ref["kept_counts"])
    sc = eng.scores.view(L, HKV, M).cpu().numpy()
    kept = eng.kept_sets()[0]
    for l in range(L):
        for kv in range(HKV):
            np.testing.assert_array_equal(kept[l][kv], O.evict(sc[l, kv], int(counts[l]), 0.1))
    outs = []
    eng.decode(dv["q_dec"], dv["keys"], dv["values"], outputs=outs)
    ref_out = O.decode_sequence(host[0]["q_dec"], host[0]["keys"], host[0]["values"], kept, M, HQ // HKV, 2,
                                layers=[1])
    np.testing.assert_allclose(outs[1].view(L, HQ, D)[1].cpu().numpy(), ref_out[1][1], rtol=1e-4, atol=1e-5)
    assert math.isclose(eng.beta_pre.sum().item(), alpha * L, rel_tol=1e-12)


def test_run_from_host_matches_device_path():
    """The host-input entry point (pinned host tensors, values gathered
    zero-copy over PCIe) gives the device path's budgets and outputs."""
    L, HQ, HKV, D, M, TAU, N = 2, 8, 2, 128, 700, 32, 5
    spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M,
                   post_vision_len=TAU, decode_len=N, seed=12)
    host, dv = make_inputs(spec, TAU)
    ref = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), decode_steps=N)
    ref.compress(dv["q_win"], dv["keys"], dv["values"])
    out_ref = ref.decode(dv["q_dec"], dv["keys"], dv["values"]).clone()
    pin = lambda t: t.cpu().contiguous().pin_memory()  # noqa: E731
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), decode_steps=N)
    counts, out, copied = eng.run_from_host(
        pin(dv["q_win"]), pin(dv["keys"][:, :, :, :M]), pin(dv["values"][:, :, :, :M]), pin(dv["q_dec"]),
        pin(dv["keys"][:, :, :, M:M + N]), pin(dv["values"][:, :, :, M:M + N]))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(counts.numpy(), ref.kept_counts.cpu().numpy())
    np.testing.assert_array_equal(out.numpy(), out_ref.cpu().numpy())
    assert eng.zero_copy_bytes(counts) == int(counts.sum()) * HKV * D * 2


def test_trace_file_to_run_from_host(tmp_path):
    """A .vlct trace written to disk, read back memory-mapped and staged with
    trace.engine_inputs drives run_from_host to the device path's results."""
    from paper_2410_23317_b200.trace import engine_inputs, generate_trace, read_trace, write_trace

    L, HQ, HKV, D, M, TAU, N = 2, 8, 2, 64, 300, 32, 3
    spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M,
                   post_vision_len=TAU, decode_len=N, seed=4)
    tr, _ = generate_trace(spec)
    write_trace(tr, tmp_path / "t.vlct")
    back = read_trace(tmp_path / "t.vlct", mmap=True)
    ins = engine_inputs(back, TAU)
    ref = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), decode_steps=N)
    dev = [t.cuda() for t in ins]
    keys = torch.cat([dev[1], dev[4]], dim=3).contiguous()
    vals = torch.cat([dev[2], dev[5]], dim=3).contiguous()
    ref.compress(dev[0], keys, vals)
    out_ref = ref.decode(dev[3], keys, vals).clone()
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), decode_steps=N)
    counts, out, _ = eng.run_from_host(*ins)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(counts.numpy(), ref.kept_counts.cpu().numpy())
    np.testing.assert_array_equal(out.numpy(), out_ref.cpu().numpy())


def test_exact_mode_overflow_raises():
    """Exact mode with a re-decision list too small for Gaussian logits (many
    entries near the threshold): check() raises ExactnessError instead of
    passing fp32 decisions silently; with room for every entry the counts
    equal the oracle's."""
    from paper_2410_23317_b200 import ExactnessError

    rng = np.random.default_rng(5)
    L, HQ, HKV, D, M, TAU = 1, 8, 2, 128, 1500, 64
    q = bf16(rng.standard_normal((1, L, HQ, TAU, D)) * 2.0)
    k = bf16(rng.standard_normal((1, L, HKV, M, D)))
    dq, dk = (torch.from_numpy(x).cuda().to(torch.bfloat16).contiguous() for x in (q, k))
    small = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), exact_capacity=8)
    small.compress(dq, dk)
    with pytest.raises(ExactnessError):
        small.check()
    st = small.exact_stats()
    assert st["overflow"] > 0 and st["listed"] > 8
    big = VLCache(Shape(1, L, HQ, HKV, D, M, TAU), exact_capacity=st["listed"] + 1024)
    big.compress(dq, dk)
    big.check()
    assert big.exact_stats()["overflow"] == 0
    ref = O.compression_pass([q[0, 0]], [k[0, 0]], M, HQ // HKV)
    ref_below = np.array([ref["stats"][(0, h)][3].sum() for h in range(HQ)])
    np.testing.assert_array_equal(big.below_head.cpu().numpy(), ref_below)


def test_exact_mode_margin_check():
    """Exact mode's fixed margins are verified at run time: the fix-ups record
    the largest tensor-core logit / row-max errors they observe.  On Gaussian
    logits (many listed entries) those stay far inside the margins; a status
    word past a margin makes check() raise ExactnessError."""
    from paper_2410_23317_b200 import ExactnessError
    from paper_2410_23317_b200.engine import EXACT_BAND_LOGIT

    rng = np.random.default_rng(6)
    L, HQ, HKV, D, M, TAU = 1, 8, 2, 128, 1500, 64
    q = bf16(rng.standard_normal((1, L, HQ, TAU, D)) * 2.0)
    k = bf16(rng.standard_normal((1, L, HKV, M, D)))
    dq, dk = (torch.from_numpy(x).cuda().to(torch.bfloat16).contiguous() for x in (q, k))
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, TAU))
    eng.compress(dq, dk)
    eng.check()
    st = eng.exact_stats()
    assert st["listed"] > 100 and st["margin_ok"]
    assert 0.0 < st["max_logit_err"] < EXACT_BAND_LOGIT / 50, st
    eng.exact_ws[20:24].view(torch.float32).fill_(EXACT_BAND_LOGIT / 4)   # [5]: a logit error past the margin
    with pytest.raises(ExactnessError):
        eng.check()


@pytest.mark.parametrize("tau", [12, 40])
def test_exact_mode_chunk_listing_straddling_heads(tau):
    """Gaussian logits put many entries in exact mode's band; with windows of
    12 / 40 rows a 32-row listing chunk spans two heads (the per-row head count
    path).  Below counts per head still equal the oracle's exactly."""
    rng = np.random.default_rng(7 + tau)
    L, HQ, HKV, D, M = 2, 8, 2, 128, 700
    q = bf16(rng.standard_normal((1, L, HQ, tau, D)) * 2.0)
    k = bf16(rng.standard_normal((1, L, HKV, M, D)))
    dq, dk = (torch.from_numpy(x).cuda().to(torch.bfloat16).contiguous() for x in (q, k))
    eng = VLCache(Shape(1, L, HQ, HKV, D, M, tau))
    eng.compress(dq, dk)
    eng.check()
    assert eng.exact_stats()["listed"] > 0
    ref = O.compression_pass([q[0, l] for l in range(L)], [k[0, l] for l in range(L)], M, HQ // HKV)
    ref_below = np.array([[ref["stats"][(l, h)][3].sum() for h in range(HQ)] for l in range(L)])
    np.testing.assert_array_equal(eng.below_head.view(L, HQ).cpu().numpy(), ref_below)
    np.testing.assert_array_equal(eng.kept_counts.cpu().numpy(), ref["kept_counts"])


def test_decode_rejects_bad_inputs():
    """K5 does pointer arithmetic with the input shapes: non-contiguous views,
    wrong dtypes and mismatched K/V raise ValidationError before any launch."""
    from paper_2410_23317_b200 import ValidationError

    spec = GenSpec(num_layers=1, num_query_heads=4, num_kv_heads=2, head_dim=64, prompt_len=200,
                   post_vision_len=16, decode_len=3, seed=8)
    host, dv = make_inputs(spec, 16)
    eng = VLCache(Shape(1, 1, 4, 2, 64, 200, 16), decode_steps=3)
    eng.compress(dv["q_win"], dv["keys"], dv["values"])
    qd, k, v = dv["q_dec"], dv["keys"], dv["values"]
    with pytest.raises(ValidationError):
        eng.decode_step(qd.transpose(3, 4).contiguous().transpose(3, 4), k, v, 0)   # non-contiguous
    with pytest.raises(ValidationError):
        eng.decode_step(qd.float(), k, v, 0)
    with pytest.raises(ValidationError):
        eng.decode_step(qd, k, v[:, :, :, :-1].contiguous(), 0)                    # V shorter than K
    with pytest.raises(ValidationError):
        eng.gather(k, v[:, :, :, :-1].contiguous())
    eng.decode(qd, k, v)   # the valid call still works


def test_decode_graph_cache_keys_on_shapes():
    """Two decode-query tensors that reuse one allocation but differ in their
    number of decode rows (so in K5's stride) must not share a captured graph."""
    spec = GenSpec(num_layers=1, num_query_heads=4, num_kv_heads=2, head_dim=64, prompt_len=200,
                   post_vision_len=16, decode_len=6, seed=10)
    host, dv = make_inputs(spec, 16)
    eng = VLCache(Shape(1, 1, 4, 2, 64, 200, 16), decode_steps=3)
    eng.compress(dv["q_win"], dv["keys"], dv["values"])
    buf = torch.empty(dv["q_dec"].numel(), dtype=torch.bfloat16, device="cuda")
    q6 = buf.view(dv["q_dec"].shape)
    q6.copy_(dv["q_dec"])
    eng.decode(q6, dv["keys"], dv["values"], n_steps=1)
    eng.decode(q6, dv["keys"], dv["values"], first_step=1, n_steps=1)        # graph with the 6-row stride
    q3 = buf[: dv["q_dec"][:, :, :, :3].numel()].view(1, 1, 4, 3, 64)       # same pointer, 3 rows
    q3.copy_(dv["q_dec"][:, :, :, :3])
    eng.decode(q3, dv["keys"], dv["values"], first_step=1, n_steps=1)        # must not replay that graph
    ref = VLCache(Shape(1, 1, 4, 2, 64, 200, 16), decode_steps=3)
    ref.compress(dv["q_win"], dv["keys"], dv["values"])
    ref.decode(dv["q_dec"], dv["keys"], dv["values"], graph=False, n_steps=2)
    np.testing.assert_array_equal(eng.out.cpu().numpy(), ref.out.cpu().numpy())
