"""Parity at the BASELINE.json configurations at FULL shape (exact mode on,
the reference generator's inputs, bf16-in):

  Y34B   LLaVA-1.6-34B shapes: L60, Hq56 / Hkv8, d128, m = 10,320
         (16 + 5 x 2,048 visual + 64), tau 64, batch 4, 10 % budget
  VID    32 frames x 196 tokens on Mistral-7B shapes: L32, Hq32 / Hkv8,
         m = 6,352 (16 + 6,272 + 64), batch 8
  SWEEP  Mistral-7B shapes at a 16,384-token prompt, budgets 1/5/10/20/100 %

Each compares, per prompt, against the CPU oracle (oracle.compression_pass, a
restatement of reference bench.py:245-323 over the reference's compiled
kernels' arithmetic, _core.pyx:110-242, pinned to reference golden vectors):
per-head below counts exactly, gamma' and every k_l bit-exactly, column scores
within rtol 1e-5, kept index sets exactly except boundary near-ties
(SURVEY.md section 8c), and the 99-step compressed decode (reference
bench.py:356-372) on sampled layers within rtol 1e-4 / atol 1e-5.
"""

import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen_inputs import generate_batch, load_bits, to_device, widen  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402
from paper_2410_23317_b200.trace import GenSpec  # noqa: E402
from test_gpu_parity import check_kept_sets  # noqa: E402

THREADS = len(os.sched_getaffinity(0))
N_OUT = 100            # output tokens -> 99 decode steps (reference bench.py:361)


def _spec(L, hq, hkv, m, seed):
    return GenSpec(num_layers=L, num_query_heads=hq, num_kv_heads=hkv, head_dim=128, prompt_len=m,
                   post_vision_len=64, decode_len=N_OUT - 1, seed=seed)


def _host(path, name):
    a = load_bits(path[name])
    return [widen(a[l]) for l in range(a.shape[0])]


def _check_prompt(eng, b, path, m, g, L, hq, hkv, alphas=(0.1,), decode_layers=()):
    """One prompt of a batch against the oracle; returns the oracle pass."""
    q_win, keys = _host(path, "q_win"), _host(path, "keys")
    ref = O.compression_pass(q_win, keys, m, g, alpha=alphas[0], threads=THREADS)
    below = np.array([[ref["stats"][(l, h)][3].sum() for h in range(hq)] for l in range(L)])
    np.testing.assert_array_equal(eng.below_head.view(-1, L, hq)[b].cpu().numpy(), below)
    np.testing.assert_array_equal(eng.gamma_mean.view(-1, L)[b].cpu().numpy(), ref["gamma_mean"])
    np.testing.assert_array_equal(eng.kept_counts.view(-1, L)[b].cpu().numpy(), ref["kept_counts"])
    np.testing.assert_allclose(eng.scores.view(-1, L, hkv, m)[b].cpu().numpy(), ref["scores"], rtol=1e-5,
                               atol=1e-12)
    check_kept_sets(eng.kept_sets()[b], ref["kept"], ref["scores"], ref["kept_counts"])
    return ref


def _check_decode(outs, b, path, kept, m, g, L, hq, layers, steps):
    q_dec, keys, values = _host(path, "q_dec"), _host(path, "keys"), _host(path, "values")
    ref_out = O.decode_sequence(q_dec, keys, values, kept, m, g, N_OUT - 1, layers=list(layers),
                                threads=min(THREADS, len(layers)))
    for s in steps:
        got = outs[s].view(-1, L, hq, 128)[b].cpu().numpy()
        for l in layers:
            np.testing.assert_allclose(got[l], ref_out[s][l], rtol=1e-4, atol=1e-5)


def _run_config(tmp_path, L, hq, hkv, m, batch, seed, decode_layers):
    g = hq // hkv
    paths = generate_batch(_spec(L, hq, hkv, m, seed), 64, batch, tmp_path)
    dv = {n: to_device(paths, n, torch) for n in ("q_win", "keys", "values", "q_dec")}
    eng = VLCache(Shape(batch, L, hq, hkv, 128, m, 64), alpha=0.1, decode_steps=N_OUT - 1, keep_scores=True)
    eng.compress(dv["q_win"], dv["keys"], dv["values"])
    eng.check()                      # includes: exact mode's list did not overflow
    st = eng.exact_stats()
    assert st["overflow"] == 0
    outs = []
    eng.decode(dv["q_dec"], dv["keys"], dv["values"], outputs=outs)
    torch.cuda.synchronize()
    kept_all = eng.kept_sets()
    for b in range(batch):
        _check_prompt(eng, b, paths[b], m, g, L, hq, hkv)
        _check_decode(outs, b, paths[b], kept_all[b], m, g, L, hq, decode_layers, (0, 49, N_OUT - 2))
    return st


def test_y34b_full_shape_batch4(tmp_path):
    """BASELINE configs[2] on one device: L60 Hq56 Hkv8 m10320, batch 4."""
    st = _run_config(tmp_path, L=60, hq=56, hkv=8, m=10320, batch=4, seed=100, decode_layers=(0, 59))
    print("exact mode:", st)


def test_vid_full_shape_batch8(tmp_path):
    """BASELINE configs[3] on one device: 32 frames x 196 tokens, L32 Hq32 Hkv8, batch 8."""
    st = _run_config(tmp_path, L=32, hq=32, hkv=8, m=6352, batch=8, seed=200, decode_layers=(0, 31))
    print("exact mode:", st)


def test_sweep_16k_all_budgets(tmp_path):
    """BASELINE configs[4]: 16,384-token prompt, 32 layers, budgets 1/5/10/20/100 %:
    one oracle stats pass, then per budget the allocation, kept indices and the
    99-step decode against the oracle's."""
    L, hq, hkv, m = 32, 32, 8, 16384
    g = hq // hkv
    paths = generate_batch(_spec(L, hq, hkv, m, 300), 64, 1, tmp_path)
    dv = {n: to_device(paths, n, torch) for n in ("q_win", "keys", "values", "q_dec")}
    ref = O.compression_pass(_host(paths[0], "q_win"), _host(paths[0], "keys"), m, g, threads=THREADS)
    below = np.array([[ref["stats"][(l, h)][3].sum() for h in range(hq)] for l in range(L)])
    for alpha in (0.01, 0.05, 0.1, 0.2, 1.0):
        eng = VLCache(Shape(1, L, hq, hkv, 128, m, 64), alpha=alpha, decode_steps=N_OUT - 1, keep_scores=True)
        eng.compress(dv["q_win"], dv["keys"], dv["values"])
        eng.check()
        np.testing.assert_array_equal(eng.below_head.view(L, hq).cpu().numpy(), below)
        np.testing.assert_array_equal(eng.gamma_mean.cpu().numpy(), ref["gamma_mean"])
        _, _, counts = O.allocate_sparsity_aware(ref["gamma_mean"], alpha, m)
        np.testing.assert_array_equal(eng.kept_counts.cpu().numpy(), counts)
        assert math.isclose(eng.beta_pre.sum().item(), alpha * L, rel_tol=1e-12)
        np.testing.assert_allclose(eng.scores.view(L, hkv, m).cpu().numpy(), ref["scores"], rtol=1e-5, atol=1e-12)
        kept_ref = [[O.evict(ref["scores"][l, kv], int(counts[l]), 0.1) for kv in range(hkv)] for l in range(L)]
        kept = eng.kept_sets()[0]
        check_kept_sets(kept, kept_ref, ref["scores"], counts)
        outs = []
        eng.decode(dv["q_dec"], dv["keys"], dv["values"], outputs=outs)
        _check_decode(outs, 0, paths[0], kept, m, g, L, hq, (0, L - 1), (N_OUT - 2,))
        del eng, outs
