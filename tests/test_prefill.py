"""Row f2 (prefill attention): oracle restatement and the B200 kernel against
the reference's own bench._prefill_layer (tests/golden/make_prefill_golden.py).

The oracle (float32 numpy, same tiling) must match the reference bit for bit.
The device kernel forms P in bf16 for the P V product (as every tensor-core
attention): outputs agree to 2e-2 absolute on unit-variance values (|P| error
<= 2^-9 relative per weight); the row statistics it emits equal K1's.
"""
import os
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_2410_23317_b200.trace import round_to_bf16

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_prefill_golden import CASES, inputs  # noqa: E402


@pytest.fixture(scope="module")
def pg():
    return np.load(os.path.join(HERE, "golden", "prefill_golden.npz"))


@pytest.mark.parametrize("case", CASES)
def test_oracle_prefill_matches_reference(pg, case):
    seed, h, hkv, d, m, tile = case
    q, k, v = inputs(seed, h, hkv, d, m, round_to_bf16)
    np.testing.assert_array_equal(O.prefill_layer(q, k, v, m, tile), pg[f"c{seed}_out"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_prefill_matches_reference(pg, case):
    from paper_2410_23317_b200.prefill import prefill_attention

    seed, h, hkv, d, m, tile = case
    q, k, v = inputs(seed, h, hkv, d, m, round_to_bf16)
    got = prefill_attention(q, k, v, m, tile)
    want = pg[f"c{seed}_out"]
    assert got.shape == want.shape and np.isfinite(got).all()
    np.testing.assert_allclose(got, want, atol=2e-2, rtol=0)
    assert np.abs(got - want).mean() < 2e-3


@pytest.mark.gpu
def test_gpu_prefill_stats_equal_k1():
    """The prefill's row max equals K1's for the window rows (same tensor-core
    dots); row sums agree to float32 rounding of a different partial order."""
    import torch

    from paper_2410_23317_b200.engine import Shape, VLCache
    from paper_2410_23317_b200.prefill import prefill

    B, L, HQ, HKV, D, M, W = 1, 2, 8, 2, 128, 700, 64
    g = torch.Generator(device="cuda").manual_seed(3)
    q = (torch.randn((B, L, HQ, M, D), device="cuda", generator=g) * 1.5).to(torch.bfloat16)
    k = torch.randn((B, L, HKV, M, D), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((B, L, HKV, M, D), device="cuda", generator=g).to(torch.bfloat16)
    _, rmax, rsum = prefill(q, k, v, M)
    eng = VLCache(Shape(B, L, HQ, HKV, D, M, W), exact=False)
    eng.score_stats(q[:, :, :, M - W:].contiguous(), k)
    torch.cuda.synchronize()
    k1_max = eng.row_max.view(B, L, HQ, W)
    k1_sum = eng.row_sum.view(B, L, HQ, W)
    assert torch.equal(rmax[..., M - W:], k1_max)
    # sums: the same exponentials in another partial order (the prefill thread sums
    # its row's 128 keys per tile in four chains) -- the parity bar of SURVEY 8c
    torch.testing.assert_close(rsum[..., M - W:], k1_sum, rtol=1e-5, atol=0)


@pytest.mark.gpu
def test_gpu_prefill_validation():
    import torch

    from paper_2410_23317_b200 import ValidationError
    from paper_2410_23317_b200.prefill import prefill

    q = torch.zeros((1, 1, 2, 16, 96), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(Exception, match="head_dim"):
        prefill(q, q[:, :, :1].contiguous(), q[:, :, :1].contiguous(), 16)
    q = torch.zeros((1, 1, 2, 16, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValidationError, match="m: must be"):
        prefill(q, q, q, 17)


@pytest.mark.gpu
def test_gpu_prefill_compress_equals_compress():
    """Row f2's fusion: K1's column pass on the prefill's own row statistics gives
    the same below counts, budgets and kept sets as the two-pass K1 (generator
    inputs, 4 layers of the M7B shapes; exact mode)."""
    import torch

    import bench
    from paper_2410_23317_b200.engine import Shape, VLCache

    c = bench.CFG
    L, m, w = 4, c["prompt_len"], c["tau"]
    qw, qd, ks, vs = bench.synth_inputs(1, 0, m, layers=L)
    dev = lambda a: torch.from_numpy(a).to(torch.bfloat16).cuda()  # noqa: E731
    q_all, keys, values = dev(qw), dev(ks), dev(vs)
    shape = Shape(1, L, c["q_heads"], c["kv_heads"], c["head_dim"], m, w)
    a = VLCache(shape, alpha=c["alpha"], decode_steps=4)
    a.compress(q_all[:, :, :, m - w:m].contiguous(), keys, values)
    b = VLCache(shape, alpha=c["alpha"], decode_steps=4)
    out = b.prefill_compress(q_all, keys, values)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    assert torch.equal(a.below_head, b.below_head)
    assert torch.equal(a.kept_counts, b.kept_counts)
    torch.testing.assert_close(b.row_sum, a.row_sum, rtol=1e-5, atol=0)
    assert torch.equal(a.row_max, b.row_max)
    ka, kb = a.kept_sets(), b.kept_sets()
    diff = sum(int((x != y).sum()) if x.shape == y.shape else 10**6
               for la, lb in zip(ka[0], kb[0]) for x, y in zip(la, lb))
    assert diff == 0


@pytest.mark.gpu
@pytest.mark.parametrize("B,L,HQ,HKV,D,M,W", [(2, 2, 8, 2, 64, 700, 64), (1, 2, 4, 4, 128, 333, 32)])
def test_gpu_prefill_compress_random_inputs(B, L, HQ, HKV, D, M, W):
    """Fusion on dense near-threshold mass (random logits; exact mode re-decides
    many entries): identical counts and budgets; kept sets equal up to score
    near-ties at the boundary (the mass uses max*log2e instead of raw max * c1)."""
    import torch

    from paper_2410_23317_b200.engine import Shape, VLCache
    from test_gpu_parity import check_kept_sets

    g = torch.Generator(device="cuda").manual_seed(11)
    q = (torch.randn((B, L, HQ, M + 5, D), device="cuda", generator=g) * 1.5).to(torch.bfloat16)
    k = torch.randn((B, L, HKV, M + 5, D), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((B, L, HKV, M + 5, D), device="cuda", generator=g).to(torch.bfloat16)
    shape = Shape(B, L, HQ, HKV, D, M, W)
    a = VLCache(shape, alpha=0.2, decode_steps=2, keep_scores=True)
    a.compress(q[:, :, :, M - W:M].contiguous(), k, v)
    b = VLCache(shape, alpha=0.2, decode_steps=2)
    out = b.prefill_compress(q, k, v)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    assert torch.equal(a.below_head, b.below_head)
    assert torch.equal(a.kept_counts, b.kept_counts)
    counts = a.kept_counts.view(B, L).cpu().numpy()
    scores = a.scores.view(B, L, HKV, M).cpu().numpy()
    ka, kb = a.kept_sets(), b.kept_sets()
    for bb in range(B):
        check_kept_sets(kb[bb], ka[bb], scores[bb], counts[bb])


def _prefill_fuzz(n=10, seed=77):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        hkv = int(rng.choice([1, 2, 4]))
        out.append((int(rng.integers(0, 1 << 30)), hkv * int(rng.choice([1, 2, 4, 8])), hkv,
                    int(rng.choice([16, 32, 64, 80, 128])), int(rng.integers(1, 700))))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("seed,h,hkv,d,m", _prefill_fuzz())
def test_gpu_prefill_fuzz(seed, h, hkv, d, m):
    """Random shapes (odd head dims padded, single-row prompts, GQA) against the
    oracle's float32 restatement of the reference prefill."""
    from paper_2410_23317_b200.prefill import prefill_attention

    rng = np.random.default_rng(seed)
    q = round_to_bf16(rng.standard_normal((h, m + 2, d)).astype(np.float32) * 1.5)
    k = round_to_bf16(rng.standard_normal((hkv, m + 2, d)).astype(np.float32))
    v = round_to_bf16(rng.standard_normal((hkv, m + 2, d)).astype(np.float32))
    got = prefill_attention(q, k, v, m)
    want = O.prefill_layer(q, k, v, m, 128)
    np.testing.assert_allclose(got, want, atol=2e-2, rtol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("growth", [0.02, 0.2])
def test_gpu_prefill_rescale_path(growth):
    """Key norms growing along the sequence make every later tile's row max
    exceed the reference max by more than 2^8, so the one-pass kernel rescales
    O (tcgen05.ld / scale / st) and the running sums many times per row; the
    output must still match the oracle's reference prefill."""
    from paper_2410_23317_b200.prefill import prefill_attention

    rng = np.random.default_rng(5)
    h, hkv, d, m = 4, 2, 64, 900
    q = round_to_bf16(rng.standard_normal((h, m, d)).astype(np.float32))
    scale = (1.0 + growth * np.arange(m, dtype=np.float32))[None, :, None]
    k = round_to_bf16(rng.standard_normal((hkv, m, d)).astype(np.float32) * scale)
    v = round_to_bf16(rng.standard_normal((hkv, m, d)).astype(np.float32))
    got = prefill_attention(q, k, v, m)
    want = O.prefill_layer(q, k, v, m, 128)
    assert np.isfinite(got).all()
    np.testing.assert_allclose(got, want, atol=2e-2, rtol=0)
