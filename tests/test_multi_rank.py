"""N>1 host logic on CPU: world_size-2 gloo ranks.

KV-head sharding must reproduce the unsharded budgets bit for bit: each rank
scores only its heads, the integer below-threshold counts are summed across
ranks (parallel.exchange_head_counts), and every rank then allocates on
identical counts.  The per-head counts here come from the CPU oracle (the
checker); on the GPU box the same exchange runs over NCCL on K1's output.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_23317_b200.parallel import HeadShard, exchange_head_counts, shard_batch

M, TAU, HQ, HKV, L, D = 160, 16, 8, 4, 3, 32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    from paper_2410_23317_b200.trace import GenSpec, iter_layers, round_to_bf16

    spec = GenSpec(num_layers=L, num_query_heads=HQ, num_kv_heads=HKV, head_dim=D, prompt_len=M,
                   post_vision_len=TAU, decode_len=1, seed=3)
    qs, ks = [], []
    for k, q in iter_layers(spec, keep_prompt_rows=TAU):
        ks.append(round_to_bf16(k))
        qs.append(round_to_bf16(q[:, :TAU]))
    return qs, ks


def _head_counts(qs, ks, heads):
    from oracle import oracle as O

    g = HQ // HKV
    out = np.zeros((1, L, len(heads)), dtype=np.int64)
    for l in range(L):
        for j, h in enumerate(heads):
            st = O.stats_tiled(qs[l][h], ks[l][h // g, :M], M - TAU, 0.01, 128)
            out[0, l, j] = st[3].sum()
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = HeadShard(rank=rank, world=world, num_kv_heads=HKV, group_size=HQ // HKV)
        qs, ks = _inputs()
        lo, hi = shard.q_range
        local = torch.from_numpy(_head_counts(qs, ks, range(lo, hi)))
        full = exchange_head_counts(local, shard)
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


def test_head_sharded_counts_equal_unsharded_and_budgets_bit_exact():
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    qs, ks = _inputs()
    ref = _head_counts(qs, ks, range(HQ))
    np.testing.assert_array_equal(got[0], ref)
    np.testing.assert_array_equal(got[1], ref)
    # budgets from the exchanged counts == budgets of the unsharded oracle pass
    causal = TAU * (M - TAU + 1) + TAU * (TAU - 1) // 2
    gamma = got[0][0] / causal
    res = O.compression_pass(qs, ks, M, HQ // HKV, tile=128)
    np.testing.assert_array_equal(gamma, res["gamma"])
    pre, beta, kept = O.allocate_sparsity_aware(gamma.mean(axis=1), 0.1, M)
    np.testing.assert_array_equal(kept, res["kept_counts"])


def test_shard_helpers():
    for batch in (1, 5, 8, 13):
        for world in (1, 2, 4, 8):
            ranges = [shard_batch(batch, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    hs = [HeadShard(r, 4, 8, 7) for r in range(4)]
    assert [h.kv_range for h in hs] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    assert hs[3].q_range == (42, 56) and hs[0].num_query_heads == 56
    from paper_2410_23317_b200.errors import ValidationError

    with pytest.raises(ValidationError):
        HeadShard(0, 3, 8, 7)


# ---------------------------------------------------------------- GPU, 2 ranks on one device
GL, GHQ, GHKV, GD, GM, GTAU, GN = 3, 56, 8, 128, 1200, 64, 4


def _gpu_inputs():
    from paper_2410_23317_b200.trace import GenSpec, iter_layers, round_to_bf16, synthesize_values

    spec = GenSpec(num_layers=GL, num_query_heads=GHQ, num_kv_heads=GHKV, head_dim=GD, prompt_len=GM,
                   post_vision_len=GTAU, decode_len=GN, seed=17)
    qw, qd, ks = [], [], []
    for k, q in iter_layers(spec, keep_prompt_rows=GTAU):
        ks.append(round_to_bf16(k))
        q = round_to_bf16(q)
        qw.append(q[:, :GTAU])
        qd.append(q[:, GTAU:])
    vs = [round_to_bf16(v) for v in synthesize_values(spec)]
    dev = lambda a: torch.from_numpy(np.stack(a)[None].copy()).cuda().to(torch.bfloat16).contiguous()  # noqa: E731
    return dev(qw), dev(qd), dev(ks), dev(vs)


def _gpu_worker(rank, world, port, q):
    """One rank of a KV-head-sharded engine (the real VLCache(head_shard=...)
    path: K1 on its heads, the count exchange, K2-K4, then the decode)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_23317_b200.engine import Shape, VLCache

        torch.cuda.set_device(0)
        shard = HeadShard(rank=rank, world=world, num_kv_heads=GHKV, group_size=GHQ // GHKV)
        (klo, khi), (qlo, qhi) = shard.kv_range, shard.q_range
        qw, qd, k, v = _gpu_inputs()
        qw, qd = qw[:, :, qlo:qhi].contiguous(), qd[:, :, qlo:qhi].contiguous()
        k, v = k[:, :, klo:khi].contiguous(), v[:, :, klo:khi].contiguous()
        eng = VLCache(Shape(1, GL, qhi - qlo, khi - klo, GD, GM, GTAU), decode_steps=GN, head_shard=shard)
        eng.compress(qw, k, v)
        eng.decode(qd, k, v)
        torch.cuda.synchronize()
        eng.check()
        q.put((rank, eng.kept_counts.cpu().numpy(), eng.gamma_mean.cpu().numpy(), eng.kept_sets()[0],
               eng.out.view(GL, qhi - qlo, GD).cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_head_sharded_engine_two_ranks_equals_unsharded():
    """Two processes on one GPU (gloo, counts staged through the host) drive
    the real head-sharded engine end to end; budgets, gamma', kept sets and
    decode outputs equal the unsharded engine's."""
    from paper_2410_23317_b200.engine import Shape, VLCache

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r, *rest = q.get(timeout=300)
        got[r] = rest
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    qw, qd, k, v = _gpu_inputs()
    full = VLCache(Shape(1, GL, GHQ, GHKV, GD, GM, GTAU), decode_steps=GN)
    full.compress(qw, k, v)
    full.decode(qd, k, v)
    ref_sets = full.kept_sets()[0]
    ref_out = full.out.view(GL, GHQ, GD).cpu().numpy()
    for r in range(2):
        counts, gm, sets, out = got[r]
        np.testing.assert_array_equal(counts, full.kept_counts.cpu().numpy())
        np.testing.assert_array_equal(gm, full.gamma_mean.cpu().numpy())
        shard = HeadShard(rank=r, world=2, num_kv_heads=GHKV, group_size=GHQ // GHKV)
        (klo, khi), (qlo, qhi) = shard.kv_range, shard.q_range
        for l in range(GL):
            for kv in range(khi - klo):
                np.testing.assert_array_equal(sets[l][kv], ref_sets[l][klo + kv])
        np.testing.assert_array_equal(out, ref_out[:, qlo:qhi])
