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
