"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (where /root/reference is mounted):  python tests/golden/make_golden.py
It copies /root/reference/pkg to a scratch dir, builds the reference's compiled
backend with its own setup.py (scratch copy only), imports ``vlcache`` and
records its outputs.  The fixtures are committed; the GPU box never reads
/root/reference.  Tests pin oracle/ (and through it the CUDA path) to them.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"


def load_reference():
    scratch = tempfile.mkdtemp(prefix="vlref_")
    dst = os.path.join(scratch, "pkg")
    shutil.copytree(REF, dst)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=dst,
                   check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(dst, "src"))
    import vlcache  # noqa: E402
    assert vlcache.BACKEND == "compiled", vlcache.BACKEND
    return vlcache


def bf16_round(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# test_kernels.py:55-62 plus two VLM-shaped cases (d=128, GQA-sized windows)
STATS_CASES = [
    (0, 96, 96, 32, 0, 32), (1, 96, 96, 32, 0, 17), (2, 40, 128, 64, 88, 33),
    (3, 4, 256, 32, 252, 64), (4, 1, 64, 16, 63, 4096), (5, 200, 200, 48, 0, 128),
    (6, 64, 700, 128, 636, 128), (7, 32, 624, 64, 592, 128),
]
DECODE_CASES = [(0, 2, 128, 32), (1, 4, 512, 64), (2, 1, 33, 16), (3, 4, 300, 128), (4, 7, 1000, 128)]
TOY = dict(num_layers=4, num_query_heads=8, num_kv_heads=8, head_dim=64, prompt_len=624,
           post_vision_len=32, decode_len=100, seed=0)


def main():
    vl = load_reference()
    from vlcache._kernels import decode_step, stats_tiled

    out = {}
    # 1. kernel known-answer vectors (fp32 random inputs, seeds as in test_kernels._random_case)
    for seed, w, n, d, qb, tile in STATS_CASES:
        rng = np.random.default_rng(seed)
        q = rng.standard_normal((w, d)).astype(np.float32)
        k = rng.standard_normal((n, d)).astype(np.float32)
        for name, val in zip(("row_max", "row_sum", "col_score", "below", "causal"),
                             stats_tiled(q, k, qb, 0.01, tile)):
            out[f"stats{seed}_{name}"] = val
    for seed, g, n, d in DECODE_CASES:
        rng = np.random.default_rng(seed)
        q = rng.standard_normal((g, d)).astype(np.float32)
        k = rng.standard_normal((n, d)).astype(np.float32)
        v = rng.standard_normal((n, d)).astype(np.float32)
        out[f"decode{seed}"] = decode_step(q, k, v)

    # 2. generator pin (conftest.make_spec defaults) and budget / eviction examples
    small = vl.GenSpec(num_layers=2, num_query_heads=4, num_kv_heads=2, head_dim=32, prompt_len=96,
                       post_vision_len=12, decode_len=4, seed=11)
    tr, planted = vl.generate_trace(small)
    out["gen_small_planted"] = planted
    out["gen_small_q_sha"] = np.array([sha(x) for x in tr.queries])
    out["gen_small_k_sha"] = np.array([sha(x) for x in tr.keys])
    out["gen_small_q0"] = tr.queries[0]
    out["gen_small_k1"] = tr.keys[1]

    rng = np.random.default_rng(1002)
    gammas, alphas, pres, betas, keeps = [], [], [], [], []
    for _ in range(200):
        nl = int(rng.integers(1, 61))
        g = rng.uniform(0.0, 0.999, size=nl)
        a = float(rng.uniform(0.01, 1.0))
        m = int(rng.integers(1, 20000))
        al = vl.allocate_sparsity_aware(g, a, m)
        gammas.append(g); alphas.append((a, m)); pres.append(al.beta_preclip)
        betas.append(al.beta); keeps.append(al.kept_counts)
    out["alloc_gamma"] = np.array(gammas, dtype=object)
    out["alloc_alpha_m"] = np.array(alphas)
    out["alloc_pre"] = np.array(pres, dtype=object)
    out["alloc_beta"] = np.array(betas, dtype=object)
    out["alloc_kept"] = np.array(keeps, dtype=object)
    rng = np.random.default_rng(1006)
    ev_scores, ev_args, ev_kept = [], [], []
    for _ in range(200):
        n = int(rng.integers(8, 513))
        k = int(rng.integers(1, n + 1))
        frac = float(rng.choice([0.0, 0.05, 0.1, 0.33, 0.5, 1.0]))
        s = rng.standard_normal(n)
        if rng.random() < 0.3:
            s = np.round(s)
        ev_scores.append(s); ev_args.append((k, frac))
        ev_kept.append(vl.evict(s, k, vl.EvictionConfig(recent_window_frac=frac)))
    out["evict_scores"] = np.array(ev_scores, dtype=object)
    out["evict_args"] = np.array(ev_args)
    out["evict_kept"] = np.array(ev_kept, dtype=object)

    # 3. library-path compression of a bf16-rounded TOY trace (Hkv=8 and Hkv=2):
    #    measure_gamma_mean -> allocate_sparsity_aware -> compress_cache(PostVision)
    for hkv in (8, 2):
        spec = vl.GenSpec(**{**TOY, "num_kv_heads": hkv})
        tr, _ = vl.generate_trace(spec)
        tr = vl.AttentionTrace(header=tr.header, layout=tr.layout,
                               queries=[bf16_round(x) for x in tr.queries],
                               keys=[bf16_round(x) for x in tr.keys])
        sp = vl.post_vision_sparsity(tr)
        gm = vl.measure_gamma_mean(tr)
        alloc = vl.allocate_sparsity_aware(gm, 0.1, tr.header.prompt_len)
        res = vl.compress_cache(tr, alloc, vl.PostVision())
        tag = f"toy{hkv}"
        out[f"{tag}_gamma"] = sp.gamma
        out[f"{tag}_gamma_mean"] = gm
        out[f"{tag}_beta_pre"] = alloc.beta_preclip
        out[f"{tag}_beta"] = alloc.beta
        out[f"{tag}_kept_counts"] = alloc.kept_counts
        out[f"{tag}_kept"] = np.array([[ks.kept for ks in row] for row in res.kept_sets], dtype=object)
        out[f"{tag}_scores"] = np.stack([
            np.stack([vl.score_tokens(tr, l, kv, vl.PostVision()) for kv in range(hkv)])
            for l in range(TOY["num_layers"])])
        # compressed decode, first 3 steps, reference bench._make_seq_buffers/_decode_sequence loop
        values = [bf16_round(v) for v in vl.synthesize_values(vl.BenchSpec(
            prompt_len=TOY["prompt_len"], n_output_tokens=TOY["decode_len"], seed=TOY["seed"],
            num_layers=TOY["num_layers"], num_query_heads=8, num_kv_heads=hkv,
            head_dim=TOY["head_dim"], post_vision_len=TOY["post_vision_len"]))]
        m, g = tr.header.prompt_len, tr.header.group_size
        steps = []
        bufs = {}
        for l in range(TOY["num_layers"]):
            for kv in range(hkv):
                idx = res.kept_sets[l][kv].kept
                bufs[(l, kv)] = [list(tr.keys[l][kv, idx]), list(values[l][kv, idx])]
        for s in range(3):
            per = []
            for l in range(TOY["num_layers"]):
                q_row = np.ascontiguousarray(tr.queries[l][:, m + s])
                o = []
                for kv in range(hkv):
                    kb, vb = bufs[(l, kv)]
                    kb.append(tr.keys[l][kv, m + s]); vb.append(values[l][kv, m + s])
                    o.append(decode_step(q_row[kv * g:(kv + 1) * g], np.array(kb), np.array(vb)))
                per.append(np.concatenate(o))
            steps.append(np.stack(per))
        out[f"{tag}_decode3"] = np.stack(steps)

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
