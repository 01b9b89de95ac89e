"""Full-shape synthetic inputs for the BASELINE.json configurations, made in
worker processes (test infrastructure).

The reference generator (trace.iter_layers, a draw-for-draw restatement of
reference trace.py:256-326) is one sequential PCG64 stream per prompt, so the
prompts of a batch are generated in parallel processes.  Each worker writes the
bf16-rounded tensors as raw bf16 bit patterns (uint16 .npy) so the parent can
memory-map them: the device gets them without a float32 copy and the oracle
widens one prompt at a time.
"""

from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

NAMES = ("keys", "values", "q_win", "q_dec")


def _bits(x: np.ndarray) -> np.ndarray:
    from paper_2410_23317_b200.trace import round_to_bf16

    return (round_to_bf16(x).view(np.uint32) >> 16).astype(np.uint16)


def _worker(job):
    spec_kw, w, outdir = job
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    from paper_2410_23317_b200.trace import GenSpec, iter_layers, synthesize_values

    spec = GenSpec(**spec_kw)
    hdr = spec.header()
    L, hq, hkv, d, t = hdr.num_layers, hdr.num_query_heads, hdr.num_kv_heads, hdr.head_dim, hdr.seq_len
    n = hdr.decode_len
    path = {k: os.path.join(outdir, f"s{spec.seed}_{k}.npy") for k in NAMES}
    out = {
        "keys": np.lib.format.open_memmap(path["keys"], mode="w+", dtype=np.uint16, shape=(L, hkv, t, d)),
        "values": np.lib.format.open_memmap(path["values"], mode="w+", dtype=np.uint16, shape=(L, hkv, t, d)),
        "q_win": np.lib.format.open_memmap(path["q_win"], mode="w+", dtype=np.uint16, shape=(L, hq, w, d)),
        "q_dec": np.lib.format.open_memmap(path["q_dec"], mode="w+", dtype=np.uint16, shape=(L, hq, n, d)),
    }
    for l, (k, q) in enumerate(iter_layers(spec, keep_prompt_rows=w)):
        out["keys"][l] = _bits(k)
        out["q_win"][l] = _bits(q[:, :w])
        out["q_dec"][l] = _bits(q[:, w:])
    for l, v in enumerate(synthesize_values(spec)):
        out["values"][l] = _bits(v)
    for a in out.values():
        a.flush()
    return path


def generate_batch(spec, w: int, batch: int, outdir: str, workers: int | None = None):
    """Prompt b uses seed spec.seed + b.  Returns one dict of .npy paths per prompt."""
    import multiprocessing as mp

    jobs = [({**spec.__dict__, "seed": spec.seed + b}, w, str(outdir)) for b in range(batch)]
    n = workers or min(batch, max(1, len(os.sched_getaffinity(0)) // 2))
    if n == 1:
        return [_worker(j) for j in jobs]
    with ProcessPoolExecutor(max_workers=n, mp_context=mp.get_context("spawn")) as pool:
        return list(pool.map(_worker, jobs))


def load_bits(path: str) -> np.ndarray:
    return np.load(path, mmap_mode="r")


def widen(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> float32 (exact)."""
    return (np.asarray(bits).astype(np.uint32) << 16).view(np.float32)


def to_device(paths, name, torch):
    """[B, ...] bf16 CUDA tensor from the prompts' bit arrays (no float32 copy)."""
    first = load_bits(paths[0][name])
    out = torch.empty((len(paths), *first.shape), dtype=torch.bfloat16, device="cuda")
    for b, p in enumerate(paths):
        a = load_bits(p[name])
        for l in range(a.shape[0]):
            out[b, l].copy_(torch.from_numpy(np.array(a[l]).view(np.int16)).view(torch.bfloat16))
    return out
