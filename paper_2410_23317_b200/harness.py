"""The reference's benchmark harness on the B200 (pkg/src/vlcache/bench.py).

Same names, fields, validation and report semantics as the reference module:
``BenchSpec``, ``BenchReport``, ``run_bench``, ``OverheadReport``,
``stats_overhead``, ``latency_throughput_curve``, ``estimate_bytes``,
``kv_cache_bytes``.  The work runs on the device: the prefill in
``vlc_prefill``, the compression pass (statistics window, budget, scoring
policy, eviction) in K1-K3, the full and compressed decodes as K4 + the K5
CUDA graph.  Times are wall-clock seconds around synchronised device work
with the trace already resident on the device, as the reference's are with
it resident in host memory.  ``threads`` and ``tile`` are the reference's
CPU knobs: validated, not used.  Memory accounting keeps the reference's
closed form (float32 bytes) so reports compare field for field.
"""

from __future__ import annotations

import math
import statistics
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._kernels import BACKEND
from .attention import DEFAULT_P
from .budget import allocate_sparsity_aware, allocate_uniform
from .errors import SpecTooLargeError, ValidationError
from .trace import AttentionTrace, GenSpec, generate_trace, round_to_bf16, synthesize_values

_BUDGET_MODES = ("sparsity_aware", "uniform")
_POLICY_NAMES = ("vlcache", "h2o", "sliding", "streaming")


@dataclass(frozen=True)
class BenchSpec:
    """reference bench.py:33-104."""

    prompt_len: int
    batch_size: int = 1
    n_output_tokens: int = 100
    alpha: float = 0.1
    policy: str = "vlcache"
    repeats: int = 3
    warmup: int = 1
    seed: int = 0
    num_layers: int = 2
    num_query_heads: int = 4
    num_kv_heads: int = 2
    head_dim: int = 64
    post_vision_len: int = 64
    stats_window: int = 50
    budget: str = "sparsity_aware"
    threads: int = 1
    tile: int = 256
    p: float = DEFAULT_P
    recent_window_frac: float = 0.10
    max_bytes: int = 6 * 1024**3

    def __post_init__(self) -> None:
        for name in ("prompt_len", "batch_size", "n_output_tokens", "repeats", "warmup", "num_layers",
                     "num_query_heads", "num_kv_heads", "head_dim", "threads", "tile"):
            if getattr(self, name) < 1:
                raise ValidationError(f"{name}: must be >= 1, got {getattr(self, name)}")
        if self.repeats < 3:
            raise ValidationError(f"repeats: must be >= 3, got {self.repeats}")
        if not 0.0 < self.alpha <= 1.0:
            raise ValidationError(f"alpha: must be in (0, 1], got {self.alpha}")
        if self.policy not in _POLICY_NAMES:
            raise ValidationError(f"policy: must be one of {_POLICY_NAMES}, got {self.policy!r}")
        if self.budget not in _BUDGET_MODES:
            raise ValidationError(f"budget: must be one of {_BUDGET_MODES}, got {self.budget!r}")
        if not 0 <= self.post_vision_len <= self.prompt_len:
            raise ValidationError(f"post_vision_len: must be in [0, {self.prompt_len}], got {self.post_vision_len}")
        if self.stats_window < 0:
            raise ValidationError(f"stats_window: must be >= 0, got {self.stats_window}")

    @property
    def seq_len(self) -> int:
        return self.prompt_len + self.n_output_tokens

    def gen_spec(self) -> GenSpec:
        return GenSpec(num_layers=self.num_layers, num_query_heads=self.num_query_heads,
                       num_kv_heads=self.num_kv_heads, head_dim=self.head_dim, prompt_len=self.prompt_len,
                       post_vision_len=self.post_vision_len, decode_len=self.n_output_tokens, seed=self.seed)


@dataclass(frozen=True)
class BenchReport:
    """reference bench.py:106-165."""

    prompt_len: int
    batch_size: int
    n_output_tokens: int
    alpha: float
    policy: str
    budget: str
    backend: str
    threads: int
    kept_counts: list
    prefill_time_s: float
    stats_overhead_time_s: float
    decode_time_full_s: float
    decode_time_compressed_s: float
    decode_times_full_s: list
    decode_times_compressed_s: list
    kv_bytes_full: int
    kv_bytes_compressed: int

    @property
    def prefill_speedup(self) -> float:
        return self.prefill_time_s / (self.prefill_time_s + self.stats_overhead_time_s)

    @property
    def decode_speedup(self) -> float:
        return self.decode_time_full_s / self.decode_time_compressed_s

    @property
    def end_to_end_speedup(self) -> float:
        full = self.prefill_time_s + self.decode_time_full_s
        return full / (self.prefill_time_s + self.stats_overhead_time_s + self.decode_time_compressed_s)

    def to_dict(self) -> dict:
        out = {k: getattr(self, k) for k in (
            "prompt_len", "batch_size", "n_output_tokens", "alpha", "policy", "budget", "backend", "threads",
            "kept_counts", "prefill_time_s", "stats_overhead_time_s", "decode_time_full_s",
            "decode_time_compressed_s", "decode_times_full_s", "decode_times_compressed_s", "kv_bytes_full",
            "kv_bytes_compressed")}
        out.update(prefill_speedup=self.prefill_speedup, decode_speedup=self.decode_speedup,
                   end_to_end_speedup=self.end_to_end_speedup)
        return out


def estimate_bytes(spec: BenchSpec) -> int:
    """Closed-form working-set bound (reference bench.py:168-176)."""
    t, d = spec.seq_len, spec.head_dim
    trace_bytes = spec.num_layers * (spec.num_query_heads + spec.num_kv_heads) * t * d * 4
    values_bytes = spec.num_layers * spec.num_kv_heads * t * d * 4
    cache_bytes = spec.batch_size * spec.num_layers * spec.num_kv_heads * 2 * t * d * 4 * 2
    return trace_bytes + values_bytes + cache_bytes


def _check_size(spec: BenchSpec) -> None:
    need = estimate_bytes(spec)
    if need > spec.max_bytes:
        raise SpecTooLargeError(f"spec needs about {need} bytes of working set, cap is {spec.max_bytes}")


def kv_cache_bytes(tokens_per_layer: list, spec: BenchSpec) -> int:
    """2 (K and V) * tokens * d * 4 bytes over layers and KV heads (reference bench.py:326-328)."""
    return sum(2 * t * spec.head_dim * 4 * spec.num_kv_heads for t in tokens_per_layer)


# ---------------------------------------------------------------- device pieces
class _Resident:
    """The trace and values of one spec as padded bf16 device tensors."""

    def __init__(self, trace: AttentionTrace, values: list, spec: BenchSpec):
        torch = _lib.require_cuda()
        h = trace.header
        self.d = h.head_dim
        self.dp = 64 if self.d <= 64 else 128
        if self.d > 128:
            raise ValidationError(f"head_dim: {self.d} > 128 is not supported")

        def stack(arrs):
            t = torch.from_numpy(np.ascontiguousarray(np.stack(arrs)[None])).to("cuda", torch.bfloat16)
            if self.dp != self.d:
                t = torch.nn.functional.pad(t, (0, self.dp - self.d))
            return t.contiguous()

        self.engines = {}                  # (start, end) -> (window engine, its query rows)
        self.q = stack(trace.queries)      # [1, L, Hq, T, dp]
        self.k = stack(trace.keys)         # [1, L, Hkv, T, dp]
        self.v = stack(values)


def _timed(fn):
    torch = _lib.require_cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def _window_engine(res: _Resident, spec: BenchSpec, start: int, end: int):
    """K1 + K2 over query rows [start, end) of every layer and head, from the
    resident tensors: column mass, below counts, gamma and gamma'."""
    from .engine import Shape, VLCache

    key = (start, end)
    if key not in res.engines:   # workspaces allocated once per window, as a server would
        shape = Shape(1, spec.num_layers, spec.num_query_heads, spec.num_kv_heads, res.dp, end, end - start)
        eng = VLCache(shape, alpha=spec.alpha, p=spec.p, recent_frac=spec.recent_window_frac, keep_scores=True,
                      scale=1.0 / math.sqrt(res.d))
        res.engines[key] = (eng, res.q[:, :, :, start:end].contiguous())
    eng, q_win = res.engines[key]
    eng.score_stats(q_win, res.k)
    eng.allocate()
    return eng


def _compression_pass(res: _Resident, spec: BenchSpec):
    """Statistics window + budget + eviction on the device, timed (reference
    bench.py:245-323): (allocation, kept [L][Hkv] index arrays, seconds)."""
    from .scoring import _select_device, _select_scores

    m = spec.prompt_len
    gamma_window = min(spec.post_vision_len, spec.stats_window)
    if gamma_window == 0:
        gamma_window = min(m, spec.stats_window) if spec.stats_window else 0
    need_gamma = spec.budget == "sparsity_aware"
    if need_gamma and gamma_window == 0:
        raise ValidationError("stats_window: sparsity-aware budget needs a non-empty window")
    score_window = None
    if spec.policy == "vlcache":
        if gamma_window == 0:
            raise ValidationError("post_vision_len: vlcache policy needs a stats window")
        score_window = (m - gamma_window, m)
    elif spec.policy == "sliding":
        w = min(spec.stats_window, m)
        if w == 0:
            raise ValidationError("stats_window: sliding policy needs a positive window")
        score_window = (m - w, m)
    elif spec.policy == "h2o":
        score_window = (0, m)
    L, Hkv = spec.num_layers, spec.num_kv_heads

    def work():
        eng_s = _window_engine(res, spec, *score_window) if score_window else None
        if need_gamma:
            eng_g = eng_s if spec.policy == "vlcache" else _window_engine(res, spec, m - gamma_window, m)
            allocation = allocate_sparsity_aware(eng_g.gamma_mean.cpu().numpy(), spec.alpha, m)
        else:
            allocation = allocate_uniform(spec.alpha, L, m)
        counts = np.asarray(allocation.kept_counts, dtype=np.int64)
        if spec.policy == "streaming":   # positional scores, then the same eviction
            kept = []
            for layer in range(L):
                c = int(counts[layer])
                n_init = -(-c // 10)
                sc = np.zeros(m, dtype=np.float64)
                sc[m - min(c - n_init, m):] = 1.0
                sc[:min(n_init, m)] = 2.0
                idx = _select_scores(sc, c, spec.recent_window_frac)
                kept.append([idx.copy() for _ in range(Hkv)])
        else:
            koff, idx = _select_device(eng_s, counts)
            kept = [[idx[koff[l * Hkv + kv]:koff[l * Hkv + kv + 1]] for kv in range(Hkv)] for l in range(L)]
        return allocation, kept

    (allocation, kept), secs = _timed(work)
    return allocation, kept, secs


def _decode_engine(res: _Resident, spec: BenchSpec, kept):
    """An engine over batch_size copies of the sequence with the given kept sets
    (None: the full prompt cache) gathered into its ragged cache (K4)."""
    torch = _lib.require_cuda()
    from .engine import Shape, VLCache

    B, L, Hkv = spec.batch_size, spec.num_layers, spec.num_kv_heads
    m, n = spec.prompt_len, spec.n_output_tokens - 1
    shape = Shape(B, L, spec.num_query_heads, Hkv, res.dp, m, max(1, min(spec.post_vision_len, m)))
    eng = VLCache(shape, alpha=1.0, decode_steps=max(n, 1), scale=1.0 / math.sqrt(res.d))
    if kept is None:
        kept = [[np.arange(m)] * Hkv for _ in range(L)]
    counts = np.array([len(kept[l][0]) for l in range(L)] * B, dtype=np.int64)
    per_slot = np.repeat(counts, Hkv)
    koff = np.concatenate([[0], np.cumsum(per_slot)])
    coff = np.concatenate([[0], np.cumsum(per_slot + eng.decode_steps)])
    idx = np.concatenate([np.asarray(kept[l][kv]) for _ in range(B) for l in range(L) for kv in range(Hkv)])
    slot = np.repeat(np.arange(B * L * Hkv), per_slot)
    eng.kept_counts.copy_(torch.from_numpy(counts))
    eng.kept_off.copy_(torch.from_numpy(koff))
    eng.cache_off.copy_(torch.from_numpy(coff))
    eng.kept_idx[: idx.size].copy_(torch.from_numpy(idx.astype(np.int32)))
    eng.kept_slot[: idx.size].copy_(torch.from_numpy(slot.astype(np.int32)))
    k = res.k.expand(B, -1, -1, -1, -1).contiguous()
    v = res.v.expand(B, -1, -1, -1, -1).contiguous()
    q = res.q[:, :, :, m:m + max(n, 1)].expand(B, -1, -1, -1, -1).contiguous()
    eng.gather(k, v)
    return eng, q, k, v


def _time_decode(res: _Resident, spec: BenchSpec, kept):
    """(median seconds, raw seconds) of the batch decode: n_output_tokens - 1
    steps of every layer and KV head, repeats after warmup (reference bench.py:375-394)."""
    eng, q, k, v = _decode_engine(res, spec, kept)
    n = spec.n_output_tokens - 1
    if n == 0:
        return 0.0, [0.0] * spec.repeats
    for _ in range(spec.warmup):
        eng.decode(q, k, v, n_steps=n, graph=True)
    times = [_timed(lambda: eng.decode(q, k, v, n_steps=n, graph=True))[1] for _ in range(spec.repeats)]
    return statistics.median(times), times


def _time_prefill(res: _Resident, spec: BenchSpec) -> float:
    """The causal prefill of every layer, once per batch sequence (reference bench.py:235-242)."""
    from .prefill import prefill

    m = spec.prompt_len
    scale = 1.0 / math.sqrt(res.d)
    prefill(res.q, res.k, res.v, m, scale=scale, stats=False)    # warm the library and shapes
    return _timed(lambda: [prefill(res.q, res.k, res.v, m, scale=scale, stats=False)
                           for _ in range(spec.batch_size)])[1]


def _setup(spec: BenchSpec):
    _check_size(spec)
    trace, _ = generate_trace(spec.gen_spec())
    # the B200 path computes in bf16: round once, so every stage sees the same values
    trace = AttentionTrace(header=trace.header, layout=trace.layout,
                           queries=[round_to_bf16(x) for x in trace.queries],
                           keys=[round_to_bf16(x) for x in trace.keys])
    values = [round_to_bf16(x) for x in synthesize_values(spec.gen_spec())]
    return trace, values, _Resident(trace, values, spec)


def run_bench(spec: BenchSpec) -> BenchReport:
    """Prefill, compression pass, and decode against the full and the compressed
    cache (reference bench.py:397-429)."""
    trace, values, res = _setup(spec)
    prefill_s = _time_prefill(res, spec)
    _compression_pass(res, spec)                                 # warm-up
    allocation, kept, stats_s = _compression_pass(res, spec)
    full_median, full_times = _time_decode(res, spec, None)
    comp_median, comp_times = _time_decode(res, spec, kept)
    m = trace.header.prompt_len
    kept_counts = [int(c) for c in allocation.kept_counts]
    return BenchReport(prompt_len=spec.prompt_len, batch_size=spec.batch_size, n_output_tokens=spec.n_output_tokens,
                       alpha=spec.alpha, policy=spec.policy, budget=spec.budget, backend=BACKEND,
                       threads=spec.threads, kept_counts=kept_counts, prefill_time_s=prefill_s,
                       stats_overhead_time_s=stats_s, decode_time_full_s=full_median,
                       decode_time_compressed_s=comp_median, decode_times_full_s=full_times,
                       decode_times_compressed_s=comp_times,
                       kv_bytes_full=kv_cache_bytes([m] * spec.num_layers, spec),
                       kv_bytes_compressed=kv_cache_bytes(kept_counts, spec))


@dataclass(frozen=True)
class OverheadReport:
    """reference bench.py:431-447."""

    stats_time_s: float
    prefill_time_s: float

    @property
    def fraction(self) -> float:
        return 0.0 if self.stats_time_s == 0.0 else self.stats_time_s / self.prefill_time_s

    def to_dict(self) -> dict:
        return {"stats_time_s": self.stats_time_s, "prefill_time_s": self.prefill_time_s, "fraction": self.fraction}


def stats_overhead(spec: BenchSpec) -> OverheadReport:
    """Cost of the statistics window + eviction pass relative to the prefill (reference bench.py:450-463)."""
    trace, values, res = _setup(spec)
    prefill_s = _time_prefill(res, spec)
    if min(trace.header.post_vision_len, spec.stats_window) == 0:
        return OverheadReport(stats_time_s=0.0, prefill_time_s=prefill_s)
    _compression_pass(res, spec)
    _, _, stats_s = _compression_pass(res, spec)
    return OverheadReport(stats_time_s=stats_s, prefill_time_s=prefill_s)


CURVE_FIELDS = ("batch", "mode", "latency_s", "throughput_tok_s")


def latency_throughput_curve(specs: list) -> list:
    """(batch, mode, latency_s, throughput_tok_s) rows per spec (reference bench.py:466-502)."""
    if not specs:
        raise ValidationError("specs: need at least one BenchSpec")
    if len({s.prompt_len for s in specs}) != 1:
        raise ValidationError("specs: all BenchSpecs must share prompt_len")
    rows = []
    for spec in specs:
        r = run_bench(spec)
        tokens = spec.batch_size * spec.n_output_tokens
        full = r.prefill_time_s + r.decode_time_full_s
        comp = r.prefill_time_s + r.stats_overhead_time_s + r.decode_time_compressed_s
        rows.append({"batch": spec.batch_size, "mode": "full", "latency_s": full, "throughput_tok_s": tokens / full})
        rows.append({"batch": spec.batch_size, "mode": "compressed", "latency_s": comp,
                     "throughput_tok_s": tokens / comp})
    return rows
