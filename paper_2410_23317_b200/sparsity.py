"""Per-layer attention sparsity (reference pkg/src/vlcache/sparsity.py:21-103).

``window_sparsity`` measures every (layer, head) of a trace in ONE batched
K1 launch plus K2 (gamma = below / causal, gamma' = numpy-order head mean),
instead of the reference's L x Hq calls to stats_tiled.  Threshold filtering
and curve similarity are analysis helpers outside the hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._device import window_tensors
from .errors import ValidationError
from .trace import AttentionTrace

DEFAULT_P = 0.01
DEFAULT_TILE = 128


@dataclass(frozen=True)
class SparsityConfig:
    p: float = DEFAULT_P
    tile: int = DEFAULT_TILE

    def __post_init__(self) -> None:
        if not 0.0 < self.p < 1.0:
            raise ValidationError(f"p: must be in (0, 1), got {self.p}")
        if self.tile < 1:
            raise ValidationError(f"tile: must be >= 1, got {self.tile}")


@dataclass(frozen=True)
class LayerSparsity:
    """gamma[l, h] for one phase (reference sparsity.py:33-43).

    ``gamma_mean`` is K2's device-computed head mean (numpy pairwise order,
    bit-identical to ``gamma.mean(axis=1)``)."""

    phase: str
    p: float
    gamma: np.ndarray
    gamma_mean: np.ndarray | None = field(default=None, repr=False, compare=False)

    def layer_means(self) -> np.ndarray:
        if self.gamma_mean is not None:
            return self.gamma_mean.copy()
        return self.gamma.mean(axis=1)


def padded_head_dim(d: int) -> int:
    """K1 runs 64- or 128-wide tiles; smaller head dims are zero-padded (the
    softmax scale of the true d is passed explicitly)."""
    if d > 128:
        raise ValidationError(f"head_dim: {d} > 128 is not supported")
    return 64 if d <= 64 else 128


def run_window(trace: AttentionTrace, start: int, end: int, p: float, keep_scores: bool = False):
    """K1 + K2 over query rows [start, end) of every (layer, head): returns the
    engine holding row stats, column mass, counts, gamma and gamma'."""
    from .engine import Shape, VLCache

    h = trace.header
    if not 0 <= start < end <= h.seq_len:
        raise ValidationError(f"window: need 0 <= start < end <= {h.seq_len}, got [{start}, {end})")
    d = h.head_dim
    dp = padded_head_dim(d)
    q, k = window_tensors(trace, start, end)
    if dp != d:
        torch = _lib.require_cuda()
        q = torch.nn.functional.pad(q, (0, dp - d)).contiguous()
        k = torch.nn.functional.pad(k, (0, dp - d)).contiguous()
    shape = Shape(B=1, L=h.num_layers, Hq=h.num_query_heads, Hkv=h.num_kv_heads, d=dp, m=end,
                  w=end - start)
    eng = VLCache(shape, p=p, keep_scores=keep_scores, scale=1.0 / math.sqrt(d))
    eng.score_stats(q, k)
    eng.allocate()
    return eng


def window_sparsity(trace: AttentionTrace, config: SparsityConfig, start: int, end: int,
                    phase: str = "window") -> LayerSparsity:
    """Sparsity over query rows [start, end) for every (layer, head) (reference sparsity.py:69-80)."""
    QueryWindowCheck(start, end)
    h = trace.header
    eng = run_window(trace, start, end, config.p)
    gamma = eng.gamma.view(h.num_layers, h.num_query_heads).cpu().numpy()
    gm = eng.gamma_mean.cpu().numpy()
    return LayerSparsity(phase=phase, p=config.p, gamma=gamma, gamma_mean=gm)


def QueryWindowCheck(start: int, end: int) -> None:
    if not (0 <= start < end):
        raise ValidationError(f"window: need 0 <= start < end, got [{start}, {end})")


def prefill_sparsity(trace: AttentionTrace, config: SparsityConfig = SparsityConfig()) -> LayerSparsity:
    """Sparsity over all m prompt rows (reference sparsity.py:83-85)."""
    return window_sparsity(trace, config, 0, trace.header.prompt_len, phase="prefill")


def post_vision_sparsity(trace: AttentionTrace, config: SparsityConfig = SparsityConfig()) -> LayerSparsity:
    """Sparsity over the last tau prompt rows; requires tau >= 1 (reference sparsity.py:88-95)."""
    h = trace.header
    if h.post_vision_len < 1:
        raise ValidationError("post_vision_len: trace has no post-vision rows")
    return window_sparsity(trace, config, h.prompt_len - h.post_vision_len, h.prompt_len,
                           phase="post_vision")


def decoding_sparsity(trace: AttentionTrace, config: SparsityConfig = SparsityConfig()) -> LayerSparsity:
    """Sparsity over the n_dec decoding rows (reference sparsity.py:98-103)."""
    h = trace.header
    if h.decode_len < 1:
        raise ValidationError("decode_len: trace has no decoding rows")
    return window_sparsity(trace, config, h.prompt_len, h.seq_len, phase="decoding")


# ---------------------------------------------------------------- host analysis helpers
# Small numpy utilities of the reference's analysis surface, kept on the host:
# they act on per-layer curves (L values) or on caller-held arrays.

def threshold_filter(a, p: float) -> np.ndarray:
    """Copy of `a` (one row or rows) with entries below p * row max set to 0
    (reference sparsity.py:46-66; the same filter K5-side contribution uses)."""
    if not 0.0 < p < 1.0:
        raise ValidationError(f"p: must be in (0, 1), got {p}")
    x = np.asarray(a)
    if x.size == 0:
        raise ValidationError("input: must be non-empty")
    if not np.isfinite(x).all():
        raise ValidationError("input: must be finite")
    if (x < 0).any():
        raise ValidationError("input: must be non-negative")
    if x.ndim > 2:
        raise ValidationError(f"input: must be 1-D or 2-D, got {x.ndim}-D")
    m2 = np.atleast_2d(x)
    kept = np.where(m2 < p * m2.max(axis=1, keepdims=True), 0.0, m2)
    return kept if x.ndim == 2 else kept[0]


def curve_similarity(a: LayerSparsity, b: LayerSparsity) -> float:
    """Pearson correlation of two per-layer head-mean sparsity curves
    (reference sparsity.py:106-124); ZeroVarianceError for a flat curve."""
    from .errors import ZeroVarianceError

    x, y = a.layer_means(), b.layer_means()
    if x.shape != y.shape:
        raise ValidationError(f"curves: layer counts differ ({x.size} vs {y.size})")
    if x.size < 2:
        raise ValidationError("curves: need at least 2 layers")
    dx, dy = x - x.mean(), y - y.mean()
    sxx, syy = float(dx @ dx), float(dy @ dy)
    if sxx == 0.0 or syy == 0.0:
        raise ZeroVarianceError("curve variance is zero; correlation undefined")
    return float(dx @ dy) / np.sqrt(sxx * syy)
