"""Prefill attention on the B200.

``prefill_attention`` keeps the contract of the reference's
``bench._prefill_layer(queries, keys, values, m, tile)`` (pkg/src/vlcache/bench.py:196-234):
causal softmax attention of the m prompt rows of every query head, float32
[H, m, d].  ``prefill`` is the batched device form over [B, L, H, T, d] bf16
tensors; it also returns the exact per-row softmax statistics (row max in
logit units, row sum), which the compression path's window statistics reuse.
Runs in ``vlc_prefill`` (csrc/prefill.cu, tcgen05 + TMEM); no CPU fallback.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from ._device import to_device_bf16
from .errors import ValidationError


def prefill(q, keys, values, m: int, scale: float | None = None, stats: bool = True):
    """Causal prefill over device bf16 tensors q [B, L, Hq, Tq, d], keys / values
    [B, L, Hkv, T, d] (Tq, T >= m; d in {64, 128}).  Returns (out f32 [B, L, Hq, m, d],
    row_max f32 [B, L, Hq, m] or None, row_sum f32 [B, L, Hq, m] or None)."""
    torch = _lib.require_cuda()
    B, L, Hq, Tq, d = q.shape
    Hkv, T = keys.shape[2], keys.shape[3]
    if keys.shape != values.shape or keys.shape[:2] != (B, L) or keys.shape[4] != d:
        raise ValidationError(f"keys / values: shapes {tuple(keys.shape)} / {tuple(values.shape)} do not match q")
    if not (1 <= m <= min(Tq, T)):
        raise ValidationError(f"m: must be in [1, {min(Tq, T)}], got {m}")
    for name, t in (("q", q), ("keys", keys), ("values", values)):
        if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
            raise ValidationError(f"{name}: expected a contiguous bf16 CUDA tensor")
    lib = _lib.load()
    ws_bytes = int(lib.vlc_prefill_ws_bytes(B * L * Hkv, d, m))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    out = torch.empty((B, L, Hq, m, d), dtype=torch.float32, device=q.device)
    rmax = torch.empty((B, L, Hq, m), dtype=torch.float32, device=q.device) if stats else None
    rsum = torch.empty_like(rmax) if stats else None
    sc = 1.0 / math.sqrt(d) if scale is None else float(scale)
    _lib.call("vlc_prefill", q.data_ptr(), Tq, keys.data_ptr(), values.data_ptr(), T, B, L, Hq, Hkv, d, int(m), sc,
              ws.data_ptr(), ws_bytes, out.data_ptr(), 0 if rmax is None else rmax.data_ptr(),
              0 if rsum is None else rsum.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return out, rmax, rsum


def prefill_attention(queries: np.ndarray, keys: np.ndarray, values: np.ndarray, m: int,
                      tile: int = 128) -> np.ndarray:
    """Causal attention outputs for the prompt rows of one layer, float32 [H, m, d]
    (reference bench.py:196-234).  ``tile`` is the reference's CPU blocking knob
    (validated, not used: the device tiles are 128 x 128).  Inputs are rounded to
    bf16 on upload; head dims below 64 / 128 are zero-padded (scale of the true d)."""
    if tile < 1:
        raise ValidationError(f"tile: must be >= 1, got {tile}")
    queries = np.asarray(queries, dtype=np.float32)
    keys = np.asarray(keys, dtype=np.float32)
    values = np.asarray(values, dtype=np.float32)
    H, _, d = queries.shape
    if keys.shape[0] < 1 or H % keys.shape[0]:
        raise ValidationError(f"keys: {keys.shape[0]} KV heads do not divide {H} query heads")
    if d > 128:
        raise ValidationError(f"head_dim: {d} > 128 is not supported")
    dp = 64 if d <= 64 else 128

    def up(a):
        t = to_device_bf16(a[:, :m])
        if dp != d:
            t = _lib.require_cuda().nn.functional.pad(t, (0, dp - d)).contiguous()
        return t[None, None]

    out, _, _ = prefill(up(queries), up(keys), up(values), m, scale=1.0 / math.sqrt(d), stats=False)
    return out[0, 0, :, :, :d].cpu().numpy()
