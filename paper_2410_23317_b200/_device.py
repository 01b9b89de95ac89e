"""Host <-> device marshalling shared by the reference-shaped API modules.

The reference API takes float32 numpy traces (reference trace.py:153-191).
The B200 path computes on bfloat16 operands with fp32 accumulation, so traces
are rounded to bf16 on upload; results equal the reference's on
bf16-representable inputs ("bf16-in") within the tolerances
pinned in tests/.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def to_device_bf16(a: np.ndarray):
    torch = _lib.require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    return t.to(device="cuda", dtype=torch.bfloat16, non_blocking=False).contiguous()


def window_tensors(trace, start: int, end: int, layers=None, kv_heads=None):
    """q_win [1, L, Hq', w, d] and keys [1, L, Hkv', end, d] bf16 on the device for
    query rows [start, end) and keys [0, end) (reference attention.py:119-120).
    kv_heads restricts to a contiguous KV-head range (lo, hi) and its query heads."""
    h = trace.header
    ls = range(h.num_layers) if layers is None else layers
    g = h.group_size
    lo, hi = (0, h.num_kv_heads) if kv_heads is None else kv_heads
    q = np.stack([trace.queries[l][lo * g:hi * g, start:end] for l in ls])[None]
    k = np.stack([trace.keys[l][lo:hi, :end] for l in ls])[None]
    return to_device_bf16(q), to_device_bf16(k)


def causal_per_column(n: int, q_base: int, w: int) -> np.ndarray:
    """causal[j] = #window rows r with j <= q_base + r (reference _core.pyx:205)."""
    j = np.arange(n, dtype=np.int64)
    last = q_base + w - 1
    return np.clip(np.minimum(w, last - j + 1), 0, None).astype(np.int64)
