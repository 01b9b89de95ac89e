"""Drop-in for the reference's kernel seam ``vlcache._kernels``.

reference pkg/src/vlcache/_kernels/__init__.py:10-27 exports BACKEND,
stats_tiled and decode_step with numpy-in/numpy-out semantics over float32
arrays.  Here both run on the B200 through the C-ABI with the reference's
float32 contract (vlc_stats_f32 / vlc_decode_f32, csrc/seam_f32.cu: float64
dots, float32 logits and exps, float64 sums, the reference's per-row and
per-column order), so they can stand in the compiled-extension slot of the
reference package and its own tests run unmodified over them
(tests/test_reference_suite.py).  There is no CPU
fallback -- without the extension or a GPU every call raises KernelError.
One (layer, head) per call makes this seam launch-bound by design; the
batched bf16 path is engine.VLCache.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from ._device import causal_per_column, to_device_bf16
from .errors import ExactnessError, ValidationError

EXACT_BAND_LOGIT = 1.0 / 512.0 / 1.4426950408889634   # include/vlc.h VLC_EXACT_BAND_LOGIT
EXACT_ROWMAX_ERR = EXACT_BAND_LOGIT / 16.0             # include/vlc.h VLC_EXACT_ROWMAX_ERR

BACKEND = "b200"


def _padded(a: np.ndarray, width: int) -> np.ndarray:
    if a.shape[1] == width:
        return a
    out = np.zeros((a.shape[0], width), dtype=np.float32)
    out[:, : a.shape[1]] = a
    return out


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def stats_tiled(q, keys, q_base, p, tile):
    """Contract of reference _core.stats_tiled (_core.pyx:210-242):
    (row_max f32[w], row_sum f64[w], col_score f64[n], below i64[n], causal i64[n])."""
    torch = _lib.require_cuda()
    q = np.asarray(q, dtype=np.float32)
    keys = np.asarray(keys, dtype=np.float32)
    if q.ndim != 2 or keys.ndim != 2 or q.shape[1] != keys.shape[1]:
        raise ValueError("stats_tiled: q [w, d] and keys [n, d] float32 with equal d")
    w, d = q.shape
    n = keys.shape[0]
    if tile < 1:
        raise ValidationError(f"tile: must be >= 1, got {tile}")
    if n < q_base + w:
        raise ValidationError(f"keys: need n >= q_base + w ({q_base + w}), got {n}")
    qd, kd = _dev(torch, q), _dev(torch, keys)
    row_max = torch.empty(w, dtype=torch.float32, device="cuda")
    row_sum = torch.empty(w, dtype=torch.float64, device="cuda")
    col = torch.empty(n, dtype=torch.float64, device="cuda")
    below = torch.empty(n, dtype=torch.int64, device="cuda")
    causal = torch.empty(n, dtype=torch.int64, device="cuda")
    _lib.call("vlc_stats_f32", qd.data_ptr(), kd.data_ptr(), w, n, d, int(q_base), float(p), int(tile),
              row_max.data_ptr(), row_sum.data_ptr(), col.data_ptr(), below.data_ptr(), causal.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    return (row_max.cpu().numpy(), row_sum.cpu().numpy(), col.cpu().numpy(), below.cpu().numpy(),
            causal.cpu().numpy())


def stats_tiled_tc(q, keys, q_base, p, tile=128):
    """K1 -- the batched hot path's tcgen05 kernel with exact mode -- on one
    slot, with stats_tiled's contract: inputs are rounded to bf16 on upload
    (the tensor cores' operand type, the "bf16-in" protocol of SURVEY.md
    section 8).  The parity tests use this to pin K1 against the oracle one
    (layer, head) at a time."""
    torch = _lib.require_cuda()
    q = np.asarray(q, dtype=np.float32)
    keys = np.asarray(keys, dtype=np.float32)
    w, d = q.shape
    n = keys.shape[0]
    if tile < 1:
        raise ValidationError(f"tile: must be >= 1, got {tile}")
    if n < q_base + w:
        raise ValidationError(f"keys: need n >= q_base + w ({q_base + w}), got {n}")
    if d > 128:
        raise ValidationError(f"head_dim: {d} > 128 is not supported")
    dp = 64 if d <= 64 else 128   # K1 tiles are 64/128 wide; zero columns add nothing
    qd = to_device_bf16(_padded(q, dp))
    kd = to_device_bf16(_padded(keys, dp))
    nrb = int(_lib.load().vlc_score_partials(w))
    f32 = dict(dtype=torch.float32, device="cuda")
    row_max = torch.empty(w, **f32)
    row_sum = torch.empty(w, **f32)
    col = torch.empty(nrb * n, **f32)
    below_head = torch.zeros(1, dtype=torch.int64, device="cuda")
    below_col = torch.zeros(n, dtype=torch.int32, device="cuda")
    # p == 1 is accepted by the reference kernel (test_kernels.py:271-277):
    # "below 1.0" equals "below the largest double under 1.0" for float exps
    p_eff = min(float(p), math.nextafter(1.0, 0.0))
    # exact mode: counts and row max decided like the reference's float64 dots.
    # The re-decision list starts at O(w + 64K) entries (not O(w * n)); on the
    # rare overflow the call is repeated with room for every listed entry.
    cap = max(1 << 16, 8 * w)
    while True:
        ws_bytes = int(_lib.load().vlc_score_exact_bytes(1, 1, w, cap))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
        below_head.zero_()
        below_col.zero_()
        _lib.call("vlc_score_stats", qd.data_ptr(), kd.data_ptr(), 1, 1, dp, n, n, w, int(q_base), p_eff,
                  1.0 / math.sqrt(d), row_max.data_ptr(), row_sum.data_ptr(), col.data_ptr(),
                  below_head.data_ptr(), below_col.data_ptr(), ws.data_ptr(), ws_bytes,
                  torch.cuda.current_stream().cuda_stream)
        status = ws[:32].cpu()
        counters = status.view(torch.int32).tolist()   # [deferred, listed, overflow, ...] (include/vlc.h)
        if counters[2] == 0:
            errs = status.view(torch.float32).tolist()
            if errs[5] + errs[6] > EXACT_BAND_LOGIT / 8 or errs[6] > EXACT_ROWMAX_ERR / 2:
                raise ExactnessError(f"exact mode: observed tensor-core logit error {errs[5]:.3g} / row-max "
                                     f"error {errs[6]:.3g} approach the exact-mode margins")
            break
        cap = max(2 * cap, counters[1] + 1024)
        del ws
    col_score = col.view(nrb, n).double().sum(0)
    return (row_max.cpu().numpy(), row_sum.double().cpu().numpy(), col_score.cpu().numpy(),
            below_col.long().cpu().numpy(), causal_per_column(n, int(q_base), w))


def decode_step(q, keys, values):
    """Contract of reference _core.decode_step (_core.pyx:245-278): one decode
    attention pass, q [G, d] against keys/values [n, d] -> f32 [G, d]."""
    torch = _lib.require_cuda()
    q = np.asarray(q, dtype=np.float32)
    keys = np.asarray(keys, dtype=np.float32)
    values = np.asarray(values, dtype=np.float32)
    g, d = q.shape
    n = keys.shape[0]
    if n < 1:
        raise ValidationError("keys: need at least one row")
    if keys.shape != values.shape or keys.shape[1] != d:
        raise ValueError("decode_step: keys / values [n, d] float32 matching q [G, d]")
    qd, kd, vd = _dev(torch, q), _dev(torch, keys), _dev(torch, values)
    scratch = torch.empty(g * n, dtype=torch.float32, device="cuda")
    denom = torch.empty(g, dtype=torch.float64, device="cuda")
    out = torch.empty((g, d), dtype=torch.float32, device="cuda")
    _lib.call("vlc_decode_f32", qd.data_ptr(), g, kd.data_ptr(), vd.data_ptr(), n, d, scratch.data_ptr(),
              denom.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return out.cpu().numpy()


__all__ = ["BACKEND", "stats_tiled", "decode_step", "stats_tiled_tc"]
