"""Batched device API: compress a prefill KV cache, then decode over it.

This is the B200 hot path behind the reference-shaped API (attention.py,
sparsity.py, budget.py, scoring.py of this package): one C-ABI call per stage
for every (batch, layer, KV head) slot at once, all enqueued on the current
torch stream, no host synchronisation between stages.

  K1 score_stats  post-vision Q.K^T statistics        reference _core.pyx:110-242
  K2 allocate     gamma -> gamma' -> beta -> k_l       budget.py:86-111, sparsity.py:79
  K3 select       recent reserve + top-k per slot      scoring.py:185-235
  K4 gather       kept K/V rows -> ragged cache        bench.py:331-353
  K5 decode_step  append + attend over ragged cache    bench.py:356-372, _core.pyx:245-278

Tensors (bf16, CUDA, contiguous):
  q_win  [B, L, Hq, w, d]   the w scoring rows (the last w prompt rows)
  keys   [B, L, Hkv, T, d]  T >= m; rows m.. are the decode steps' new keys
  values [B, L, Hkv, T, d]
  q_dec  [B, L, Hq, n, d]   decode-step queries
"""

from __future__ import annotations

import math
from collections import OrderedDict
from dataclasses import dataclass

from . import _lib
from ._kernels import EXACT_BAND_LOGIT, EXACT_ROWMAX_ERR
from .errors import DegenerateSparsityError, ExactnessError, ValidationError

_ROW_BLOCK = 128  # K1 rows per CTA; col_partial has 2 partials (64-row halves) per block
_MAX_GRAPHS = 16  # captured decode graphs kept per engine (least recently used evicted)


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def _stream() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def kept_rows_bound(batch, layers, kv_heads, prompt_len, alpha, beta_min):
    """Upper bound on sum of kept rows: k_l <= beta_l*m + 1 and
    sum_l beta_l <= alpha*L + L*beta_min (clip raises a layer by <= beta_min)."""
    per = min(layers * prompt_len, math.ceil(prompt_len * layers * (alpha + beta_min)) + 2 * layers)
    return batch * kv_heads * per


@dataclass
class Shape:
    B: int
    L: int
    Hq: int
    Hkv: int
    d: int
    m: int          # prompt length (keys visible to the window)
    w: int          # scoring window rows (tau, or min(tau, stats_window))

    def __post_init__(self):
        for k in ("B", "L", "Hq", "Hkv", "d", "m", "w"):
            if getattr(self, k) < 1:
                raise ValidationError(f"{k}: must be >= 1, got {getattr(self, k)}")
        if self.Hq % self.Hkv:
            raise ValidationError("num_kv_heads: must divide num_query_heads")
        if self.w > self.m:
            raise ValidationError(f"window: {self.w} rows exceed prompt_len {self.m}")

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv

    @property
    def slots(self) -> int:
        return self.B * self.L * self.Hkv

    @property
    def nrb(self) -> int:
        """col_partial rows per slot (vlc_score_partials)."""
        return 2 * ((self.G * self.w + _ROW_BLOCK - 1) // _ROW_BLOCK)

    @property
    def causal_per_head(self) -> int:
        q_base = self.m - self.w
        return self.w * (q_base + 1) + self.w * (self.w - 1) // 2


class VLCache:
    """Owns every device buffer of the path for one shape, so repeated calls
    (and CUDA-graph replays) reuse memory.

    compress(q_win, keys, values) enqueues K1..K4; decode_step / decode
    enqueue K5.  Results stay on the device; ``check()`` synchronises and
    raises DegenerateSparsityError like reference budget.py:108-109.
    """

    def __init__(self, shape: Shape, *, alpha=0.1, p=0.01, recent_frac=0.10, beta_min=0.01,
                 beta_max=1.0, decode_steps=0, keep_scores=False, device=None, head_shard=None,
                 scale=None, exact=True, exact_capacity=None):
        torch = _lib.require_cuda()
        if not 0.0 < alpha <= 1.0:
            raise ValidationError(f"alpha: must be in (0, 1], got {alpha}")
        if not 0.0 < p < 1.0:
            raise ValidationError(f"p: must be in (0, 1), got {p}")
        if not 0.0 <= recent_frac <= 1.0:
            raise ValidationError(f"recent_window_frac: must be in [0, 1], got {recent_frac}")
        if not 0.0 < beta_min <= beta_max:
            raise ValidationError("beta_min: need 0 < beta_min <= beta_max")
        self.shape = s = shape
        self.alpha, self.p, self.recent_frac = float(alpha), float(p), float(recent_frac)
        self.beta_min, self.beta_max = float(beta_min), float(beta_max)
        self.decode_steps = int(decode_steps)
        # softmax scale; None -> 1/sqrt(d) (pass the true d's when d is zero-padded)
        self.scale = 0.0 if scale is None else float(scale)
        dev = torch.device(device or "cuda")
        f32, f64, i64, i32 = torch.float32, torch.float64, torch.int64, torch.int32
        R = s.G * s.w
        self.row_max = torch.empty(s.slots * R, dtype=f32, device=dev)
        self.row_sum = torch.empty(s.slots * R, dtype=f32, device=dev)
        self.col_partial = torch.empty(s.slots * s.nrb * s.m, dtype=f32, device=dev)
        self.below_head = torch.zeros(s.B * s.L * s.Hq, dtype=i64, device=dev)
        # KV-head sharding (parallel.py): K2 sees the counts of every head
        self.head_shard = head_shard
        if head_shard is not None and (head_shard.kv_per_rank != s.Hkv or head_shard.group_size != s.G):
            raise ValidationError("head_shard: local shape does not match the shard")
        self.hq_alloc = head_shard.num_query_heads if head_shard is not None else s.Hq
        self.below_alloc = self.below_head
        self.gamma = torch.empty(s.B * s.L * self.hq_alloc, dtype=f64, device=dev)
        self.gamma_mean = torch.empty(s.B * s.L, dtype=f64, device=dev)
        self.beta_pre = torch.empty(s.B * s.L, dtype=f64, device=dev)
        self.beta = torch.empty(s.B * s.L, dtype=f64, device=dev)
        self.kept_counts = torch.empty(s.B * s.L, dtype=i64, device=dev)
        self.kept_off = torch.empty(s.slots + 1, dtype=i64, device=dev)
        self.cache_off = torch.empty(s.slots + 1, dtype=i64, device=dev)
        self.status = torch.zeros(s.B, dtype=i32, device=dev)
        self._alloc_last = False   # the last launch on the path was K2 (see select)
        self.max_rows = kept_rows_bound(s.B, s.L, s.Hkv, s.m, alpha, beta_min)
        self.kept_idx = torch.empty(self.max_rows, dtype=i32, device=dev)
        self.kept_slot = torch.empty(self.max_rows, dtype=i32, device=dev)
        self.scores = torch.empty(s.slots * s.m, dtype=f64, device=dev) if keep_scores else None
        self.key_scratch = (torch.empty(s.slots * s.m, dtype=i64, device=dev)
                            if s.m > 24 * 1024 else None)
        self.cache_rows = self.max_rows + s.slots * self.decode_steps
        # zero-initialised: K5 tiles may cover rows no step has written yet
        self.k_cache = torch.zeros(self.cache_rows * s.d, dtype=torch.bfloat16, device=dev)
        self.v_cache = torch.zeros(self.cache_rows * s.d, dtype=torch.bfloat16, device=dev)
        self.out = torch.empty(s.B * s.L * s.Hq * s.d, dtype=f32, device=dev)
        # K1 exact mode (vlc.h): room for one listed entry per window row and slot
        # by default; an overflow falls back to fp32 decisions and check() raises
        cap = max(1 << 16, s.slots * R) if exact_capacity is None else int(exact_capacity)
        if cap < 1:
            raise ValidationError(f"exact_capacity: must be >= 1, got {cap}")
        self.exact_capacity = cap
        self.exact_ws_bytes = int(_lib.load().vlc_score_exact_bytes(s.slots, s.G, s.w, cap))
        self.exact_ws = torch.empty(self.exact_ws_bytes, dtype=torch.uint8, device=dev) if exact else None
        self._graphs = OrderedDict()

    # ------------------------------------------------------------ stages
    def _check_inputs(self, q_win, keys, values=None):
        s = self.shape
        import torch

        if tuple(q_win.shape) != (s.B, s.L, s.Hq, s.w, s.d):
            raise ValidationError(f"q_win: expected {(s.B, s.L, s.Hq, s.w, s.d)}, got {tuple(q_win.shape)}")
        if keys.dim() != 5 or tuple(keys.shape[:3]) != (s.B, s.L, s.Hkv) or keys.shape[4] != s.d \
                or keys.shape[3] < s.m:
            raise ValidationError(f"keys: expected [B, L, Hkv, T>=m, d], got {tuple(keys.shape)}")
        for name, t in (("q_win", q_win), ("keys", keys), ("values", values)):
            if t is None:
                continue
            if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
                raise ValidationError(f"{name}: must be a contiguous bf16 CUDA tensor")
        if values is not None and tuple(values.shape) != tuple(keys.shape):
            raise ValidationError("values: must match keys")

    def score_stats(self, q_win, keys, below_col=None):
        """K1 over all slots; fills row_max/row_sum/col_partial/below_head."""
        s = self.shape
        self._check_inputs(q_win, keys)
        self._alloc_last = False   # col_partial is being rewritten
        _lib.call("vlc_score_stats", q_win.data_ptr(), keys.data_ptr(), s.slots, s.G, s.d,
                  keys.shape[3], s.m, s.w, s.m - s.w, self.p, self.scale, _ptr(self.row_max), _ptr(self.row_sum),
                  _ptr(self.col_partial), _ptr(self.below_head), _ptr(below_col), _ptr(self.exact_ws),
                  self.exact_ws_bytes, _stream())

    def allocate(self):
        """K2 from the below-threshold counts currently in below_head."""
        s = self.shape
        self._alloc_last = True   # the next select() may rank under this launch
        _lib.call("vlc_allocate", _ptr(self.below_alloc), s.B, s.L, self.hq_alloc, s.Hkv, s.w, s.m, s.m - s.w,
                  s.m, self.alpha, self.beta_min, self.beta_max, self.decode_steps, _ptr(self.gamma),
                  _ptr(self.gamma_mean), _ptr(self.beta_pre), _ptr(self.beta), _ptr(self.kept_counts),
                  _ptr(self.kept_off), _ptr(self.cache_off), _ptr(self.status), _stream())

    def allocate_from_gamma(self, gamma_mean):
        """K2 from a given head-mean sparsity gamma_mean (f64 CUDA [B, L]) instead of
        K1's counts (reference budget.allocate_sparsity_aware on measured
        sparsity, budget.py:86-111).  gamma_mean = 0 with alpha = 1 keeps every
        token: the full-cache decode baseline on the same kernels."""
        s = self.shape
        import torch

        if tuple(gamma_mean.shape) != (s.B, s.L) or gamma_mean.dtype != torch.float64 or not gamma_mean.is_cuda:
            raise ValidationError(f"gamma_mean: expected a float64 CUDA tensor [{s.B}, {s.L}]")
        self.gamma_mean.copy_(gamma_mean.reshape(-1))
        self._alloc_last = True   # the next select() may rank under this launch
        _lib.call("vlc_allocate_from_gamma", _ptr(self.gamma_mean), s.B, s.L, s.Hkv, s.m, self.alpha, self.beta_min,
                  self.beta_max, self.decode_steps, _ptr(self.beta_pre), _ptr(self.beta), _ptr(self.kept_counts),
                  _ptr(self.kept_off), _ptr(self.cache_off), _ptr(self.status), _stream())

    def select(self):
        """K3.  Directly after allocate() (and with col_partial written before it)
        K3 sums the scores while K2 runs (vlc_select_after_allocate)."""
        s = self.shape
        fn = "vlc_select_after_allocate" if self._alloc_last else "vlc_select"
        self._alloc_last = False
        _lib.call(fn, _ptr(self.col_partial), 0, s.slots, s.Hkv, s.L, s.G, s.m, s.w,
                  _ptr(self.kept_counts), _ptr(self.kept_off), self.recent_frac, _ptr(self.kept_idx),
                  _ptr(self.kept_slot), _ptr(self.scores), _ptr(self.key_scratch), _stream())

    def gather(self, keys, values):
        s = self.shape
        self._check_inputs_kv(keys, values)
        _lib.call("vlc_gather", keys.data_ptr(), values.data_ptr(), s.slots, s.d, keys.shape[3],
                  _ptr(self.kept_idx), _ptr(self.kept_slot), _ptr(self.kept_off), _ptr(self.cache_off),
                  self.max_rows, _ptr(self.k_cache), _ptr(self.v_cache), _stream())

    def _check_inputs_kv(self, keys, values):
        """K4 reads only the kept rows, so keys / values may also be pinned host
        tensors: the kernel then pulls just those rows over PCIe (zero-copy)."""
        s = self.shape
        import torch

        for name, t in (("keys", keys), ("values", values)):
            host_ok = (not t.is_cuda) and t.is_pinned()
            if t.dtype != torch.bfloat16 or not (t.is_cuda or host_ok) or not t.is_contiguous():
                raise ValidationError(f"{name}: must be a contiguous bf16 CUDA or pinned host tensor")
            if t.dim() != 5 or tuple(t.shape[:3]) != (s.B, s.L, s.Hkv) or t.shape[4] != s.d:
                raise ValidationError(f"{name}: expected [B, L, Hkv, T, d], got {tuple(t.shape)}")
        if tuple(values.shape) != tuple(keys.shape):
            raise ValidationError(f"values: shape {tuple(values.shape)} must match keys {tuple(keys.shape)}")
        if keys.shape[3] < s.m:
            raise ValidationError(f"keys: T = {keys.shape[3]} < prompt_len {s.m}")

    def score_stats_given(self, q_win, keys, stat_max, stat_sum):
        """K1's column pass only, with the window rows' softmax statistics from the
        prefill (stat_max logit units / stat_sum f32 [B, L, Hq, m]): row f2's fusion."""
        s = self.shape
        self._check_inputs(q_win, keys)
        if tuple(stat_max.shape[-1:]) != (s.m,) or stat_max.numel() != s.B * s.L * s.Hq * s.m:
            raise ValidationError(f"stat_max: expected [B, L, Hq, {s.m}] prefill statistics")
        self._alloc_last = False   # col_partial is being rewritten
        _lib.call("vlc_score_stats_given", q_win.data_ptr(), keys.data_ptr(), s.slots, s.G, s.d,
                  keys.shape[3], s.m, s.w, s.m - s.w, self.p, self.scale, stat_max.data_ptr(), stat_sum.data_ptr(),
                  s.m, _ptr(self.row_max), _ptr(self.row_sum), _ptr(self.col_partial), _ptr(self.below_head), 0,
                  _ptr(self.exact_ws), self.exact_ws_bytes, _stream())

    def prefill_compress(self, q_prompt, keys, values):
        """Row f2 end to end: causal prefill of the m prompt rows (vlc_prefill,
        returns its f32 [B, L, Hq, m, d] output), K1's column pass on the
        prefill's own row statistics for the window rows, then K2 -> K3 -> K4.
        q_prompt: bf16 [B, L, Hq, >= m, d]; keys / values as for compress()."""
        from .prefill import prefill

        s = self.shape
        if self.head_shard is not None:
            raise ValidationError("prefill_compress: head-sharded engines are not supported")
        out, rmax, rsum = prefill(q_prompt, keys, values, s.m, scale=self.scale or None)
        q_win = q_prompt[:, :, :, s.m - s.w:s.m].contiguous()
        self.score_stats_given(q_win, keys, rmax, rsum)
        self.allocate()
        self.select()
        self.gather(keys, values)
        return out

    def compress(self, q_win, keys, values=None, group=None):
        """K1 -> (count exchange across ranks when head-sharded) -> K2 -> K3 -> K4."""
        self.score_stats(q_win, keys)
        if self.head_shard is not None:
            from .parallel import exchange_head_counts

            s = self.shape
            local = self.below_head.view(s.B, s.L, s.Hq)
            self.below_alloc = exchange_head_counts(local, self.head_shard, group).reshape(-1)
        self.allocate()
        self.select()
        if values is not None:
            self.gather(keys, values)
        return self

    # ------------------------------------------------------------ decode
    def decode_step(self, q_dec, keys, values, step, chained=False, row0=None):
        """K5 for decode step `step`: appends row row0+step of keys / values
        (row0 defaults to m: full [B, L, Hkv, T, d] tensors; pass row0=0 for
        decode-row tensors [B, L, Hkv, n, d]) and attends the G query rows
        q_dec[..., step, :] of each KV head.  chained=True promises the previous
        kernel on the stream is step-1 (prefetch under programmatic dependent
        launch)."""
        s = self.shape
        if not 0 <= step < self.decode_steps:
            raise ValidationError(f"step: must be in [0, {self.decode_steps}), got {step}")
        self._check_decode_inputs(q_dec, keys, values)
        n_dec, T = q_dec.shape[3], keys.shape[3]
        r0 = s.m if row0 is None else int(row0)
        if step >= n_dec or r0 + step >= T:
            raise ValidationError("step: beyond the provided decode rows")
        esz = 2
        _lib.call("vlc_decode_step", q_dec.data_ptr() + step * s.d * esz, n_dec * s.d,
                  keys.data_ptr() + (r0 + step) * s.d * esz, values.data_ptr() + (r0 + step) * s.d * esz,
                  T * s.d, _ptr(self.k_cache), _ptr(self.v_cache), self.cache_rows, _ptr(self.cache_off),
                  _ptr(self.kept_counts), step, s.B, s.L, s.Hkv, s.G, s.d, self.scale, int(bool(chained)),
                  _ptr(self.out), _stream())
        return self.out

    def _check_decode_inputs(self, q_dec, keys, values):
        """K5 does raw pointer arithmetic with these shapes: bf16, CUDA,
        contiguous, q_dec [B, L, Hq, n, d], keys == values [B, L, Hkv, T, d]."""
        import torch

        s = self.shape
        for name, t in (("q_dec", q_dec), ("keys", keys), ("values", values)):
            if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous() or t.dim() != 5:
                raise ValidationError(f"{name}: must be a contiguous 5-D bf16 CUDA tensor")
        if tuple(q_dec.shape[:3]) != (s.B, s.L, s.Hq) or q_dec.shape[4] != s.d or q_dec.shape[3] < 1:
            raise ValidationError(f"q_dec: expected [{s.B}, {s.L}, {s.Hq}, n, {s.d}], got {tuple(q_dec.shape)}")
        if tuple(keys.shape[:3]) != (s.B, s.L, s.Hkv) or keys.shape[4] != s.d:
            raise ValidationError(f"keys: expected [{s.B}, {s.L}, {s.Hkv}, T, {s.d}], got {tuple(keys.shape)}")
        if tuple(values.shape) != tuple(keys.shape):
            raise ValidationError(f"values: shape {tuple(values.shape)} must match keys {tuple(keys.shape)}")

    def decode(self, q_dec, keys, values, n_steps=None, graph=True, outputs=None, row0=None, first_step=0):
        """Decode steps first_step .. first_step + n_steps - 1 (default: all of
        them); with graph=True the launch sequence is captured once into a CUDA
        graph (per input pointers and step range) and replayed."""
        import torch

        t0 = int(first_step)
        n = self.decode_steps - t0 if n_steps is None else int(n_steps)
        if not (0 <= t0 and n >= 1 and t0 + n <= self.decode_steps):
            raise ValidationError(f"steps: [{t0}, {t0 + n}) outside [0, {self.decode_steps})")
        if outputs is not None or not graph:
            for t in range(t0, t0 + n):
                self.decode_step(q_dec, keys, values, t, row0=row0)
                if outputs is not None:
                    outputs.append(self.out.clone())
            return self.out
        self._check_decode_inputs(q_dec, keys, values)
        # the captured launches bake in pointers AND strides (n_dec, T): key on both
        key = (q_dec.data_ptr(), tuple(q_dec.shape), keys.data_ptr(), values.data_ptr(), tuple(keys.shape),
               t0, n, row0)
        g = self._graphs.get(key)
        if g is not None:
            self._graphs.move_to_end(key)
        else:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for t in range(t0, t0 + n):   # warm-up launch outside capture
                    self.decode_step(q_dec, keys, values, t, chained=t > t0, row0=row0)
            torch.cuda.current_stream().wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for t in range(t0, t0 + n):
                    self.decode_step(q_dec, keys, values, t, chained=t > t0, row0=row0)
            self._graphs[key] = g
            while len(self._graphs) > _MAX_GRAPHS:
                self._graphs.popitem(last=False)
        g.replay()
        return self.out

    # ------------------------------------------------------------ host entry
    def score_stats_layers(self, q_win, keys, b, l0, l1):
        """K1 over the slots of prompt b, layers [l0, l1) only (their outputs
        land where score_stats would put them): lets the compression start on
        the first layers while later ones are still in flight."""
        s = self.shape
        self._check_inputs(q_win, keys)
        if not (0 <= b < s.B and 0 <= l0 < l1 <= s.L):
            raise ValidationError(f"layers: need 0 <= l0 < l1 <= {s.L} and 0 <= b < {s.B}")
        slot0 = (b * s.L + l0) * s.Hkv
        R, esz = s.G * s.w, 2
        T = keys.shape[3]
        self._alloc_last = False   # col_partial is being rewritten
        _lib.call("vlc_score_stats", q_win.data_ptr() + slot0 * R * s.d * esz, keys.data_ptr() + slot0 * T * s.d * esz,
                  (l1 - l0) * s.Hkv, s.G, s.d, T, s.m, s.w, s.m - s.w, self.p, self.scale,
                  _ptr(self.row_max) + slot0 * R * 4, _ptr(self.row_sum) + slot0 * R * 4,
                  _ptr(self.col_partial) + slot0 * s.nrb * s.m * 4, _ptr(self.below_head) + slot0 * s.G * 8,
                  0, _ptr(self.exact_ws), self.exact_ws_bytes, _stream())

    def run_from_host(self, q_win, k_prompt, v_prompt, q_dec, k_dec, v_dec, chunks=4, dec_chunks=8, dec_early=2,
                      check=True):
        """End-to-end call with pinned HOST inputs (the reference API's setting:
        traces live in host memory): copies Q windows, prompt keys, decode
        queries and the decode steps' K/V rows to the device, compresses --
        K4 pulls only the kept value rows straight from pinned host memory --
        decodes every step, and returns (kept_counts, last decode output) on the
        host.  The copies run on a side stream in `chunks` layer groups per
        prompt and K1 starts on each group as soon as it has landed, so the
        scoring hides under the PCIe transfer.  Shapes: q_win [B,L,Hq,w,d],
        k/v_prompt [B,L,Hkv,m,d], q_dec [B,L,Hq,n,d], k/v_dec [B,L,Hkv,n,d],
        bf16, pinned.  Returns (kept_counts, out, bytes copied host->device);
        the values pulled zero-copy are zero_copy_bytes(kept_counts) once the
        stream has synced.  check=True synchronises at the end and raises like
        check() (degenerate budget, exact-mode overflow); check=False leaves
        the copies in flight for the caller to synchronise."""
        import torch

        s = self.shape
        for name, t in (("q_win", q_win), ("k_prompt", k_prompt), ("v_prompt", v_prompt), ("q_dec", q_dec),
                        ("k_dec", k_dec), ("v_dec", v_dec)):
            if t.is_cuda or not t.is_pinned() or t.dtype != torch.bfloat16 or not t.is_contiguous():
                raise ValidationError(f"{name}: must be a contiguous pinned bf16 host tensor")
        st = getattr(self, "_stage", None)
        if st is None or st[0].shape != q_win.shape or st[1].shape != k_prompt.shape or st[2].shape != q_dec.shape:
            st = (torch.empty_like(q_win, device="cuda"), torch.empty_like(k_prompt, device="cuda"),
                  torch.empty_like(q_dec, device="cuda"), torch.empty_like(k_dec, device="cuda"),
                  torch.empty_like(v_dec, device="cuda"),
                  torch.empty(s.B * s.L, dtype=torch.int64).pin_memory(),
                  torch.empty(self.out.numel(), dtype=torch.float32).pin_memory())
            self._stage = st
            self._copy_stream = torch.cuda.Stream()
            self._graphs.clear()   # graphs captured on the old staging buffers are stale
        d_qw, d_k, d_qd, d_kn, d_vn, h_counts, h_out = st
        comp, cs = torch.cuda.current_stream(), self._copy_stream
        cs.wait_stream(comp)                  # staging buffers free (previous call done with them)
        per = -(-s.L // max(1, int(chunks)))
        groups = []
        with torch.cuda.stream(cs):
            for b in range(s.B):
                for l0 in range(0, s.L, per):
                    l1 = min(s.L, l0 + per)
                    d_qw[b, l0:l1].copy_(q_win[b, l0:l1], non_blocking=True)
                    d_k[b, l0:l1].copy_(k_prompt[b, l0:l1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    groups.append((b, l0, l1, ev))
        # decode inputs in step groups: the first `dec_early` groups cross PCIe
        # right behind the keys (filling the link while K1's last group, K2 and
        # K3 run); the rest are queued behind K4 so they do not compete with its
        # zero-copy value reads, and the decode chases them group by group
        n = q_dec.shape[3]
        per_s = -(-n // max(1, int(dec_chunks)))
        bounds = [(s0, min(n, s0 + per_s)) for s0 in range(0, n, per_s)]
        steps = []

        def copy_steps(part):
            with torch.cuda.stream(cs):
                for s0, s1 in part:
                    for dst, src in ((d_qd, q_dec), (d_kn, k_dec), (d_vn, v_dec)):
                        rows = src.numel() // (n * s.d)           # B*L*H
                        pitch = n * s.d * 2
                        _lib.call("vlc_copy_2d", dst.data_ptr() + s0 * s.d * 2, pitch,
                                  src.data_ptr() + s0 * s.d * 2, pitch, (s1 - s0) * s.d * 2, rows, cs.cuda_stream)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    steps.append((s0, s1, ev))

        copy_steps(bounds[:dec_early])
        for b, l0, l1, ev in groups:
            comp.wait_event(ev)
            self.score_stats_layers(d_qw, d_k, b, l0, l1)
        self.allocate()
        self.select()
        self.gather(d_k, v_prompt)             # keys from the device copy, values zero-copy
        k4_done = torch.cuda.Event()
        k4_done.record(comp)
        cs.wait_event(k4_done)
        copy_steps(bounds[dec_early:])
        for s0, s1, ev in steps:
            if s0 >= self.decode_steps:
                break
            comp.wait_event(ev)
            self.decode(d_qd, d_kn, d_vn, row0=0, first_step=s0, n_steps=min(s1, self.decode_steps) - s0)
        h_counts.copy_(self.kept_counts, non_blocking=True)
        h_out.copy_(self.out, non_blocking=True)
        copied = sum(t.numel() * 2 for t in (q_win, k_prompt, q_dec, k_dec, v_dec))
        if check:
            comp.synchronize()
            self.check()
        return h_counts, h_out, copied

    def zero_copy_bytes(self, host_counts) -> int:
        """Value bytes K4 pulled from host memory: every kept row of every KV head."""
        s = self.shape
        return int(host_counts.sum().item()) * s.Hkv * s.d * 2

    # ------------------------------------------------------------ results
    def exact_stats(self) -> dict:
        """Exact mode's counters from the last K1 call (synchronises): chunks
        (a key x 32 window rows) K1 listed for a float64 re-decision, entries
        deferred to an exact row max, rows scanned for it, `overflow` -- chunks
        that found the list full (their below counts may then differ from the
        reference's) -- and the observed tensor-core errors against exact
        mode's margins.  Empty when exact mode is off."""
        import torch

        if self.exact_ws is None:
            return {}
        w = self.exact_ws[:32].cpu()
        c = w.view(torch.int32).tolist()
        f = w.view(torch.float32).tolist()
        return {"listed": c[1], "deferred": c[0], "rows_scanned": c[3], "overflow": c[2],
                "capacity": self.exact_capacity, "max_logit_err": f[5], "max_rowmax_err": f[6],
                "margin_ok": bool(f[5] + f[6] <= EXACT_BAND_LOGIT / 8 and f[6] <= EXACT_ROWMAX_ERR / 2)}

    def check(self):
        """Synchronise and raise like the reference on a degenerate budget
        (DegenerateSparsityError, reference budget.py:108-109); in exact mode
        also raise ExactnessError when K1's re-decision list overflowed, so a
        below count that may differ from the reference's never passes silently."""
        bad = self.status.nonzero()
        if bad.numel():
            raise DegenerateSparsityError(
                f"every layer is fully sparse; cannot split the budget (batch {bad.flatten().tolist()})")
        if self.exact_ws is not None:
            st = self.exact_stats()
            if st["overflow"]:
                raise ExactnessError(
                    f"exact mode: {st['overflow']} of {st['listed']} near-threshold entries found the "
                    f"re-decision list full (capacity {st['capacity']}) and kept fp32 decisions; "
                    f"construct VLCache(exact_capacity=...) with room for {st['listed']}")
            if not st["margin_ok"]:
                raise ExactnessError(
                    f"exact mode: observed tensor-core logit error {st['max_logit_err']:.3g} / row-max error "
                    f"{st['max_rowmax_err']:.3g} approach the margins K1 decides with ({EXACT_BAND_LOGIT:.3g} / "
                    f"{EXACT_ROWMAX_ERR:.3g} logit units); below counts may differ from the reference's")

    def kept_sets(self):
        """Host copy: kept[b][l][kv] -> int64 numpy array of ascending indices."""
        s = self.shape
        self.check()
        off = self.kept_off.cpu().numpy()
        idx = self.kept_idx[: int(off[-1])].cpu().numpy().astype("int64")
        out = []
        for b in range(s.B):
            layer_rows = []
            for l in range(s.L):
                row = []
                for kv in range(s.Hkv):
                    sl = (b * s.L + l) * s.Hkv + kv
                    row.append(idx[off[sl]:off[sl + 1]])
                layer_rows.append(row)
            out.append(layer_rows)
        return out
