/*
 * vlc.h -- C-ABI of the B200 (sm_100a) VL-Cache compress + compressed-decode path.
 *
 * Shared library: paper_2410_23317_b200/libvlc_b200.so (built by
 * __graft_entry__.build()).  Plain pointers and sizes only; every pointer
 * argument is DEVICE memory owned by the caller unless stated otherwise, every
 * call is ordered on `stream` (a cudaStream_t / CUstream, NULL = legacy
 * default) and returns 0 or a negative VLC_E* code; vlc_last_error() gives the
 * message of the last failure on the calling thread.  No global mutable
 * state: calls on different streams may run concurrently.
 *
 * It replaces the reference's kernel seam `vlcache._kernels`
 * (reference pkg/src/vlcache/_kernels/__init__.py:10-27, which binds
 * _core.stats_tiled / _core.decode_step), batched over every
 * (batch b, layer l, KV head kv) "slot" at once, plus the numpy stages the
 * reference runs between those kernels (budget.py, scoring.py, bench.py).
 *
 * Data layout (row-major, contiguous, bf16 = IEEE bfloat16):
 *   window queries  q_win [B, L, Hq, w, d]     the w scoring rows of each head
 *   keys / values   [B, L, Hkv, T, d]          T >= n_keys (+ decode rows)
 *   slot s = (b*L + l)*Hkv + kv ; head h = kv*G + g, G = Hq/Hkv
 *   window row r of slot s = g*w + i  (i = position in the window)
 */
#ifndef VLC_H
#define VLC_H

#include <stdint.h>

#if defined(__GNUC__)
#define VLC_API __attribute__((visibility("default")))
#else
#define VLC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define VLC_OK 0
#define VLC_EINVAL (-1)       /* argument contract violated  -> ValidationError   */
#define VLC_EUNSUPPORTED (-2) /* shape outside this build     -> ValidationError   */
#define VLC_ECUDA (-3)        /* CUDA launch/runtime failure  -> KernelError        */

VLC_API int vlc_abi_version(void);
VLC_API const char *vlc_strerror(int code);
VLC_API const char *vlc_last_error(void);

/* float32 t* = smallest x with (double)expf(x) >= p (host libm expf): the
 * below-threshold test "(double)expf(l - max) < p" of reference
 * _core.pyx:201-204 is exactly "l - max < t*". */
VLC_API float vlc_threshold_logit(double p);

/* Rows of col_partial per slot for a window of `rows` = G*w rows (one
 * partial per 64 window rows; 2 per 128-row block). */
VLC_API int64_t vlc_score_partials(int64_t rows);

/*
 * K1 score_stats.  Replaces _kernels.stats_tiled (reference _core.pyx:210-242)
 * for all G heads of every slot: causal logits q.k/sqrt(d) of window row
 * (absolute index q_base + i) against keys [0, min(n_keys, q_base+i+1)).
 *   row_max, row_sum : f32 [slots*G*w]       (_core.pyx:142-155)
 *   col_partial      : f32 [slots, vlc_score_partials(G*w), n_keys] column
 *                      mass of each 64-row half (their sum is the slot's
 *                      col_score summed over its G heads)
 *   below_head       : u64 [slots*G]  entries with exp(l - max) < p, per head
 *   below_col        : i32 [slots, n_keys] or NULL (per-column counts)
 * scale <= 0 selects 1/sqrt(head_dim) (zero-padded operands pass the true d's).
 * exact_ws (NULL: off) -- exact mode: every below decision within a small
 * band of flipping, and the near-max entries of every row, are re-decided
 * from float64 dots exactly as the reference computes them, so below counts
 * and row_max equal the reference's for bf16-representable inputs.
 * exact_ws: 256-byte aligned, >= vlc_score_exact_bytes(slots, group, window,
 * E) bytes for room for E listed chunks (a key x 32 window rows each; E >=
 * slots*G*w is ample; beyond capacity the fp32 decisions are kept).  After the call (stream-ordered) its
 * first 32 bytes hold the status words, int32 unless noted:
 *   [0] entries deferred to an exact row max   [1] chunks listed by K1
 *   [2] OVERFLOW: chunks that found the list full (their near-threshold
 *       entries stay undecided: the below counts may differ from the reference's)
 *   [3] rows whose exact max was recomputed    [4] keys the row scan listed
 *   [5] f32: largest observed difference between a listed chunk's smallest
 *       |logit - threshold| from the tensor cores and from float64 (logit units)
 *   [6] f32: largest observed |fp32 row max - exact row max| (recomputed rows)
 * [5] and [6] check the margins exact mode relies on (VLC_EXACT_BAND_LOGIT,
 * VLC_EXACT_ROWMAX_ERR): callers treat [5] + [6] > VLC_EXACT_BAND_LOGIT / 8
 * or [6] > VLC_EXACT_ROWMAX_ERR / 2 like an overflow.
 * Requires n_keys >= q_base + window, head_dim in {64, 128} (zero-pad smaller
 * dims and pass their scale), 16-byte aligned q_win / keys.
 */
/* exact mode's fixed margins (logit units): K1 decides itself every entry
 * farther than BAND from the threshold; the fix-up decides against K1's fp32
 * row max when farther than ROWMAX_ERR */
#define VLC_EXACT_BAND_LOGIT (1.0 / 512.0 / 1.4426950408889634)
#define VLC_EXACT_ROWMAX_ERR (1.0 / 512.0 / 1.4426950408889634 / 16.0)
VLC_API int64_t vlc_score_exact_bytes(int32_t slots, int32_t group, int64_t window, int64_t entries);
VLC_API int vlc_score_stats(const void *q_win, const void *keys, int32_t slots, int32_t group,
                    int32_t head_dim, int64_t key_rows, int64_t n_keys, int64_t window,
                    int64_t q_base, double p, double scale, float *row_max, float *row_sum,
                    float *col_partial, uint64_t *below_head, int32_t *below_col,
                    void *exact_ws, int64_t exact_ws_bytes, void *stream);

/*
 * K1 riding on the prefill (row f2): as vlc_score_stats, but the window rows'
 * softmax statistics come from vlc_prefill (stat_max in logit units, stat_sum;
 * [B*L*Hq, stat_ld] with the window at columns q_base .. q_base + window - 1),
 * so K1 runs its column pass only.  row_max / row_sum echo the given values.
 */
VLC_API int vlc_score_stats_given(const void *q_win, const void *keys, int32_t slots, int32_t group,
                    int32_t head_dim, int64_t key_rows, int64_t n_keys, int64_t window, int64_t q_base,
                    double p, double scale, const float *stat_max, const float *stat_sum, int64_t stat_ld,
                    float *row_max, float *row_sum, float *col_partial, uint64_t *below_head,
                    int32_t *below_col, void *exact_ws, int64_t exact_ws_bytes, void *stream);

/*
 * K2 allocate.  gamma[b,l,h] = below/causal (reference sparsity.py:79),
 * gamma_mean = mean over heads (sparsity.py:41-43), then
 * allocate_sparsity_aware (budget.py:86-111): bit-identical to numpy given
 * equal counts.  Also the ragged offsets of kept sets (kept_off) and of cache
 * segments of kept + cache_extra rows (cache_off), both [B*L*Hkv + 1].
 * status[b] = 1 when every layer of prompt b is fully sparse (Z == 0,
 * budget.py:108-109 -> DegenerateSparsityError).
 */
VLC_API int vlc_allocate(const uint64_t *below_head, int32_t batch, int32_t layers, int32_t q_heads,
                 int32_t kv_heads, int64_t window, int64_t n_keys, int64_t q_base,
                 int64_t prompt_len, double alpha, double beta_min, double beta_max,
                 int64_t cache_extra, double *gamma, double *gamma_mean, double *beta_pre,
                 double *beta, int64_t *kept_counts, int64_t *kept_off, int64_t *cache_off,
                 int32_t *status, void *stream);

/* K2 from a given gamma_mean [B, L] (reference budget.allocate_sparsity_aware
 * called directly on measured sparsity, budget.py:86-111). */
VLC_API int vlc_allocate_from_gamma(const double *gamma_mean, int32_t batch, int32_t layers,
                 int32_t kv_heads, int64_t prompt_len, double alpha, double beta_min,
                 double beta_max, int64_t cache_extra, double *beta_pre, double *beta,
                 int64_t *kept_counts, int64_t *kept_off, int64_t *cache_off, int32_t *status,
                 void *stream);

/*
 * K3 select.  score = (sum of the slot's column mass) / G (reference
 * scoring.py:185-201) -- or, when scores_in (f64 [slots, n_keys]) is given,
 * those scores; then evict (scoring.py:213-235): the last
 * min(ceil(recent_frac*k), k) positions plus the top of the rest by score,
 * ties toward the larger index (scoring.py:204-210).  k of slot s is
 * kept_counts[s / kv_heads].  Writes ascending indices into
 * kept_idx[kept_off[s] ...] and the owning slot into kept_slot.
 * scores_out (f64 [slots, n_keys]) may be NULL; key_scratch (u64
 * [slots, n_keys]) is required only when n_keys > 24576.
 */
VLC_API int vlc_select(const float *col_partial, const double *scores_in, int32_t slots,
               int32_t kv_heads, int32_t layers, int32_t group, int64_t n_keys, int64_t window,
               const int64_t *kept_counts, const int64_t *kept_off, double recent_frac,
               int32_t *kept_idx, int32_t *kept_slot, double *scores_out, uint64_t *key_scratch,
               void *stream);

/*
 * vlc_select for a launch that directly follows vlc_allocate /
 * vlc_allocate_from_gamma on the same stream, with col_partial written before
 * that allocation (the engine's compress order K1 -> K2 -> K3).  Same
 * arguments and results; K3 sums and ranks the scores while K2 still runs and
 * waits for K2 only to read the budgets.  scores_in must be NULL.
 */
VLC_API int vlc_select_after_allocate(const float *col_partial, const double *scores_in, int32_t slots,
               int32_t kv_heads, int32_t layers, int32_t group, int64_t n_keys, int64_t window,
               const int64_t *kept_counts, const int64_t *kept_off, double recent_frac,
               int32_t *kept_idx, int32_t *kept_slot, double *scores_out, uint64_t *key_scratch,
               void *stream);

/*
 * K4 gather.  Copies keys/values[s, kept_idx] into the cache segment of slot s
 * (reference bench.py:331-353).  max_rows: host upper bound on sum of kept
 * counts (sizes the grid; the device total is kept_off[slots]).
 */
VLC_API int vlc_gather(const void *keys, const void *values, int32_t slots, int32_t head_dim,
               int64_t key_rows, const int32_t *kept_idx, const int32_t *kept_slot,
               const int64_t *kept_off, const int64_t *cache_off, int64_t max_rows,
               void *k_cache, void *v_cache, void *stream);

/*
 * K5 decode step `step` (0-based).  Appends k_new/v_new of every slot at row
 * base_len[b,l] + step of its segment, then out[b,l,h] = softmax(q.K^T/sqrt(d)) V
 * over the first base_len + step + 1 rows (reference bench.py:362-372 +
 * _core.pyx:245-278).  q head (b,l,h) is at q + ((b*L+l)*Hq+h)*q_stride,
 * slot s's new row at k_new/v_new + s*kv_stride (elements).  out: f32
 * [B*L*Hq, head_dim].  head_dim in {64, 128}, G <= 8; scale as in K1.
 * k_cache / v_cache: bf16 [cache_rows, head_dim], 16-byte aligned, rows that
 * no step has written yet must hold finite values (zero-initialise once).
 * No workspace; one CTA per slot.  Launched with programmatic dependent
 * launch: chained != 0 promises that the previous kernel on `stream` is this
 * cache's step `step - 1`, letting the step prefetch every row but that
 * step's append while the previous kernel drains (pass 0 otherwise).
 */
VLC_API int vlc_decode_step(const void *q, int64_t q_stride, const void *k_new, const void *v_new,
                    int64_t kv_stride, void *k_cache, void *v_cache, int64_t cache_rows,
                    const int64_t *cache_off,
                    const int64_t *base_len, int64_t step, int32_t batch, int32_t layers,
                    int32_t kv_heads, int32_t group, int32_t head_dim, double scale, int32_t chained,
                    float *out, void *stream);

/*
 * Staging helper: `height` rows of `width` bytes, `spitch` / `dpitch` bytes
 * apart, host or device to host or device, ordered on `stream` (asynchronous
 * from pinned host memory).  Used to stream a strided slab of the host inputs
 * (e.g. the rows of a group of decode steps) while earlier stages compute.
 */
VLC_API int vlc_copy_2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width,
                    int64_t height, void *stream);

/*
 * Prefill: causal attention of the m prompt rows
 * of every query head, out[s, r] = softmax_j<=r(q_r . k_j * scale) V (reference
 * bench.py:196-234 _prefill_layer), on tcgen05, plus the exact per-row softmax
 * statistics the compression path needs (row_max in logit units as K1's, row_sum
 * = sum exp(l - max); NULL to skip).  q: bf16 [B*L*Hq, q_rows, d]; k, v: bf16
 * [B*L*Hkv, kv_rows, d] (q_rows, kv_rows >= m); head_dim in {64, 128}.  P is
 * rounded to bf16 for the P V product (relative error ~2^-9 per weight, as
 * every tensor-core attention).  out: f32 [B*L*Hq, m, d].  ws: device
 * workspace of vlc_prefill_ws_bytes() bytes (V^T), 256-byte aligned.
 */
VLC_API int64_t vlc_prefill_ws_bytes(int32_t kv_slots, int32_t head_dim, int64_t prompt_len);
VLC_API int vlc_prefill(const void *q, int64_t q_rows, const void *k, const void *v, int64_t kv_rows,
                    int32_t batch, int32_t layers, int32_t q_heads, int32_t kv_heads, int32_t head_dim,
                    int64_t prompt_len, double scale, void *ws, int64_t ws_bytes, float *out,
                    float *row_max, float *row_sum, void *stream);

/*
 * Analysis rows.  Dense causal softmax of fp32
 * query rows against fp32 keys: row r (absolute query first_row + r) of head h
 * sees keys [0, min(key_limit, first_row + r + 1)) of KV head h / group;
 *   probs[h, r, j] = double(e_j) / sum double(e),  e_j = float32 exp(l_j - max l),
 *   l_j = float32(float64 dot(q, k_j) * (1/sqrt(d)))
 * exactly as reference attention.py:72-90 (dense_attention_rows, key_limit =
 * first_row + rows) and evaluate.py:78-104 (oracle_scores, key_limit = m).
 * q: f32 [heads, rows, d]; k: f32 [heads/group, key_rows, d] (16-byte aligned
 * when d % 4 == 0, the vector path).
 * probs: f64 [heads*rows, out_cols] or NULL (zeros past the visible keys).
 * mass: f64 [heads*rows, 3] or NULL: after the threshold filter (keep
 * prob >= filter_p * row max; sparsity.py:46-66) the mass on prompt columns
 * [vision_start, vision_end), on the other prompt columns [0, prompt_len), and
 * their sum (evaluate.py:161-185).  Visible key span <= ~55K (shared memory).
 */
VLC_API int vlc_attention_rows(const float *q, const float *k, int32_t heads, int32_t group,
                    int32_t head_dim, int64_t rows, int64_t key_rows, int64_t first_row,
                    int64_t key_limit, int64_t out_cols, double *probs, double filter_p,
                    int64_t prompt_len, int64_t vision_start, int64_t vision_end, double *mass,
                    void *stream);

/*
 * The reference kernel seam's float32 contract, for the numpy-in / numpy-out
 * drop-in of vlcache._kernels (paper_2410_23317_b200._kernels):
 *
 * vlc_stats_f32 replaces _core.stats_tiled (reference _core.pyx:210-242):
 * q f32 [w, d], keys f32 [n, d] (n >= q_base + w), row r sees keys j <= q_base
 * + r; the reference's arithmetic restated per operation (float64 dots,
 * float32 logits and exps, float64 sums, `tile`-key blocks in pass 1).
 * Outputs row_max f32 [w], row_sum f64 [w], col_score f64 [n], below i64 [n],
 * causal i64 [n] (NULL to skip).  Device pointers.
 *
 * vlc_decode_f32 replaces _core.decode_step (reference _core.pyx:245-278):
 * q f32 [g, d], keys / values f32 [n, d] -> out f32 [g, d]; scratch f32
 * [g, n] and denom f64 [g] are caller workspace.
 *
 * One (layer, head) per call, launch-bound by design; the batched bf16 path is
 * vlc_score_stats .. vlc_decode_step.
 */
VLC_API int vlc_stats_f32(const float *q, const float *keys, int64_t w, int64_t n, int32_t head_dim,
                    int64_t q_base, double p, int64_t tile, float *row_max, double *row_sum,
                    double *col_score, int64_t *below, int64_t *causal, void *stream);
VLC_API int vlc_decode_f32(const float *q, int32_t g, const float *keys, const float *values, int64_t n,
                    int32_t head_dim, float *scratch, double *denom, float *out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* VLC_H */
