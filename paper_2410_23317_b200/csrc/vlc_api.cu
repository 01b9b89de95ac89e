// vlc_api.cu -- extern "C" boundary (include/vlc.h): argument contracts,
// error codes, and dispatch to the sm_100a kernels.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "../../include/vlc.h"
#include "vlc_kernels.h"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return VLC_OK;
    return fail(VLC_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

float threshold_logit(double p) {
    // walk the float grid around log(p) with the host libm expf -- the same
    // function the reference's compiled kernel calls (_core.pyx:201)
    float x = (float)std::log(p);
    while ((double)expf(x) >= p) x = std::nextafterf(x, -INFINITY);
    while ((double)expf(x) < p) x = std::nextafterf(x, INFINITY);
    return x;
}

float cached_threshold(double p) {
    static std::mutex mu;
    static std::unordered_map<double, float> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(p);
    if (it != cache.end()) return it->second;
    const float t = threshold_logit(p);
    cache.emplace(p, t);
    return t;
}

}  // namespace

extern "C" {

int vlc_abi_version(void) { return 1; }

const char* vlc_strerror(int code) {
    switch (code) {
        case VLC_OK: return "ok";
        case VLC_EINVAL: return "invalid argument";
        case VLC_EUNSUPPORTED: return "unsupported shape";
        case VLC_ECUDA: return "CUDA error";
        default: return "unknown error";
    }
}

const char* vlc_last_error(void) { return g_err; }

float vlc_threshold_logit(double p) { return threshold_logit(p); }

int64_t vlc_score_partials(int64_t rows) { return vlc::score_partials(rows); }

int64_t vlc_score_exact_bytes(int32_t slots, int32_t group, int64_t window, int64_t entries) {
    if (slots < 1 || group < 1 || window < 1 || entries < 1) return -1;
    return vlc::exact_ws_bytes(slots, (int64_t)group * window, entries);
}

static int score_stats_impl(const void* q_win, const void* keys, int32_t slots, int32_t group,
                            int32_t head_dim, int64_t key_rows, int64_t n_keys, int64_t window,
                            int64_t q_base, double p, double scale, const float* stat_max, const float* stat_sum,
                            int64_t stat_ld, int64_t stat_row0, float* row_max, float* row_sum, float* col_partial,
                            uint64_t* below_head, int32_t* below_col, void* exact_ws, int64_t exact_ws_bytes,
                            void* stream);

int vlc_score_stats(const void* q_win, const void* keys, int32_t slots, int32_t group,
                    int32_t head_dim, int64_t key_rows, int64_t n_keys, int64_t window,
                    int64_t q_base, double p, double scale, float* row_max, float* row_sum, float* col_partial,
                    uint64_t* below_head, int32_t* below_col, void* exact_ws, int64_t exact_ws_bytes,
                    void* stream) {
    return score_stats_impl(q_win, keys, slots, group, head_dim, key_rows, n_keys, window, q_base, p, scale,
                            nullptr, nullptr, 0, 0, row_max, row_sum, col_partial, below_head, below_col,
                            exact_ws, exact_ws_bytes, stream);
}

int vlc_score_stats_given(const void* q_win, const void* keys, int32_t slots, int32_t group,
                          int32_t head_dim, int64_t key_rows, int64_t n_keys, int64_t window,
                          int64_t q_base, double p, double scale, const float* stat_max, const float* stat_sum,
                          int64_t stat_ld, float* row_max, float* row_sum, float* col_partial,
                          uint64_t* below_head, int32_t* below_col, void* exact_ws, int64_t exact_ws_bytes,
                          void* stream) {
    if (!stat_max || !stat_sum) return fail(VLC_EINVAL, "score_stats_given: null statistics");
    if (stat_ld < q_base + window) return fail(VLC_EINVAL, "score_stats_given: stat_ld < q_base + window");
    return score_stats_impl(q_win, keys, slots, group, head_dim, key_rows, n_keys, window, q_base, p, scale,
                            stat_max, stat_sum, stat_ld, q_base, row_max, row_sum, col_partial, below_head,
                            below_col, exact_ws, exact_ws_bytes, stream);
}

static int score_stats_impl(const void* q_win, const void* keys, int32_t slots, int32_t group,
                            int32_t head_dim, int64_t key_rows, int64_t n_keys, int64_t window,
                            int64_t q_base, double p, double scale, const float* stat_max, const float* stat_sum,
                            int64_t stat_ld, int64_t stat_row0, float* row_max, float* row_sum, float* col_partial,
                            uint64_t* below_head, int32_t* below_col, void* exact_ws, int64_t exact_ws_bytes,
                            void* stream) {
    if (!q_win || !keys || !row_max || !row_sum || !col_partial || !below_head)
        return fail(VLC_EINVAL, "score_stats: null pointer");
    if (slots < 1 || group < 1 || window < 1 || n_keys < 1 || q_base < 0)
        return fail(VLC_EINVAL, "score_stats: need slots, group, window, n_keys >= 1 and q_base >= 0");
    if (!(p > 0.0 && p < 1.0)) return fail(VLC_EINVAL, "p: must be in (0, 1), got %g", p);
    if (n_keys < q_base + window)
        return fail(VLC_EINVAL, "score_stats: n_keys %lld < q_base + window %lld",
                    (long long)n_keys, (long long)(q_base + window));
    if (key_rows < n_keys) return fail(VLC_EINVAL, "score_stats: key_rows < n_keys");
    if (head_dim != 64 && head_dim != 128)
        return fail(VLC_EUNSUPPORTED, "score_stats: head_dim %d not in {64, 128} (zero-pad and pass scale)", head_dim);
    if ((reinterpret_cast<uintptr_t>(q_win) | reinterpret_cast<uintptr_t>(keys)) & 15)
        return fail(VLC_EINVAL, "score_stats: q_win/keys must be 16-byte aligned");
    vlc::ScoreArgs a{};
    a.q = q_win; a.k = keys; a.slots = slots; a.G = group; a.d = head_dim;
    a.T = key_rows; a.n = n_keys; a.w = window; a.q_base = q_base;
    a.inv_scale = (float)(scale > 0.0 ? scale : 1.0 / std::sqrt((double)head_dim));
    a.t_star = cached_threshold(p);
    a.row_max = row_max; a.row_sum = row_sum; a.col_partial = col_partial;
    a.below_head = reinterpret_cast<unsigned long long*>(below_head);
    a.below_col = below_col;
    a.inv_scale_d = scale > 0.0 ? scale : 1.0 / std::sqrt((double)head_dim);
    a.stat_max = stat_max; a.stat_sum = stat_sum; a.stat_ld = stat_ld; a.stat_row0 = stat_row0;
    if (exact_ws) {
        const int64_t rows = (int64_t)group * window;
        const int cap = vlc::exact_ws_cap(exact_ws_bytes, slots, rows);
        if (cap < 1 || (reinterpret_cast<uintptr_t>(exact_ws) & 255))
            return fail(VLC_EINVAL, "score_stats: exact_ws must be 256-byte aligned and hold "
                                    ">= vlc_score_exact_bytes(slots, group, window, 1) bytes");
        uint8_t* ws = static_cast<uint8_t*>(exact_ws);
        const int64_t rk = (slots * rows * 4 + 255) / 256 * 256;
        a.fix_counts = reinterpret_cast<int*>(ws);
        a.rmax_key = reinterpret_cast<unsigned*>(ws + 256);
        a.rows = reinterpret_cast<int*>(ws + 256 + rk);
        a.cand = reinterpret_cast<int4*>(ws + 256 + 2 * rk);
        a.flag = a.cand + cap;
        a.cap = cap;
        // margins (include/vlc.h); the fix-ups record the errors they observe against them
        a.band = (float)(VLC_EXACT_BAND_LOGIT * 1.4426950408889634);   // log2 units: 2^-9
        a.err_max = (float)VLC_EXACT_ROWMAX_ERR;                         // logit units
    }
    return cuda_status(vlc::launch_score_stats(a, (cudaStream_t)stream), "score_stats");
}

int vlc_allocate(const uint64_t* below_head, int32_t batch, int32_t layers, int32_t q_heads,
                 int32_t kv_heads, int64_t window, int64_t n_keys, int64_t q_base,
                 int64_t prompt_len, double alpha, double beta_min, double beta_max,
                 int64_t cache_extra, double* gamma, double* gamma_mean, double* beta_pre,
                 double* beta, int64_t* kept_counts, int64_t* kept_off, int64_t* cache_off,
                 int32_t* status, void* stream) {
    if (!below_head || !gamma || !gamma_mean || !beta_pre || !beta || !kept_counts || !kept_off ||
        !cache_off || !status)
        return fail(VLC_EINVAL, "allocate: null pointer");
    if (!(alpha > 0.0 && alpha <= 1.0)) return fail(VLC_EINVAL, "alpha: must be in (0, 1], got %g", alpha);
    if (!(beta_min > 0.0 && beta_min <= beta_max))
        return fail(VLC_EINVAL, "beta_min: need 0 < beta_min <= beta_max");
    if (prompt_len < 1) return fail(VLC_EINVAL, "prompt_len: must be >= 1, got %lld", (long long)prompt_len);
    if (batch < 1 || batch > 1024 || layers < 1 || q_heads < 1 || kv_heads < 1 || q_heads % kv_heads)
        return fail(VLC_EINVAL, "allocate: bad batch/layers/heads");
    if (window < 1 || n_keys < q_base + window || cache_extra < 0)
        return fail(VLC_EINVAL, "allocate: bad window");
    // causal entries of one head's window: sum_i min(n, q_base + i + 1)
    int64_t causal = 0;
    for (int64_t i = 0; i < window; ++i) causal += std::min<int64_t>(n_keys, q_base + i + 1);
    vlc::BudgetArgs a{};
    a.below_head = reinterpret_cast<const unsigned long long*>(below_head);
    a.B = batch; a.L = layers; a.Hq = q_heads; a.Hkv = kv_heads;
    a.causal_per_head = causal; a.prompt_len = prompt_len;
    a.alpha_times_L = alpha * (double)layers;   // budget.py:110 "alpha * g.size"
    a.beta_min = beta_min; a.beta_max = beta_max; a.cache_extra = cache_extra;
    a.gamma = gamma; a.gamma_mean = gamma_mean; a.beta_pre = beta_pre; a.beta = beta;
    a.kept_counts = kept_counts; a.kept_off = kept_off; a.cache_off = cache_off; a.status = status;
    return cuda_status(vlc::launch_allocate(a, (cudaStream_t)stream), "allocate");
}

int vlc_allocate_from_gamma(const double* gamma_mean, int32_t batch, int32_t layers,
                            int32_t kv_heads, int64_t prompt_len, double alpha, double beta_min,
                            double beta_max, int64_t cache_extra, double* beta_pre, double* beta,
                            int64_t* kept_counts, int64_t* kept_off, int64_t* cache_off,
                            int32_t* status, void* stream) {
    if (!gamma_mean || !beta_pre || !beta || !kept_counts || !kept_off || !cache_off || !status)
        return fail(VLC_EINVAL, "allocate: null pointer");
    if (!(alpha > 0.0 && alpha <= 1.0)) return fail(VLC_EINVAL, "alpha: must be in (0, 1], got %g", alpha);
    if (!(beta_min > 0.0 && beta_min <= beta_max))
        return fail(VLC_EINVAL, "beta_min: need 0 < beta_min <= beta_max");
    if (prompt_len < 1) return fail(VLC_EINVAL, "prompt_len: must be >= 1, got %lld", (long long)prompt_len);
    if (batch < 1 || batch > 1024 || layers < 1 || kv_heads < 1 || cache_extra < 0)
        return fail(VLC_EINVAL, "allocate: bad batch/layers/heads");
    vlc::BudgetArgs a{};
    a.below_head = nullptr; a.gamma_mean_in = gamma_mean;
    a.B = batch; a.L = layers; a.Hq = 1; a.Hkv = kv_heads; a.prompt_len = prompt_len;
    a.alpha_times_L = alpha * (double)layers;
    a.beta_min = beta_min; a.beta_max = beta_max; a.cache_extra = cache_extra;
    a.gamma = nullptr; a.gamma_mean = const_cast<double*>(gamma_mean);
    a.beta_pre = beta_pre; a.beta = beta;
    a.kept_counts = kept_counts; a.kept_off = kept_off; a.cache_off = cache_off; a.status = status;
    return cuda_status(vlc::launch_allocate(a, (cudaStream_t)stream), "allocate");
}

static int select_impl(const float* col_partial, const double* scores_in, int32_t slots, int32_t kv_heads,
                       int32_t layers, int32_t group, int64_t n_keys, int64_t window,
                       const int64_t* kept_counts, const int64_t* kept_off, double recent_frac,
                       int32_t* kept_idx, int32_t* kept_slot, double* scores_out, uint64_t* key_scratch,
                       void* stream, int scores_ready) {
    if ((!col_partial && !scores_in) || !kept_counts || !kept_off || !kept_idx || !kept_slot)
        return fail(VLC_EINVAL, "select: null pointer");
    if (slots < 1 || kv_heads < 1 || layers < 1 || group < 1 || n_keys < 1 || window < 1)
        return fail(VLC_EINVAL, "select: bad shape");
    if (slots % (kv_heads * layers)) return fail(VLC_EINVAL, "select: slots not a multiple of L*Hkv");
    if (!(recent_frac >= 0.0 && recent_frac <= 1.0))
        return fail(VLC_EINVAL, "recent_window_frac: must be in [0, 1], got %g", recent_frac);
    if (n_keys > (1ll << 31) - 1) return fail(VLC_EUNSUPPORTED, "select: n_keys exceeds int32 indices");
    if (n_keys > 24 * 1024 && !key_scratch)
        return fail(VLC_EINVAL, "select: n_keys > 24576 needs key_scratch");
    vlc::SelectArgs a{};
    a.col_partial = col_partial; a.slots = slots;
    a.nrb = (int)vlc::score_partials((int64_t)group * window);
    a.Hkv = kv_heads; a.L = layers; a.G = group; a.n = n_keys;
    a.kept_counts = kept_counts; a.kept_off = kept_off; a.recent_frac = recent_frac;
    a.kept_idx = kept_idx; a.kept_slot = kept_slot; a.scores = scores_out; a.scores_in = scores_in;
    a.key_scratch = reinterpret_cast<unsigned long long*>(key_scratch);
    a.scores_ready = scores_ready;
    return cuda_status(vlc::launch_select(a, (cudaStream_t)stream), "select");
}

int vlc_select(const float* col_partial, const double* scores_in, int32_t slots, int32_t kv_heads,
               int32_t layers, int32_t group, int64_t n_keys, int64_t window,
               const int64_t* kept_counts, const int64_t* kept_off, double recent_frac,
               int32_t* kept_idx, int32_t* kept_slot, double* scores_out, uint64_t* key_scratch,
               void* stream) {
    return select_impl(col_partial, scores_in, slots, kv_heads, layers, group, n_keys, window, kept_counts,
                       kept_off, recent_frac, kept_idx, kept_slot, scores_out, key_scratch, stream, 0);
}

// K2 waits for every earlier kernel before it releases K3 (pdl_wait_then_release),
// so col_partial is final when K3 launches: K3 reads it before its own wait
int vlc_select_after_allocate(const float* col_partial, const double* scores_in, int32_t slots,
                              int32_t kv_heads, int32_t layers, int32_t group, int64_t n_keys, int64_t window,
                              const int64_t* kept_counts, const int64_t* kept_off, double recent_frac,
                              int32_t* kept_idx, int32_t* kept_slot, double* scores_out, uint64_t* key_scratch,
                              void* stream) {
    if (scores_in) return fail(VLC_EINVAL, "select_after_allocate: scores_in must be NULL");
    return select_impl(col_partial, scores_in, slots, kv_heads, layers, group, n_keys, window, kept_counts,
                       kept_off, recent_frac, kept_idx, kept_slot, scores_out, key_scratch, stream, 1);
}

int vlc_gather(const void* keys, const void* values, int32_t slots, int32_t head_dim,
               int64_t key_rows, const int32_t* kept_idx, const int32_t* kept_slot,
               const int64_t* kept_off, const int64_t* cache_off, int64_t max_rows,
               void* k_cache, void* v_cache, void* stream) {
    if (!keys || !values || !kept_idx || !kept_slot || !kept_off || !cache_off || !k_cache || !v_cache)
        return fail(VLC_EINVAL, "gather: null pointer");
    if (slots < 1 || key_rows < 1 || max_rows < 0) return fail(VLC_EINVAL, "gather: bad shape");
    if (head_dim % 8 || head_dim < 8) return fail(VLC_EUNSUPPORTED, "gather: head_dim %% 8 != 0");
    vlc::GatherArgs a{};
    a.k = keys; a.v = values; a.slots = slots; a.d = head_dim; a.T = key_rows;
    a.kept_idx = kept_idx; a.kept_slot = kept_slot; a.kept_off = kept_off; a.cache_off = cache_off;
    a.max_rows = max_rows; a.k_cache = k_cache; a.v_cache = v_cache;
    return cuda_status(vlc::launch_gather(a, (cudaStream_t)stream), "gather");
}

int64_t vlc_prefill_ws_bytes(int32_t kv_slots, int32_t head_dim, int64_t prompt_len) {
    return (int64_t)kv_slots * head_dim * vlc::prefill_tpad(prompt_len) * 2;
}

int vlc_prefill(const void* q, int64_t q_rows, const void* k, const void* v, int64_t kv_rows, int32_t batch,
                int32_t layers, int32_t q_heads, int32_t kv_heads, int32_t head_dim, int64_t prompt_len, double scale,
                void* ws, int64_t ws_bytes, float* out, float* row_max, float* row_sum, void* stream) {
    if (!q || !k || !v || !ws || !out) return fail(VLC_EINVAL, "prefill: null pointer");
    if ((row_max == nullptr) != (row_sum == nullptr)) return fail(VLC_EINVAL, "prefill: row_max and row_sum go together");
    if (batch < 1 || layers < 1 || q_heads < 1 || kv_heads < 1 || q_heads % kv_heads || prompt_len < 1)
        return fail(VLC_EINVAL, "prefill: bad shape");
    if (head_dim != 64 && head_dim != 128) return fail(VLC_EUNSUPPORTED, "head_dim: %d not in {64, 128}", head_dim);
    if (q_rows < prompt_len || kv_rows < prompt_len) return fail(VLC_EINVAL, "prefill: q_rows / kv_rows < prompt_len");
    const int64_t need = vlc_prefill_ws_bytes(batch * layers * kv_heads, head_dim, prompt_len);
    if (ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255))
        return fail(VLC_EINVAL, "prefill: ws must be 256-byte aligned with %lld bytes", (long long)need);
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(out)) & 15)
        return fail(VLC_EINVAL, "prefill: q / k / out must be 16-byte aligned");
    if (!(scale > 0.0)) return fail(VLC_EINVAL, "scale: must be > 0");
    vlc::PrefillArgs a{};
    a.q = q; a.k = k; a.v = v; a.vt = ws; a.q_rows = q_rows; a.kv_rows = kv_rows; a.m = prompt_len;
    a.B = batch; a.L = layers; a.Hq = q_heads; a.Hkv = kv_heads; a.d = head_dim; a.inv_scale = (float)scale;
    a.out = out; a.row_max = row_max; a.row_sum = row_sum;
    return cuda_status(vlc::launch_prefill(a, (cudaStream_t)stream), "prefill");
}

int vlc_attention_rows(const float* q, const float* k, int32_t heads, int32_t group, int32_t head_dim,
                       int64_t rows, int64_t key_rows, int64_t first_row, int64_t key_limit, int64_t out_cols,
                       double* probs, double filter_p, int64_t prompt_len, int64_t vision_start,
                       int64_t vision_end, double* mass, void* stream) {
    if (!q || !k) return fail(VLC_EINVAL, "attention_rows: null pointer");
    if (!probs && !mass) return fail(VLC_EINVAL, "attention_rows: nothing to write (probs and mass NULL)");
    if (heads < 1 || group < 1 || heads % group || rows < 1 || first_row < 0 || key_limit < 1 || out_cols < 0)
        return fail(VLC_EINVAL, "attention_rows: bad shape");
    if (head_dim < 1 || head_dim > 4096) return fail(VLC_EINVAL, "head_dim: must be in [1, 4096], got %d", head_dim);
    const int64_t span = std::min(key_limit, first_row + rows);
    if (span > key_rows) return fail(VLC_EINVAL, "attention_rows: rows see %lld keys, key_rows is %lld",
                                     (long long)span, (long long)key_rows);
    if (vlc::attention_rows_smem(head_dim, span) > 227 * 1024)
        return fail(VLC_EUNSUPPORTED, "attention_rows: %lld visible keys exceed shared memory", (long long)span);
    if (mass && (vision_start < 0 || vision_end < vision_start || prompt_len < 0))
        return fail(VLC_EINVAL, "attention_rows: bad modality range");
    if (head_dim % 4 == 0 && ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k)) & 15))
        return fail(VLC_EINVAL, "attention_rows: q / k must be 16-byte aligned when head_dim %% 4 == 0");
    vlc::RowsArgs a{};
    a.q = q; a.k = k; a.heads = heads; a.group = group; a.d = head_dim; a.rows = rows; a.key_rows = key_rows;
    a.first_row = first_row; a.key_limit = key_limit; a.out_cols = out_cols;
    a.inv_scale = 1.0 / std::sqrt((double)head_dim);
    a.probs = probs; a.filter_p = filter_p; a.prompt_len = prompt_len;
    a.vis_start = vision_start; a.vis_end = vision_end; a.mass = mass;
    return cuda_status(vlc::launch_attention_rows(a, (cudaStream_t)stream), "attention_rows");
}

int vlc_copy_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                void* stream) {
    if (!dst || !src) return fail(VLC_EINVAL, "copy_2d: null pointer");
    if (width < 0 || height < 0 || dpitch < width || spitch < width) return fail(VLC_EINVAL, "copy_2d: bad extent");
    if (width == 0 || height == 0) return VLC_OK;
    return cuda_status(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)height,
                                         cudaMemcpyDefault, (cudaStream_t)stream), "copy_2d");
}

int vlc_decode_step(const void* q, int64_t q_stride, const void* k_new, const void* v_new,
                    int64_t kv_stride, void* k_cache, void* v_cache, int64_t cache_rows,
                    const int64_t* cache_off,
                    const int64_t* base_len, int64_t step, int32_t batch, int32_t layers,
                    int32_t kv_heads, int32_t group, int32_t head_dim, double scale, int32_t chained,
                    float* out, void* stream) {
    if (!q || !k_new || !v_new || !k_cache || !v_cache || !cache_off || !base_len || !out)
        return fail(VLC_EINVAL, "decode_step: null pointer");
    if ((reinterpret_cast<uintptr_t>(k_cache) | reinterpret_cast<uintptr_t>(v_cache) |
         reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new)) & 15)
        return fail(VLC_EINVAL, "decode_step: buffers must be 16-byte aligned");
    if (batch < 1 || layers < 1 || kv_heads < 1 || group < 1 || step < 0)
        return fail(VLC_EINVAL, "decode_step: bad shape");
    if (group > 8) return fail(VLC_EUNSUPPORTED, "decode_step: group size %d > 8", group);
    if (head_dim != 64 && head_dim != 128)
        return fail(VLC_EUNSUPPORTED, "decode_step: head_dim %d not in {64, 128}", head_dim);
    if (q_stride % 8 || kv_stride % 8) return fail(VLC_EINVAL, "decode_step: strides must be 16-byte multiples");
    vlc::DecodeArgs a{};
    a.q = q; a.q_stride = q_stride; a.k_new = k_new; a.v_new = v_new; a.kv_stride = kv_stride;
    a.k_cache = k_cache; a.v_cache = v_cache; a.cache_off = cache_off; a.base_len = base_len;
    a.cache_rows = cache_rows;
    a.chained = (chained != 0 && step > 0) ? 1 : 0;
    if (cache_rows < 1) return fail(VLC_EINVAL, "decode_step: cache_rows must be >= 1");
    a.step = step; a.slots = batch * layers * kv_heads; a.Hkv = kv_heads; a.L = layers; a.G = group;
    a.d = head_dim; a.out = out;
    // reference _core.pyx:257: inv = <float>(1.0 / sqrt(<double> d))
    a.inv_scale = (float)(scale > 0.0 ? scale : 1.0 / std::sqrt((double)head_dim));
    return cuda_status(vlc::launch_decode(a, (cudaStream_t)stream), "decode_step");
}

int vlc_stats_f32(const float* q, const float* keys, int64_t w, int64_t n, int32_t head_dim, int64_t q_base,
                  double p, int64_t tile, float* row_max, double* row_sum, double* col_score, int64_t* below,
                  int64_t* causal, void* stream) {
    if (!q || !keys || !row_max || !row_sum || !col_score || !below) return fail(VLC_EINVAL, "stats_f32: null pointer");
    if (w < 1 || n < 1 || head_dim < 1 || q_base < 0 || tile < 1)
        return fail(VLC_EINVAL, "stats_f32: need w, n, head_dim, tile >= 1 and q_base >= 0");
    if (n < q_base + w)
        return fail(VLC_EINVAL, "stats_f32: n %lld < q_base + w %lld", (long long)n, (long long)(q_base + w));
    if (!(p >= 0.0)) return fail(VLC_EINVAL, "p: must be >= 0, got %g", p);
    vlc::SeamStatsArgs a{};
    a.q = q; a.k = keys; a.w = w; a.n = n; a.q_base = q_base; a.tile = tile; a.d = head_dim;
    a.inv = 1.0 / std::sqrt((double)head_dim);   // reference _core.pyx:222
    a.p = p; a.row_max = row_max; a.row_sum = row_sum; a.col_score = col_score; a.below = below; a.causal = causal;
    return cuda_status(vlc::launch_seam_stats(a, (cudaStream_t)stream), "stats_f32");
}

int vlc_decode_f32(const float* q, int32_t g, const float* keys, const float* values, int64_t n, int32_t head_dim,
                   float* scratch, double* denom, float* out, void* stream) {
    if (!q || !keys || !values || !scratch || !denom || !out) return fail(VLC_EINVAL, "decode_f32: null pointer");
    if (g < 1 || g > 65535 || n < 1 || head_dim < 1) return fail(VLC_EINVAL, "decode_f32: need g in [1, 65535], n, head_dim >= 1");
    vlc::SeamDecodeArgs a{};
    a.q = q; a.k = keys; a.v = values; a.n = n; a.g = g; a.d = head_dim;
    a.inv = (float)(1.0 / std::sqrt((double)head_dim));   // reference _core.pyx:257
    a.scratch = scratch; a.denom = denom; a.out = out;
    return cuda_status(vlc::launch_seam_decode(a, (cudaStream_t)stream), "decode_f32");
}

}  // extern "C"
