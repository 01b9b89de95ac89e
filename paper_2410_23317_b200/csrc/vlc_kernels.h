// vlc_kernels.h -- internal launcher interface between the C-ABI (vlc_api.cu)
// and the sm_100a kernels.  Not part of the public boundary (see include/vlc.h).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace vlc {

// 2-D bf16 TMA map over [rows, d] (row-major): box = 64 elements (one 128-byte
// swizzle row) x box_rows, SWIZZLE_128B.  False if the driver entry is missing.
bool make_tmap_2d(CUtensorMap* map, const void* base, int64_t rows, int d, int box_rows);
// 2-D bf16 TMA map over `rows` rows of `cols` elements, `row_stride` elements
// apart (multiple of 8): box = 64 x box_rows, SWIZZLE_128B or none.
bool make_tmap_2d_strided(CUtensorMap* map, const void* base, int64_t rows, int cols, int64_t row_stride,
                          int box_rows, bool swizzle);

constexpr int kDecodeChunk = 32;   // keys per K5 bulk-copy stage
constexpr int kDecodeCluster = 8;  // CTAs per (b, l, kv) slot in K5 (one cluster)

// Exact-mode workspace of K1: [counts (256 B)] [rmax_key u32 slots*R] [rows
// i32 slots*R] (each 256 B aligned) [cand int4 x cap] [flag int4 x cap].
int64_t exact_ws_bytes(int64_t slots, int64_t rows, int64_t cap);
int exact_ws_cap(int64_t bytes, int64_t slots, int64_t rows);    // <= 0: too small

// K1: post-vision attention statistics for every (b, l, kv) slot.
// Slot s = (b*L + l)*Hkv + kv owns window rows [s*R, s*R + R), R = G*w, i.e.
// heads kv*G .. kv*G+G-1 of the [B, L, Hq, w, d] window tensor.
// K1's epilogue chunk: TMEM columns a thread holds at a time, and so the rows of
// one exact-mode listing record (score_stats_tc.cu, score_stats.cu)
#ifndef VLC_K1_SUB
#define VLC_K1_SUB 32
#endif
constexpr int kScoreSub = VLC_K1_SUB;

struct ScoreArgs {
    const void* q;          // bf16 [B*L*Hq, w, d]   (window query rows)
    const void* k;          // bf16 [B*L*Hkv, T, d]  (keys; rows >= n never read)
    int slots, G, d;
    int64_t T, n, w, q_base;
    float inv_scale, t_star;
    float* row_max;                    // [slots*R]
    float* row_sum;                    // [slots*R]
    float* col_partial;                // [slots, score_partials(G*w), n] column sums per 64-row half
    unsigned long long* below_head;    // [slots*G]  (zeroed by the launcher)
    int* below_col;                    // optional [slots, n] (zeroed by the launcher)
    // exact mode (fix != nullptr): entries whose below-threshold decision is
    // within `band` (log2 units) of flipping, and the near-max entries that
    // decide the row max, are listed and re-decided in float64 afterwards
    int* fix_counts;                   // device [n_defer, n_flag, overflow, n_rows, n_scan, max logit err (f32), max row-max err (f32), -] (zeroed by the launcher)
    unsigned* rmax_key;                // [slots*R] 1 = row listed, then key of its exact f32 max (0 = none)
    int* rows;                         // [slots*R] rows whose exact max is needed
    int4* cand;                        // [cap] (slot, row, key, mult) entries waiting for an exact row max
    int4* flag;                        // [cap] (slot, row, key, mult) near-threshold entries
    int cap;                           // 0: exact mode off
    float band;                        // log2 units, K1's listing band
    float err_max;                     // logit units: |fp32 row max - exact row max| bound
    double inv_scale_d;                // the reference's 1/sqrt(d) (or scale) in double
    // row statistics given (f2 fusion): the prefill's exact row max (logit
    // units) and row sum of every prompt row; K1 then runs pass 2 only.
    // Row i of head g in slot s is at ((s*G + g) * stat_ld + stat_row0 + i).
    const float* stat_max;
    const float* stat_sum;
    int64_t stat_ld, stat_row0;
};
int score_partials(int64_t rows);    // col_partial rows per slot for R window rows
cudaError_t launch_score_stats(const ScoreArgs& a, cudaStream_t st);
cudaError_t launch_score_stats_tc(const ScoreArgs& a, int nparts, cudaStream_t st);  // head_dim 64 / 128

// K2: numpy-exact gamma -> gamma' -> beta -> kept counts, plus ragged offsets.
struct BudgetArgs {
    const unsigned long long* below_head;  // [B, L, Hq]  (NULL: gamma_mean_in given)
    const double* gamma_mean_in;           // [B, L]  used when below_head is NULL
    int B, L, Hq, Hkv;
    int64_t causal_per_head;   // sum of causal entries of one head's window
    int64_t prompt_len;        // m (kept counts clip to [1, m])
    double alpha_times_L, beta_min, beta_max;
    int64_t cache_extra;       // headroom rows per cache segment (decode appends)
    double* gamma;             // [B, L, Hq]
    double* gamma_mean;        // [B, L]
    double* beta_pre;          // [B, L]
    double* beta;              // [B, L]
    int64_t* kept_counts;      // [B, L]
    int64_t* kept_off;         // [B*L*Hkv + 1]  prefix of kept counts per slot
    int64_t* cache_off;        // [B*L*Hkv + 1]  prefix of (kept + cache_extra)
    int* status;               // [B]  0 ok, 1 degenerate (Z == 0)
};
cudaError_t launch_allocate(const BudgetArgs& a, cudaStream_t st);

// K3: per-slot top-k with recent reserve -> ascending kept indices.
struct SelectArgs {
    const float* col_partial;  // [slots, nrb, n]  (nrb = score_partials rows)
    int slots, nrb, Hkv, L, G;
    int64_t n;                 // prompt_len m
    const int64_t* kept_counts;  // [B, L]
    const int64_t* kept_off;     // [slots + 1]
    double recent_frac;
    int32_t* kept_idx;         // [sum k]
    int32_t* kept_slot;        // [sum k]  slot of each kept row
    double* scores;            // optional out [slots, n]
    const double* scores_in;   // optional in [slots, n]: rank these instead of col_partial
    unsigned long long* key_scratch;  // [slots, n] when n > 24576
    int scores_ready;          // col_partial final at launch (K2 precedes): sum before the PDL wait
};
cudaError_t launch_select(const SelectArgs& a, cudaStream_t st);

// K4: compact kept K/V rows into ragged per-slot cache segments.
struct GatherArgs {
    const void* k;             // bf16 [slots, T, d]
    const void* v;             // bf16 [slots, T, d]
    int slots, d;
    int64_t T;
    const int32_t* kept_idx;   // [sum k]
    const int32_t* kept_slot;  // [sum k]
    const int64_t* kept_off;   // [slots + 1]
    const int64_t* cache_off;  // [slots + 1]
    int64_t max_rows;          // host upper bound on sum k (grid sizing)
    void* k_cache;             // bf16 [cache rows, d]
    void* v_cache;
};
cudaError_t launch_gather(const GatherArgs& a, cudaStream_t st);

// K5: one decode step over the ragged compressed cache (append + attend).
struct DecodeArgs {
    const void* q;             // bf16, head (b,l,h) at q + idx*q_stride
    int64_t q_stride;          // elements between consecutive (b,l,h) heads
    const void* k_new;         // bf16, slot s at k_new + s*kv_stride
    const void* v_new;
    int64_t kv_stride;
    void* k_cache;
    void* v_cache;
    const int64_t* cache_off;  // [slots + 1]
    const int64_t* base_len;   // [B, L] rows present before step 0 (kept counts)
    int64_t step;              // rows appended so far = step
    int slots, Hkv, L, G, d;
    float inv_scale;
    float* out;                // f32 [B*L*Hq, d]
    int64_t cache_rows;        // rows of k_cache / v_cache (TMA bounds)
    int chained;               // the previous kernel on the stream is decode step `step - 1`
    int early;                 // set by the launcher: release the successor at once (see decode.cu)
};
cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t st);
cudaError_t launch_decode_wide(const DecodeArgs& a, cudaStream_t st);   // decode_wide.cu

// f2: causal prefill attention over the prompt (prefill.cu).
struct PrefillArgs {
    const void* q;             // bf16 [B*L*Hq, q_rows, d] (prompt rows first)
    const void* k;             // bf16 [B*L*Hkv, kv_rows, d]
    const void* v;
    void* vt;                  // workspace: bf16 V^T [B*L*Hkv, d, prefill_tpad(m)]
    int64_t q_rows, kv_rows, m;
    int B, L, Hq, Hkv, d;
    float inv_scale;
    float* out;                // f32 [B*L*Hq, m, d]
    float* row_max;            // f32 [B*L*Hq, m] (logit units) or null
    float* row_sum;            // f32 [B*L*Hq, m] (sum of exp(l - max)) or null
};
int64_t prefill_tpad(int64_t m);
cudaError_t launch_prefill(const PrefillArgs& a, cudaStream_t st);

// f4 analysis: dense causal softmax rows over fp32 trace rows (eval_rows.cu).
struct RowsArgs {
    const float* q;            // f32 [heads, rows, d]: query rows first_row .. first_row+rows-1
    const float* k;            // f32 [heads / group, key_rows, d]
    int64_t heads, group, d, rows, key_rows, first_row;
    int64_t key_limit;         // row r sees keys [0, min(key_limit, first_row + r + 1))
    int64_t out_cols;          // probs columns written per row (zeros past the visible keys)
    double inv_scale;          // 1 / sqrt(d) in double
    double* probs;             // f64 [heads*rows, out_cols] or null
    double filter_p;           // threshold filter (keep prob >= p * row max) for mass
    int64_t prompt_len, vis_start, vis_end;
    double* mass;              // f64 [heads*rows, 3]: filtered (vision, language, prompt) mass, or null
};
int64_t attention_rows_smem(int64_t d, int64_t span);
cudaError_t launch_attention_rows(const RowsArgs& a, cudaStream_t st);

// The reference kernel seam's float32 contract (seam_f32.cu).
struct SeamStatsArgs {
    const float* q;            // f32 [w, d]
    const float* k;            // f32 [n, d]
    int64_t w, n, q_base, tile;
    int d;
    double inv;                // 1 / sqrt(d), float64
    double p;
    float* row_max;            // f32 [w]
    double* row_sum;           // f64 [w]
    double* col_score;         // f64 [n]
    int64_t* below;            // i64 [n]
    int64_t* causal;           // i64 [n] or null
};
cudaError_t launch_seam_stats(const SeamStatsArgs& a, cudaStream_t st);

struct SeamDecodeArgs {
    const float* q;            // f32 [g, d]
    const float* k;            // f32 [n, d]
    const float* v;            // f32 [n, d]
    int64_t n;
    int g, d;
    float inv;                 // float32(1 / sqrt(d))
    float* scratch;            // f32 [g, n]
    double* denom;             // f64 [g]
    float* out;                // f32 [g, d]
};
cudaError_t launch_seam_decode(const SeamDecodeArgs& a, cudaStream_t st);

}  // namespace vlc
