// score_stats.cu -- K1 launcher: zeroes the count outputs, runs the tcgen05
// kernel (score_stats_tc.cu) and, in exact mode, the float64 fix-up of the
// entries K1 listed.  reference _core.pyx:210-242.
//
// Exact mode.  The reference decides "below" as expf(l32 - rmax) < p with
// l32 = float32(float64 dot(q, k) * (1/sqrt(d))) and rmax the float32 row max
// (_core.pyx:144-145, 201-204), i.e. l32 - rmax < t* (vlc_threshold_logit).
// K1's logits come from fp32 tensor-core accumulation, a few ulps away.  K1
// decides every entry farther than `band` (log2 units, ~100x that error) from
// the threshold itself and lists the rest.  Here each listed entry gets its
// exact logit from a float64 dot (bf16 products are exact in float64 and their
// sums order-independent) and is decided against K1's row max when it is
// farther than that max's own error from the threshold; the few that are not
// wait for their row's exact max (a float64 scan of the row's visible keys).
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {

// col_partial rows per slot: 2 row halves of 64 rows per 128-row block
int score_partials(int64_t rows) { return (int)(2 * ((rows + 127) / 128)); }

namespace {

constexpr int64_t kAlign = 256;
int64_t up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// order-preserving float <-> unsigned (0 is below every float key)
VLC_DEV unsigned fkey(float x) {
    const unsigned u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
VLC_DEV float funkey(unsigned k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); }

// float32(float64 dot(q_row, k_row) * inv) over bf16 operands
VLC_DEV float exact_logit(const ScoreArgs& a, int slot, int row, int key) {
    const int64_t R = (int64_t)a.G * a.w;
    const uint4* q = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.q) + ((int64_t)slot * R + row) * a.d);
    const uint4* k = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.k) + ((int64_t)slot * a.T + key) * a.d);
    double acc = 0.0;
    for (int c = 0; c < a.d / 8; ++c) {
        const uint4 qv = q[c], kv = k[c];
        const uint32_t qa[4] = {qv.x, qv.y, qv.z, qv.w}, ka[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            acc = fma((double)bf16_lo(qa[e]), (double)bf16_lo(ka[e]), acc);
            acc = fma((double)bf16_hi(qa[e]), (double)bf16_hi(ka[e]), acc);
        }
    }
    return (float)(acc * a.inv_scale_d);
}

VLC_DEV void add_below(const ScoreArgs& a, const int4& e) {
    atomicAdd(a.below_head + (int64_t)e.x * a.G + e.y / a.w, (unsigned long long)e.w);
    if (a.below_col) atomicAdd(a.below_col + (int64_t)e.x * a.n + e.z, e.w);
}

// 1: decide each listed entry against K1's row max; undecidable ones (within
// the row max's own error of the threshold) wait for the exact row max
__global__ void fix_flags(ScoreArgs a) {
    const int n = min(a.fix_counts[1], a.cap);
    const int64_t R = (int64_t)a.G * a.w;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int4 e = a.flag[i];
        const int64_t rr = (int64_t)e.x * R + e.y;
        const float x = exact_logit(a, e.x, e.y, e.z) - a.row_max[rr];
        if (x < a.t_star - a.err_max) {
            add_below(a, e);
        } else if (x < a.t_star + a.err_max) {
            const int at = atomicAdd(a.fix_counts, 1);
            if (at < a.cap) {
                a.cand[at] = e;
            } else {   // no room: decide against the fp32 row max
                atomicAdd(a.fix_counts + 2, 1);
                if (x < a.t_star) add_below(a, e);
            }
            if (atomicExch(a.rmax_key + rr, 1u) == 0u) a.rows[atomicAdd(a.fix_counts + 3, 1)] = (int)rr;
        }
    }
}

// 2: exact row max of each listed row, one key per thread (blockIdx.x walks a
// row's keys, blockIdx.y the listed rows), combined with atomicMax on the
// order-preserving key
__global__ void fix_rowscan(ScoreArgs a) {
    const int nrows = a.fix_counts[3];
    const int64_t R = (int64_t)a.G * a.w;
    for (int q = blockIdx.y; q < nrows; q += gridDim.y) {
        const int64_t rr = a.rows[q];
        const int slot = (int)(rr / R), row = (int)(rr % R);
        const int64_t lim = imin(a.n, a.q_base + row % a.w + 1);
        float mx = -INFINITY;
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < lim; j += (int64_t)gridDim.x * blockDim.x)
            mx = fmaxf(mx, exact_logit(a, slot, row, (int)j));
        mx = warp_max(mx);
        if ((threadIdx.x & 31) == 0 && mx != -INFINITY) atomicMax(a.rmax_key + rr, fkey(mx));
    }
}

// 3: the waiting entries against the exact row max, which also replaces the
// fp32 row max of those rows
__global__ void fix_deferred(ScoreArgs a) {
    const int n = min(a.fix_counts[0], a.cap);
    const int64_t R = (int64_t)a.G * a.w;
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int4 e = a.cand[i];
        if (exact_logit(a, e.x, e.y, e.z) - funkey(a.rmax_key[(int64_t)e.x * R + e.y]) < a.t_star) add_below(a, e);
    }
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < a.fix_counts[3]; q += stride) {
        const int64_t rr = a.rows[q];
        a.row_max[rr] = funkey(a.rmax_key[rr]);
    }
}

}  // namespace

int64_t exact_ws_bytes(int64_t slots, int64_t rows, int64_t cap) {
    return kAlign + 2 * up(slots * rows * 4) + 2 * cap * 16;
}

int exact_ws_cap(int64_t bytes, int64_t slots, int64_t rows) {
    const int64_t cap = (bytes - kAlign - 2 * up(slots * rows * 4)) / 32;
    return (int)(cap > (1 << 30) ? (1 << 30) : cap);
}

cudaError_t launch_score_stats(const ScoreArgs& a, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(a.below_head, 0, sizeof(unsigned long long) * a.slots * a.G, st);
    if (e != cudaSuccess) return e;
    if (a.below_col) {
        e = cudaMemsetAsync(a.below_col, 0, sizeof(int) * a.slots * a.n, st);
        if (e != cudaSuccess) return e;
    }
    if (a.cap > 0) {
        e = cudaMemsetAsync(a.fix_counts, 0, 4 * sizeof(int), st);
        if (e == cudaSuccess) e = cudaMemsetAsync(a.rmax_key, 0, sizeof(unsigned) * a.slots * a.G * a.w, st);
        if (e != cudaSuccess) return e;
    }
    e = launch_score_stats_tc(a, score_partials((int64_t)a.G * a.w), st);
    if (e != cudaSuccess || a.cap <= 0) return e;
    fix_flags<<<296, 256, 0, st>>>(a);
    fix_rowscan<<<dim3(16, 148), 256, 0, st>>>(a);
    fix_deferred<<<148, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace vlc
