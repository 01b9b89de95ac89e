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

#ifndef VLC_RS_X
#define VLC_RS_X 24   // exact row scan: blocks per row
#endif
#ifndef VLC_RS_Y
#define VLC_RS_Y 48   // rows in flight: 24 x 48 CTAs = one resident wave (148 was 2.5 us slower at M7B, where few rows are scanned)
#endif
#ifndef VLC_RS_U
#define VLC_RS_U 4    // keys per half-warp in flight
#endif
constexpr int64_t kAlign = 256;
int64_t up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// order-preserving float <-> unsigned (0 is below every float key)
VLC_DEV unsigned fkey(float x) {
    const unsigned u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
VLC_DEV float funkey(unsigned k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); }

// float32(float64 dot(q_row, k_row) * inv) over bf16 operands; D known at
// compile time so all 2*D/8 16-byte loads are in flight before the fp64 chain
template <int D>
VLC_DEV float exact_logit(const ScoreArgs& a, int slot, int row, int key) {
    const int64_t R = (int64_t)a.G * a.w;
    const uint4* q = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.q) + ((int64_t)slot * R + row) * D);
    const uint4* k = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.k) + ((int64_t)slot * a.T + key) * D);
    uint4 qv[D / 8], kv[D / 8];
#pragma unroll
    for (int c = 0; c < D / 8; ++c) { qv[c] = q[c]; kv[c] = k[c]; }
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < D / 8; ++c) {
        const uint32_t qa[4] = {qv[c].x, qv[c].y, qv[c].z, qv[c].w}, ka[4] = {kv[c].x, kv[c].y, kv[c].z, kv[c].w};
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

// 1: K1 listed chunks -- key j x kSub consecutive window rows (.y = the first)
// -- holding an entry within its band of a decision.  One warp per chunk,
// lane = row: each entry gets its exact logit and is decided against K1's row
// max, or waits for the exact row max when within that max's own error of the
// threshold (the exact logit travels in the waiting entry's .w).  Lane 0
// compares the chunk's smallest exact |u| with the tensor-core one K1 saw
// (the runtime margin check).
template <int D>
__global__ void fix_flags(ScoreArgs a) {
    pdl_wait_then_release();
    const int n = min(a.fix_counts[1], a.cap);
    const int64_t R = (int64_t)a.G * a.w;
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x / 32;
    for (int i = blockIdx.x * wpb + threadIdx.x / 32; i < n; i += gridDim.x * wpb) {
        const int4 f = a.flag[i];
        const int row = f.y + lane;
        const bool ok = lane < kScoreSub && row < R && f.z <= a.q_base + (row % a.w) && f.z < a.n;
        float minu = INFINITY;
        if (ok) {
            const int4 e = make_int4(f.x, row, f.z, 1);
            const int64_t rr = (int64_t)e.x * R + e.y;
            const float l = exact_logit<D>(a, e.x, e.y, e.z);
            const float x = l - a.row_max[rr];
            minu = fabsf((x - a.t_star) * kLog2e);
            if (x < a.t_star - a.err_max) {
                add_below(a, e);
            } else if (x < a.t_star + a.err_max) {
                const int at = atomicAdd(a.fix_counts, 1);
                if (at < a.cap) {
                    a.cand[at] = make_int4(e.x, e.y, e.z, __float_as_int(l));
                } else {   // no room: decide against the fp32 row max
                    atomicAdd(a.fix_counts + 2, 1);
                    if (x < a.t_star) add_below(a, e);
                }
                if (atomicExch(a.rmax_key + rr, 1u) == 0u) a.rows[atomicAdd(a.fix_counts + 3, 1)] = (int)rr;
            }
        }
        minu = warp_min(minu);
        if (lane == 0 && minu != INFINITY)
            atomicMax(reinterpret_cast<unsigned*>(a.fix_counts + 5),
                      __float_as_uint(fabsf(minu - __int_as_float(f.w)) / kLog2e));
    }
}

// fp64 dot of one bf16 query row and one bf16 key row, sequential (the
// reference's order)
template <int D>
VLC_DEV float exact_dot(const uint4* q, const uint4* k, double inv) {
    double acc = 0.0;
#pragma unroll 8
    for (int c = 0; c < D / 8; ++c) {
        const uint4 qv = q[c], kv = k[c];
        const uint32_t qa[4] = {qv.x, qv.y, qv.z, qv.w}, ka[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            acc = fma((double)bf16_lo(qa[e]), (double)bf16_lo(ka[e]), acc);
            acc = fma((double)bf16_hi(qa[e]), (double)bf16_hi(ka[e]), acc);
        }
    }
    return (float)(acc * inv);
}

// 2: exact row max of each listed row (blockIdx.y walks the listed rows,
// blockIdx.x and the half-warps of a block walk the row's keys), combined with
// atomicMax on the order-preserving key.  A half-warp reads one key row
// coalesced (16 lanes x 16 B for D = 128) and forms its float32 dot and
// sum |q k| by shuffles; only keys whose dot plus the rigorous fp32 error bound
// ((D + 4) 2^-24 sum |q k|, any summation order) reaches K1's row max minus
// its error bound get the float64 dot.
template <int D>
__global__ void __launch_bounds__(256) fix_rowscan(ScoreArgs a) {
    pdl_wait_then_release();
    constexpr int kLanes = D / 8;                 // lanes per key: 16 B each
    constexpr int kPerWarp = 32 / kLanes;         // keys per warp and step
    constexpr float kRel = (float)(D + 4) * 5.9604645e-8f;
    const int nrows = a.fix_counts[3];
    const int64_t R = (int64_t)a.G * a.w;
    const int lane = threadIdx.x & 31, sub = lane % kLanes, grp = lane / kLanes;
    const int64_t kslot0 = (int64_t)blockIdx.x * (blockDim.x / 32) * kPerWarp + (threadIdx.x / 32) * kPerWarp + grp;
    const int64_t kstride = (int64_t)gridDim.x * (blockDim.x / 32) * kPerWarp;
    for (int q = blockIdx.y; q < nrows; q += gridDim.y) {
        const int64_t rr = a.rows[q];
        const int slot = (int)(rr / R), row = (int)(rr % R);
        const int64_t lim = imin(a.n, a.q_base + row % a.w + 1);
        const float floor_logit = a.row_max[rr] - a.err_max;   // exact max >= this
        const uint4* qrow = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.q) + ((int64_t)slot * R + row) * D);
        const uint4 qv = qrow[sub];
        const uint32_t qa[4] = {qv.x, qv.y, qv.z, qv.w};
        float mx = -INFINITY;
        constexpr int kU = VLC_RS_U;   // keys per half-warp in flight
        for (int64_t j0 = kslot0 - grp; j0 < lim; j0 += kU * kstride) {   // warp-uniform trip count
            uint4 kv[kU];
            const uint4* krow[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t j = j0 + grp + u * kstride;
                krow[u] = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.k) +
                                                         ((int64_t)slot * a.T + (j < lim ? j : 0)) * D);
                kv[u] = krow[u][sub];
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t j = j0 + grp + u * kstride;
                const uint32_t ka[4] = {kv[u].x, kv[u].y, kv[u].z, kv[u].w};
                float f = 0.f, sa = 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float q0 = bf16_lo(qa[e]), q1 = bf16_hi(qa[e]), k0 = bf16_lo(ka[e]), k1 = bf16_hi(ka[e]);
                    f = fmaf(q1, k1, fmaf(q0, k0, f));
                    sa = fmaf(fabsf(q1), fabsf(k1), fmaf(fabsf(q0), fabsf(k0), sa));
                }
#pragma unroll
                for (int o = kLanes / 2; o >= 1; o >>= 1) {
                    f += __shfl_xor_sync(kFull, f, o);
                    sa += __shfl_xor_sync(kFull, sa, o);
                }
                const float hi = (f + 2.f * kRel * sa) * a.inv_scale;
                const bool lst = j < lim && sub == 0 && hi >= floor_logit - fabsf(floor_logit) * 1e-6f;
                // list it (the flag list is free once fix_flags ran; scored in parallel
                // next) -- one counter atomic per warp: rows whose max ties across many
                // keys (the generator's planted keys) list hundreds of them
                const unsigned bal = __ballot_sync(kFull, lst);
                if (bal) {
                    int base = 0;
                    if (lane == __ffs(bal) - 1) base = atomicAdd(a.fix_counts + 4, __popc(bal));
                    base = __shfl_sync(kFull, base, __ffs(bal) - 1);
                    if (lst) {
                        const int at = base + __popc(bal & ((1u << lane) - 1u));
                        if (at < a.cap) a.flag[at] = make_int4(slot, row, (int)j, 0);
                        else mx = fmaxf(mx, exact_dot<D>(qrow, krow[u], a.inv_scale_d));
                    }
                }
            }
        }
        mx = warp_max(mx);
        if (lane == 0 && mx != -INFINITY) atomicMax(a.rmax_key + rr, fkey(mx));
    }
}

// 2b: the row scan's candidates, one float64 dot per thread
template <int D>
__global__ void fix_rowmax(ScoreArgs a) {
    pdl_wait_then_release();
    const int n = min(a.fix_counts[4], a.cap);
    const int64_t R = (int64_t)a.G * a.w;
    const int stride = gridDim.x * blockDim.x;
    const int n_up = (n + 31) / 32 * 32;   // warp-uniform trip count (the match below needs full warps)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_up; i += stride) {
        const bool ok = i < n;
        const int4 e = a.flag[ok ? i : 0];
        unsigned key = 0u;
        int64_t rr = -1;
        if (ok) {
            const uint4* q = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.q) + ((int64_t)e.x * R + e.y) * D);
            const uint4* k = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.k) + ((int64_t)e.x * a.T + e.z) * D);
            key = fkey(exact_dot<D>(q, k, a.inv_scale_d));
            rr = (int64_t)e.x * R + e.y;
        }
        // lanes of the same row (listed consecutively) reduce first: one atomicMax per row and warp
        const unsigned peers = __match_any_sync(kFull, (unsigned long long)rr);
        const unsigned m = __reduce_max_sync(peers, key);
        if (ok && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMax(a.rmax_key + rr, m);
    }
}

// 3: the waiting entries against the exact row max, which also replaces the
// fp32 row max of those rows
__global__ void fix_deferred(ScoreArgs a) {
    pdl_wait_then_release();
    const int n = min(a.fix_counts[0], a.cap);
    const int64_t R = (int64_t)a.G * a.w;
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int4 e = a.cand[i];
        if (__int_as_float(e.w) - funkey(a.rmax_key[(int64_t)e.x * R + e.y]) < a.t_star)
            add_below(a, make_int4(e.x, e.y, e.z, 1));
    }
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < a.fix_counts[3]; q += stride) {
        const int64_t rr = a.rows[q];
        const float exact = funkey(a.rmax_key[rr]);
        atomicMax(reinterpret_cast<unsigned*>(a.fix_counts + 6), __float_as_uint(fabsf(exact - a.row_max[rr])));
        a.row_max[rr] = exact;
    }
}

template <int D>
cudaError_t launch_fixups(const ScoreArgs& a, cudaStream_t st) {
    cudaError_t e = launch_pdl(fix_flags<D>, dim3(592), dim3(256), 0, st, a);
    if (e == cudaSuccess) e = launch_pdl(fix_rowscan<D>, dim3(VLC_RS_X, VLC_RS_Y), dim3(256), 0, st, a);
    if (e == cudaSuccess) e = launch_pdl(fix_rowmax<D>, dim3(296), dim3(256), 0, st, a);
    if (e == cudaSuccess) e = launch_pdl(fix_deferred, dim3(148), dim3(256), 0, st, a);
    return e;
}

}  // namespace

int64_t exact_ws_bytes(int64_t slots, int64_t rows, int64_t cap) {
    return kAlign + 2 * up(slots * rows * 4) + 2 * cap * 16;
}

int exact_ws_cap(int64_t bytes, int64_t slots, int64_t rows) {
    const int64_t cap = (bytes - kAlign - 2 * up(slots * rows * 4)) / 32;
    return (int)(cap > (1 << 30) ? (1 << 30) : cap);
}

// the count outputs and exact mode's counters / row keys, zeroed in one launch
__global__ void zero_outputs(unsigned* p0, int64_t n0, unsigned* p1, int64_t n1, unsigned* p2, int64_t n2,
                             unsigned* p3, int64_t n3) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // K1's prologue and pass 1 run under it
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n0 + n1 + n2 + n3; i += stride) {
        if (i < n0) p0[i] = 0u;
        else if (i < n0 + n1) p1[i - n0] = 0u;
        else if (i < n0 + n1 + n2) p2[i - n0 - n1] = 0u;
        else p3[i - n0 - n1 - n2] = 0u;
    }
}

cudaError_t launch_score_stats(const ScoreArgs& a, cudaStream_t st) {
    const int64_t nh = 2 * (int64_t)a.slots * a.G;                       // u64 below_head
    const int64_t nc = a.below_col ? (int64_t)a.slots * a.n : 0;
    const int64_t nf = a.cap > 0 ? 8 : 0, nr = a.cap > 0 ? (int64_t)a.slots * a.G * a.w : 0;
    const int64_t tot = nh + nc + nf + nr;
    zero_outputs<<<(unsigned)imin(4 * 148, (tot + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<unsigned*>(a.below_head), nh, reinterpret_cast<unsigned*>(a.below_col), nc,
        reinterpret_cast<unsigned*>(a.fix_counts), nf, a.rmax_key, nr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = launch_score_stats_tc(a, score_partials((int64_t)a.G * a.w), st);
    if (e != cudaSuccess || a.cap <= 0) return e;
#ifdef VLC_FIX_PROBE   // timing probe (wrong results): 1 = no fix-up launches, 2 = fix_flags only
    if (VLC_FIX_PROBE == 1) return cudaGetLastError();
    if (VLC_FIX_PROBE == 2) {
        e = a.d == 64 ? launch_pdl(fix_flags<64>, dim3(592), dim3(256), 0, st, a)
                      : launch_pdl(fix_flags<128>, dim3(592), dim3(256), 0, st, a);
        return e != cudaSuccess ? e : cudaGetLastError();
    }
#endif
    e = a.d == 64 ? launch_fixups<64>(a, st) : launch_fixups<128>(a, st);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace vlc
