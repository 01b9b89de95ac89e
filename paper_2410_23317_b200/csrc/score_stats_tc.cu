// score_stats_tc.cu -- K1 on the 5th-generation tensor cores (sm_100a).
//
// reference: pkg/src/vlcache/_kernels/_core.pyx:110-242 (two-pass tiled
// statistics) for all G query heads of a KV head at once.
//
// CTA = (slot, block of 128 window rows).  Warp roles (384 threads):
//   warp 0      TMA producer: the Q block once, then every 128-key tile of the
//               slot twice (pass 1, pass 2) into a 3-stage swizzled ring
//   warp 1      MMA issuer, M=128 x N=128, K = head_dim, bf16 in, fp32
//               accumulate in TMEM (two accumulator stages, 256 columns).
//               Pass 1 computes Q K^T (rows on TMEM lanes), pass 2 K Q^T
//               (keys on TMEM lanes) from the same shared-memory operands.
//   warp 2      TMEM allocator
//   warps 4-11  epilogue, tcgen05.ld 32 columns at a time:
//               pass 1: thread = window row -> running max / sum (serial);
//               pass 2: thread = key -> column mass and below-threshold
//               counts, serial over the block's rows, so neither pass needs a
//               cross-lane reduction per entry.
// The score matrix never leaves the SM: TMEM -> registers -> statistics.
#include <cuda.h>

#include "vlc_common.cuh"
#include "sm100.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kM = 128;          // window rows per CTA (UMMA M)
constexpr int kN = 128;          // keys per tile (UMMA N)
#ifndef VLC_K1_STAGES
#define VLC_K1_STAGES 3
#endif
#ifndef VLC_K1_SUB
#define VLC_K1_SUB 32
#endif
#ifndef VLC_K1_MINB
#define VLC_K1_MINB 1
#endif
constexpr int kStages = VLC_K1_STAGES;   // K tile ring
constexpr int kSub = VLC_K1_SUB;         // TMEM columns an epilogue thread holds at a time (16 / 32)
constexpr int kNSub = 32 / kSub;
constexpr int kEpiWarps = 16;    // 4 per TMEM lane quarter, one 32-column group each
constexpr int kThreads = 128 + kEpiWarps * 32;
constexpr uint32_t kTmemCols = 2 * kN;

template <int D>
struct Layout {
    static constexpr int KB = D / 64;                       // 64-element (128 B) k-blocks
    static constexpr uint32_t kQRegion = kM * 128;          // bytes per Q k-block
    static constexpr uint32_t kKRegion = kN * 128;          // bytes per K k-block
    static constexpr uint32_t kQBytes = KB * kQRegion;
    static constexpr uint32_t kKBytes = KB * kKRegion;      // one stage
    static constexpr uint32_t kBytes = kQBytes + kStages * kKBytes + 1024;   // + alignment slack
};

template <int N>
VLC_DEV float maxn(const float (&l)[N]) {
    float m[N / 4];
#pragma unroll
    for (int k = 0; k < N / 4; ++k) m[k] = fmaxf(fmaxf(l[4 * k], l[4 * k + 1]), fmaxf(l[4 * k + 2], l[4 * k + 3]));
#pragma unroll
    for (int w = N / 8; w >= 1; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) m[k] = fmaxf(m[k], m[k + w]);
    return m[0];
}

template <int N>
VLC_DEV void tmem_ld(uint32_t taddr, float (&v)[N]) {
    if constexpr (N == 32) sm100::tmem_ld32(taddr, v);
    else sm100::tmem_ld16(taddr, v);
}

template <int D, bool EXACT>
__global__ void __launch_bounds__(kThreads, VLC_K1_MINB)
score_stats_tc(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
               ScoreArgs a, int nparts) {
    using LY = Layout<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // small state in static shared memory (plain LDS/STS, not generic accesses)
    __shared__ uint64_t full[kStages], empty[kStages], qfull[1], tfull[2], tempty[2];
    __shared__ uint32_t tmem_slot[1];
    __shared__ float2 rowstat[4 * kM];                  // (max, sum) per column group and row
    __shared__ __align__(16) float c_mb[kM];            // row max (raw dot) * c1
    __shared__ __align__(16) float c_is[kM];            // 1 / row sum (0: no row)
    __shared__ __align__(16) float c_t2[kM];            // threshold on u (-inf: no row)
    __shared__ int c_lim[kM];                           // last visible key (-1: no row)
    __shared__ int hcnt[kM];                            // below counts per head of the block

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.y, rb = blockIdx.x;
    const int64_t R = (int64_t)a.G * a.w;
    const int64_t r_first = (int64_t)rb * kM;
    const int64_t r_last = imin(R, r_first + kM) - 1;
    const int64_t i_max = (r_last / a.w == r_first / a.w) ? r_last % a.w : a.w - 1;
    const int64_t blk_end = imin(a.n, a.q_base + i_max + 1);   // keys any row here can see
    const int T = (int)((blk_end + kN - 1) / kN);
    const int iters = 2 * T;
    const int64_t head0 = r_first / a.w;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) { sm100::mbar_init(full + i, 1); sm100::mbar_init(empty + i, 1); }
        sm100::mbar_init(qfull, 1);
        for (int i = 0; i < 2; ++i) { sm100::mbar_init(tfull + i, 1); sm100::mbar_init(tempty + i, kEpiWarps); }
        sm100::fence_barrier_init();
        sm100::fence_proxy_async();
    }
    if (threadIdx.x < kM) hcnt[threadIdx.x] = 0;
    if (warp == 2) sm100::tmem_alloc(tmem_slot, kTmemCols);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ------------------------------------------------ TMA producer
        sm100::tma_prefetch(&qmap);
        sm100::tma_prefetch(&kmap);
        sm100::mbar_expect_tx(qfull, LY::kQBytes);
        for (int kb = 0; kb < LY::KB; ++kb)
            sm100::tma_load_2d(smem + kb * LY::kQRegion, &qmap, qfull, kb * 64, (int)(s * R + r_first));
        for (int it = 0; it < iters; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            const int t = it < T ? it : it - T;
            sm100::mbar_wait(empty + st, ph ^ 1);
            sm100::mbar_expect_tx(full + st, LY::kKBytes);
            uint8_t* kdst = smem + LY::kQBytes + st * LY::kKBytes;
            for (int kb = 0; kb < LY::KB; ++kb)
                sm100::tma_load_2d(kdst + kb * LY::kKRegion, &kmap, full + st, kb * 64,
                                   (int)(s * a.T + (int64_t)t * kN));
        }
    } else if (warp == 1 && lane == 0) {
        // ------------------------------------------------ MMA issuer
        // pass 1: D[row, key] = Q K^T (rows on TMEM lanes); pass 2: D[key, row]
        // = K Q^T (keys on TMEM lanes) -- same operands, swapped roles
        constexpr uint32_t idesc = sm100::idesc_bf16_f32(kM, kN);
        const uint32_t q_addr = sm100::smem_u32(smem);
        sm100::mbar_wait(qfull, 0);
        for (int it = 0; it < iters; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            const int acc = it & 1;
            const uint32_t aph = (it >> 1) & 1;
            sm100::mbar_wait(tempty + acc, aph ^ 1);
            sm100::mbar_wait(full + st, ph);
            sm100::tc_fence_after();
            const uint32_t k_addr = sm100::smem_u32(smem + LY::kQBytes + st * LY::kKBytes);
            const bool rows_on_lanes = it < T;
#pragma unroll
            for (int kb = 0; kb < LY::KB; ++kb) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {   // 4 x 16 elements = one 128 B swizzle row
                    const uint64_t qd = sm100::sdesc_k_sw128(q_addr + kb * LY::kQRegion + kk * 32);
                    const uint64_t kd = sm100::sdesc_k_sw128(k_addr + kb * LY::kKRegion + kk * 32);
                    sm100::mma_bf16(tmem + acc * kN, rows_on_lanes ? qd : kd, rows_on_lanes ? kd : qd, idesc,
                                    (kb | kk) != 0);
                }
            }
            sm100::mma_commit(empty + st);   // K stage reusable once these MMAs retire
            sm100::mma_commit(tfull + acc);  // accumulator ready for the epilogue
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        // warp -> (TMEM lane quarter `sub`, 32-column group `cg`)
        const int ew = warp - 4, sub = warp & 3, cg = ew >> 2;
        const int lane_idx = 32 * sub + lane;                  // TMEM lane of this thread
        const uint32_t lane_addr = tmem + (uint32_t(32 * sub) << 16) + cg * 32;
        const float c1 = a.inv_scale * kLog2e;
        float l[kSub];

        // ---- pass 1 (thread = window row): running max of raw dots, rescaled sum
        {
            const int64_t r = r_first + lane_idx;
            const bool row_ok = r < R;
            const int64_t i = row_ok ? r % a.w : 0;
            const int64_t row_end = row_ok ? imin(a.n, a.q_base + i + 1) : 0;
            float m = -INFINITY, sum = 0.f;
            for (int it = 0; it < T; ++it) {
                const int acc = it & 1;
                sm100::mbar_wait(tfull + acc, (it >> 1) & 1);
                sm100::tc_fence_after();
#pragma unroll
                for (int h = 0; h < kNSub; ++h) {
                tmem_ld(lane_addr + acc * kN + h * kSub, l);
                if (h == kNSub - 1) {
                    sm100::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) sm100::mbar_arrive(tempty + acc);   // registers hold the chunk now
                }
                const int valid = (int)imax(0, imin(kSub, row_end - ((int64_t)it * kN + cg * 32 + h * kSub)));
                const bool full_chunk = __all_sync(kFull, valid == kSub);
                float cmax;
                if (full_chunk) {
                    cmax = maxn(l);
                } else {
                    cmax = -INFINITY;
#pragma unroll
                    for (int k = 0; k < kSub; ++k) cmax = k < valid ? fmaxf(cmax, l[k]) : cmax;
                }
                if (cmax > m) {
                    sum *= ex2((m - cmax) * c1);   // 0 while m == -inf
                    m = cmax;
                }
                const float mb = m * c1;
                float acc_s = 0.f;
                if (full_chunk) {
#pragma unroll
                    for (int k = 0; k < kSub; ++k) acc_s += ex2(fmaf(l[k], c1, -mb));
                } else {
#pragma unroll
                    for (int k = 0; k < kSub; ++k) acc_s += k < valid ? ex2(fmaf(l[k], c1, -mb)) : 0.f;
                }
                sum += acc_s;
                }
            }
            rowstat[cg * kM + lane_idx] = make_float2(m, sum);
            sm100::named_bar_sync(1, kEpiWarps * 32);
            if (cg == 0) {
                float M = -INFINITY;
#pragma unroll
                for (int g4 = 0; g4 < 4; ++g4) M = fmaxf(M, rowstat[g4 * kM + lane_idx].x);
                float S = 0.f;
#pragma unroll
                for (int g4 = 0; g4 < 4; ++g4) {
                    const float2 h = rowstat[g4 * kM + lane_idx];
                    if (h.x != -INFINITY) S += h.y * ex2((h.x - M) * c1);
                }
                if (row_ok) {
                    a.row_max[(int64_t)s * R + r] = M * a.inv_scale;
                    a.row_sum[(int64_t)s * R + r] = S;
                    c_mb[lane_idx] = M * c1;
                    c_is[lane_idx] = 1.f / S;
                    c_t2[lane_idx] = a.t_star * kLog2e;
                    c_lim[lane_idx] = (int)(a.q_base + i);
                } else {
                    c_mb[lane_idx] = INFINITY;    // u = -inf: no mass
                    c_is[lane_idx] = 0.f;
                    c_t2[lane_idx] = -INFINITY;   // never below
                    c_lim[lane_idx] = -1;         // sees no key
                }
            }
            sm100::named_bar_sync(1, kEpiWarps * 32);
        }

        // ---- pass 2 (thread = key): column mass and below-threshold counts over
        //   the 32 rows of group cg.  u = l*c1 - mb_r ~ log2(exp(logit - max));
        //   below <=> u < t* log2e; mass = 2^(u - log2 S_r).  Serial per key: no
        //   cross-lane reduction, and every key column follows the same order.
        //   Each row group writes its own partial row of col_partial (no barrier).
        const int r0 = cg * 32;
        const int64_t rg = r_first + r0;
        const bool one_head = rg / a.w == (rg + 31) / a.w;
        float* colp = a.col_partial + ((int64_t)s * nparts + rb * 4 + cg) * a.n;
        for (int it = T; it < iters; ++it) {
            const int acc = it & 1;
            const int t = it - T;
            const int j = t * kN + lane_idx;                     // this thread's key
            const bool all_visible = (int64_t)t * kN + kN - 1 <= a.q_base;   // CTA-uniform
            sm100::mbar_wait(tfull + acc, (it >> 1) & 1);
            sm100::tc_fence_after();
            // exact mode: an entry whose decision u < t2 is within `band` of flipping
            // (fp32 logits vs the reference's float64 dots) is not counted here but
            // listed for a float64 re-decision.  band = 0: plain decisions.
            const float band = EXACT ? a.band : 0.f;
            float csum = 0.f;
            int cnt = 0;
#pragma unroll
            for (int h = 0; h < kNSub; ++h) {
            const int rh = r0 + h * kSub;                        // first row of this sub-chunk
            float cntf = 0.f, cnth = 0.f;                        // cnth - cntf: entries inside the band
            tmem_ld(lane_addr + acc * kN + h * kSub, l);
            if (h == kNSub - 1) {
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(tempty + acc);
            }
            // per entry: u = l*c1 - mb_r (log2 of exp(logit - max)), below <=> u < t2_r,
            // mass += 2^u * (1 / S_r) -- one FFMA, one MUFU, one FFMA; the count
            // as a float (set + add).  The same operation order in every branch,
            // so identical key columns give bit-identical mass.
            const float4* mb4 = reinterpret_cast<const float4*>(c_mb + rh);
            const float4* is4 = reinterpret_cast<const float4*>(c_is + rh);
            if (all_visible && r_first + r0 + 31 < R) {   // every row real and every key visible
                const float t2c = a.t_star * kLog2e, t2lo = t2c - band;
#pragma unroll
                for (int q4 = 0; q4 < kSub / 4; ++q4) {
                    const float4 mb = mb4[q4], iv = is4[q4];
                    const float mbv[4] = {mb.x, mb.y, mb.z, mb.w}, ivv[4] = {iv.x, iv.y, iv.z, iv.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float u = fmaf(l[4 * q4 + e], c1, -mbv[e]);
                        cntf += u < t2lo ? 1.f : 0.f;
                        if (EXACT) cnth += u < t2c + band ? 1.f : 0.f;
                        csum = fmaf(ex2(u), ivv[e], csum);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < kSub; ++k) {
                    const bool vis = all_visible || j <= c_lim[rh + k];
                    const float u = fmaf(l[k], c1, -c_mb[rh + k]);
                    const float t2 = c_t2[rh + k];
                    cntf += (vis && u < t2 - band) ? 1.f : 0.f;
                    if (EXACT) cnth += (vis && u < t2 + band) ? 1.f : 0.f;
                    csum = vis ? fmaf(ex2(u), c_is[rh + k], csum) : csum;
                }
            }
            if (EXACT && __any_sync(kFull, cnth != cntf)) {
                // reserve this thread's entries with one atomic, then write them
                const int nf = (int)(cnth - cntf);
                int at = nf ? atomicAdd(a.fix_counts + 1, nf) : 0;
#pragma unroll
                for (int k = 0; k < kSub; ++k) {   // static indices: l stays in registers
                    const bool vis = j < a.n && (all_visible || j <= c_lim[rh + k]);
                    const float u = fmaf(l[k], c1, -c_mb[rh + k]);
                    const float t2 = c_t2[rh + k];
                    if (nf && vis && u >= t2 - band && u < t2 + band) {
                        if (at < a.cap) {
                            a.flag[at] = make_int4(s, (int)(r_first + rh + k), j, 1);
                        } else {   // list full: keep the fp32 decision
                            atomicAdd(a.fix_counts + 2, 1);
                            cnt += u < t2 ? 1 : 0;
                        }
                        ++at;
                    }
                }
            }
            cnt += (int)cntf;
            if (!one_head) {
#pragma unroll
                for (int k = 0; k < kSub; ++k) {
                    const bool vis = all_visible || j <= c_lim[rh + k];
                    const float u = fmaf(l[k], c1, -c_mb[rh + k]);
                    const int tot = __reduce_add_sync(kFull, (vis && u < c_t2[rh + k] - band) ? 1 : 0);
                    if (lane == 0 && tot) atomicAdd(hcnt + (int)((r_first + rh + k) / a.w - head0), tot);
                }
            }
            }
            if (j < a.n) colp[j] = csum;
            if (a.below_col && cnt && j < a.n) atomicAdd(a.below_col + (int64_t)s * a.n + j, cnt);
            // per-head totals (warp reduce, one shared atomic per warp)
            if (one_head) {   // (mixed-head groups were counted row by row above)
                const int tot = __reduce_add_sync(kFull, cnt);
                if (lane == 0 && tot) atomicAdd(hcnt + (int)(rg / a.w - head0), tot);
            }
        }
        // columns no row of this block can see
        for (int64_t jj = (int64_t)T * kN + lane_idx; jj < a.n; jj += kN) colp[jj] = 0.f;
        sm100::named_bar_sync(1, kEpiWarps * 32);
        const int nheads = (int)(r_last / a.w - head0 + 1);
        for (int h = ew * 32 + lane; h < nheads; h += kEpiWarps * 32)
            if (hcnt[h]) atomicAdd(a.below_head + (int64_t)s * a.G + head0 + h, (unsigned long long)hcnt[h]);
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(tmem, kTmemCols);
    }
}

// ---------------------------------------------------------------- host side
template <int D, bool EXACT>
cudaError_t launch_tc_e(const ScoreArgs& a, int nparts, cudaStream_t st) {
    CUtensorMap qmap, kmap;
    const int64_t R = (int64_t)a.G * a.w;
    if (!make_tmap_2d(&qmap, a.q, (int64_t)a.slots * R, a.d, kM)) return cudaErrorInvalidValue;
    if (!make_tmap_2d(&kmap, a.k, (int64_t)a.slots * a.T, a.d, kN)) return cudaErrorInvalidValue;
    const size_t sm = Layout<D>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(score_stats_tc<D, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 grid(nparts / 4, a.slots);
    score_stats_tc<D, EXACT><<<grid, kThreads, sm, st>>>(qmap, kmap, a, nparts);
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_tc(const ScoreArgs& a, int nparts, cudaStream_t st) {
    return a.cap > 0 ? launch_tc_e<D, true>(a, nparts, st) : launch_tc_e<D, false>(a, nparts, st);
}

}  // namespace

cudaError_t launch_score_stats_tc(const ScoreArgs& a, int nparts, cudaStream_t st) {
    if (a.d == 64) return launch_tc<64>(a, nparts, st);
    if (a.d == 128) return launch_tc<128>(a, nparts, st);
    return cudaErrorInvalidValue;
}

}  // namespace vlc
