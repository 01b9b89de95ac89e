// score_stats_tc.cu -- K1 on the 5th-generation tensor cores (sm_100a).
//
// reference: pkg/src/vlcache/_kernels/_core.pyx:110-242 (two-pass tiled
// statistics) for all G query heads of a KV head at once.
//
// CTA = (slot, block of 128 window rows).  Warp roles (640 threads):
//   warp 0      TMA producer: the Q block once, then every 128-key tile of the
//               slot twice (pass 1, pass 2) into a 3-stage swizzled ring
//   warp 1      MMA issuer, M=128 x N=128, K = head_dim, bf16 in, fp32
//               accumulate in TMEM (four accumulator stages, all 512 columns).
//               Pass 1 computes Q K^T (rows on TMEM lanes), pass 2 K Q^T
//               (keys on TMEM lanes) from the same shared-memory operands.
//   warp 2      TMEM allocator
//   warps 4-19  epilogue in two sets of 8, set p reading the tiles it = p
//               (mod 2) from accumulator stages p, p + 2; tcgen05.ld 32
//               columns at a time; 112 registers each (setmaxnreg):
//               pass 1: thread = window row -> running max / sum (serial);
//               pass 2: thread = key -> column mass and below-threshold
//               counts, serial over the block's rows, so neither pass needs a
//               cross-lane reduction per entry.
// The score matrix never leaves the SM: TMEM -> registers -> statistics.
#include <cuda.h>

#include "vlc_common.cuh"
#include "sm100.cuh"
#include "vlc_kernels.h"

#ifndef VLC_K1_PDL
#define VLC_K1_PDL 1   // launched under zero_outputs (programmatic dependent launch); waits before pass 2
#endif

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
#ifndef VLC_K1_SPLIT_TAIL
#define VLC_K1_SPLIT_TAIL 1
#endif
#ifndef VLC_K1_MINB
#define VLC_K1_MINB 1
#endif
constexpr int kStages = VLC_K1_STAGES;   // K tile ring
#ifndef VLC_K1_L2AHEAD
#define VLC_K1_L2AHEAD 0
#endif
constexpr int kL2Ahead = VLC_K1_L2AHEAD;   // key tiles prefetched into L2 beyond the ring
constexpr int kSub = VLC_K1_SUB;         // TMEM columns an epilogue thread holds at a time (16 / 32)
#ifndef VLC_K1_SETS
#define VLC_K1_SETS 2
#endif
constexpr int kSets = VLC_K1_SETS;          // epilogue warp sets taking tiles round robin
constexpr int kSetWarps = 8;                // 4 lane quarters x 2 column halves of 64
constexpr int kEpiWarps = kSets * kSetWarps;
constexpr int kCh = 64 / kSub;             // TMEM loads per warp and tile
constexpr int kThreads = 128 + kEpiWarps * 32;
#ifndef VLC_K1_ACC
#define VLC_K1_ACC (kSets == 2 ? 4 : kSets)
#endif
constexpr int kAcc = VLC_K1_ACC;           // accumulator stages (a multiple of kSets; set p owns stages = p mod kSets)
static_assert(kAcc % kSets == 0 && kAcc * 128 <= 512, "accumulator stages");
// registers: launch at 65536 / threads, then the control warpgroup drops to 32
// and the epilogue warpgroups take the rest (setmaxnreg)
constexpr int kRegLaunch = (65536 / ((128 + kEpiWarps * 32) * VLC_K1_MINB)) & ~7;
constexpr int kRegEpi = ((kRegLaunch * (128 + kEpiWarps * 32) - 128 * 32) / (kEpiWarps * 32)) & ~7;
constexpr uint32_t kTmemCols = kAcc * kN <= 256 ? 256u : 512u;   // tcgen05.alloc: a power of two

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
// split issue / wait: the next chunk's TMEM load runs under this chunk's math
template <int N>
VLC_DEV void tmem_issue(uint32_t taddr, uint32_t (&r)[N]) {
    if constexpr (N == 32) sm100::tmem_ld32_issue(taddr, r);
    else sm100::tmem_ld16_issue(taddr, r);
}
template <int N>
VLC_DEV void tmem_wait(uint32_t (&r)[N]) {
    if constexpr (N == 32) sm100::tmem_ld32_wait(r);
    else sm100::tmem_ld16_wait(r);
}
#ifndef VLC_K1_PIPE
#define VLC_K1_PIPE 0
#endif
constexpr bool kPipe = VLC_K1_PIPE;   // software-pipelined TMEM loads in the epilogue
#ifndef VLC_K1_PROBE
#define VLC_K1_PROBE 0   // timing probes (wrong results), bits: 1 = no epilogue math, 2 = no MMA, 4 = no TMA after the first ring, 8 = one TMEM load per tile, 16 = exact mode without its listing path
#endif

template <int D, bool EXACT>
__global__ void __launch_bounds__(kThreads, VLC_K1_MINB)
score_stats_tc(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
               ScoreArgs a, int nparts, int nblk, int n_full) {
    using LY = Layout<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // small state in static shared memory (plain LDS/STS, not generic accesses)
    __shared__ uint64_t full[kStages], empty[kStages], qfull[1], tfull[kAcc], tempty[kAcc];
    __shared__ uint32_t tmem_slot[1];
    __shared__ float2 rowstat[2 * kSets * kM];          // (max, sum) per (set, column half) and row
    // pass-2 row constants, packed per row pair {mbt_r, mbt_r+1, is_r, is_r+1}:
    //   mbt = row max * c1 + t2 (u' = l c1 - mbt = log2 e - t2, below <=> u' < 0)
    //   is  = 2^t2 / row sum   (mass = 2^u' * is = e / S)
    __shared__ __align__(16) float4 c_pk[kM / 2];
    __shared__ int c_lim[kM];                           // last visible key (-1: no row)
    __shared__ int hcnt[kM];                            // below counts per head of the block

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the fix-ups wait for completion
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // CTA -> (slot s, row block rb, key part).  The first n_full CTAs take whole
    // units; the rest -- the units of the last, partial wave -- come in pairs
    // that both run pass 1 (the row statistics need every key) and split pass
    // 2's key tiles, so the tail wave takes about 0.7 of a unit instead of 1.
    const int bid = blockIdx.x;
    const int u = bid < n_full ? bid : n_full + (bid - n_full) / 2;
    const int part = bid < n_full ? -1 : (bid - n_full) & 1;     // -1: whole unit
    const int s = u / nblk, rb = u % nblk;
    const int64_t R = (int64_t)a.G * a.w;
    const int64_t r_first = (int64_t)rb * kM;
    const int64_t r_last = imin(R, r_first + kM) - 1;
    const int64_t i_max = (r_last / a.w == r_first / a.w) ? r_last % a.w : a.w - 1;
    const int64_t blk_end = imin(a.n, a.q_base + i_max + 1);   // keys any row here can see
    const int T = (int)((blk_end + kN - 1) / kN);
    const int P1 = a.stat_max ? 0 : T;    // pass-1 tiles (none when the row statistics are given)
    const int tlo = part == 1 ? (T + 1) / 2 : 0, thi = part == 0 ? (T + 1) / 2 : T;   // pass-2 key tiles
    const int iters = P1 + (thi - tlo);
    const int64_t head0 = r_first / a.w;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) { sm100::mbar_init(full + i, 1); sm100::mbar_init(empty + i, 1); }
        sm100::mbar_init(qfull, 1);
        for (int i = 0; i < kAcc; ++i) { sm100::mbar_init(tfull + i, 1); sm100::mbar_init(tempty + i, kSetWarps); }
        sm100::fence_barrier_init();
        sm100::fence_proxy_async();
    }
    if (threadIdx.x < kM) hcnt[threadIdx.x] = 0;
    if (warp == 2) sm100::tmem_alloc(tmem_slot, kTmemCols);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // registers: the control warpgroup (warps 0-3) gives its share to the four
    // epilogue warpgroups (launch 96 x 640 = 32 x 128 + 112 x 512)
    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 32;\n");
        if (warp == 0 && lane == 0) {
            // ------------------------------------------------ TMA producer
            sm100::tma_prefetch(&qmap);
            sm100::tma_prefetch(&kmap);
            sm100::mbar_expect_tx(qfull, LY::kQBytes);
            for (int kb = 0; kb < LY::KB; ++kb)
                sm100::tma_load_2d(smem + kb * LY::kQRegion, &qmap, qfull, kb * 64, (int)(s * R + r_first));
            // pull the first pass's key tiles into L2 ahead of their loads (the
            // ring holds only kStages tiles; the rest of the L2 latency is hidden)
            auto l2_prefetch = [&](int t) {
                for (int kb = 0; kb < LY::KB; ++kb)
                    sm100::tma_prefetch_2d(&kmap, kb * 64, (int)(s * a.T + (int64_t)t * kN));
            };
            const int pf_first = P1 > 0 ? P1 : iters;   // tiles of the first pass over the keys
            for (int t = kStages; t < kStages + kL2Ahead && t < pf_first; ++t) l2_prefetch(t);
            for (int it = 0; it < iters; ++it) {
                const int st = it % kStages;
                const uint32_t ph = (it / kStages) & 1;
                const int t = it < P1 ? it : tlo + (it - P1);
                if ((VLC_K1_PROBE & 4) && it >= kStages) break;
                if (kL2Ahead > 0 && it + kStages + kL2Ahead < pf_first) l2_prefetch(it + kStages + kL2Ahead);
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
                const int acc = it % kAcc;
                const uint32_t aph = (it / kAcc) & 1;
                sm100::mbar_wait(tempty + acc, aph ^ 1);
                if (!((VLC_K1_PROBE & 4) && it >= kStages)) sm100::mbar_wait(full + st, ph);
                sm100::tc_fence_after();
                const uint32_t k_addr = sm100::smem_u32(smem + LY::kQBytes + st * LY::kKBytes);
                const bool rows_on_lanes = it < P1;
#pragma unroll
                for (int kb = 0; kb < LY::KB; ++kb) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {   // 4 x 16 elements = one 128 B swizzle row
                        const uint64_t qd = sm100::sdesc_k_sw128(q_addr + kb * LY::kQRegion + kk * 32);
                        const uint64_t kd = sm100::sdesc_k_sw128(k_addr + kb * LY::kKRegion + kk * 32);
                        if (!(VLC_K1_PROBE & 2))   // timing probe: no MMA
                        sm100::mma_bf16(tmem + acc * kN, rows_on_lanes ? qd : kd, rows_on_lanes ? kd : qd, idesc,
                                        (kb | kk) != 0);
                    }
                }
                sm100::mma_commit(empty + st);   // K stage reusable once these MMAs retire
                sm100::mma_commit(tfull + acc);  // accumulator ready for the epilogue
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegEpi));
        // ------------------------------------------------ epilogue
        // Two warp sets, set p taking tiles it = p (mod 2) from accumulator stages
        // p and p + 2, so one set's TMEM-load latency overlaps the other's math and
        // the MMA runs a tile ahead of each set.  Within a set,
        // warp -> (TMEM lane quarter `sub`, 64-column half `half`).
        const int ew = warp - 4, sub = warp & 3, set = ew >> 3, half = (ew >> 2) & 1;   // 8 warps per set
        const int lane_idx = 32 * sub + lane;                  // TMEM lane of this thread
        const uint32_t lane_addr = tmem + (uint32_t(32 * sub) << 16) + half * 64;
        const float c1 = a.inv_scale * kLog2e;
        float l[kSub];

        // ---- pass 1 (thread = window row): running max of raw dots, rescaled sum
        {
            const int64_t r = r_first + lane_idx;
            const bool row_ok = r < R;
            const int64_t i = row_ok ? r % a.w : 0;
            const int row_end32 = row_ok ? (int)imin(a.n, a.q_base + i + 1) : 0;
            float m = -INFINITY, sum = 0.f;
            for (int it = set; it < P1; it += kSets) {
                const int acc = it % kAcc;
                sm100::mbar_wait(tfull + acc, (it / kAcc) & 1);
                sm100::tc_fence_after();
                uint32_t rbuf[2][kSub];
                if (kPipe) tmem_issue(lane_addr + acc * kN, rbuf[0]);
#pragma unroll
                for (int h = 0; h < kCh; ++h) {
                if (kPipe) {
                    tmem_wait(rbuf[h & 1]);
                    if (h + 1 < kCh) tmem_issue(lane_addr + acc * kN + (h + 1) * kSub, rbuf[(h + 1) & 1]);
#pragma unroll
                    for (int i = 0; i < kSub; ++i) l[i] = __uint_as_float(rbuf[h & 1][i]);
                } else {
                    if (!((VLC_K1_PROBE & 8) && h > 0)) tmem_ld(lane_addr + acc * kN + h * kSub, l);   // probe 8: one load per tile
                }
                if (h == kCh - 1) {
                    sm100::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) sm100::mbar_arrive(tempty + acc);   // registers hold the tile now
                }
                if (VLC_K1_PROBE & 1) { sum += l[0]; continue; }   // timing probe: no epilogue math
                const int valid = max(0, min(kSub, row_end32 - (it * kN + half * 64 + h * kSub)));
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
                // four add chains (row k -> chain k & 3) as two packed pairs:
                // FFMA2 for the exponent arguments, FADD2 for the sums
                float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
                const float2 c1v = make_float2(c1, c1), nmb = make_float2(-mb, -mb);
                if (full_chunk) {
#pragma unroll
                    for (int k = 0; k < kSub; k += 4) {
                        const float2 u0 = __ffma2_rn(make_float2(l[k], l[k + 1]), c1v, nmb);
                        const float2 u1 = __ffma2_rn(make_float2(l[k + 2], l[k + 3]), c1v, nmb);
#ifdef VLC_K1_NOEX2_TEST
                        s01 = __fadd2_rn(s01, __ffma2_rn(u0, make_float2(0.01f, 0.01f), make_float2(1.f, 1.f)));
                        s23 = __fadd2_rn(s23, __ffma2_rn(u1, make_float2(0.01f, 0.01f), make_float2(1.f, 1.f)));
#else
                        s01 = __fadd2_rn(s01, make_float2(ex2(u0.x), ex2(u0.y)));
                        s23 = __fadd2_rn(s23, make_float2(ex2(u1.x), ex2(u1.y)));
#endif
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < kSub; k += 4) {
                        const float2 u0 = __ffma2_rn(make_float2(l[k], l[k + 1]), c1v, nmb);
                        const float2 u1 = __ffma2_rn(make_float2(l[k + 2], l[k + 3]), c1v, nmb);
                        s01 = __fadd2_rn(s01, make_float2(k < valid ? ex2(u0.x) : 0.f, k + 1 < valid ? ex2(u0.y) : 0.f));
                        s23 = __fadd2_rn(s23, make_float2(k + 2 < valid ? ex2(u1.x) : 0.f, k + 3 < valid ? ex2(u1.y) : 0.f));
                    }
                }
                sum += (s01.x + s01.y) + (s23.x + s23.y);
                }
            }
            rowstat[(set * 2 + half) * kM + lane_idx] = make_float2(m, sum);
            sm100::named_bar_sync(1, kEpiWarps * 32);
            if (ew < 4) {
                float M = -INFINITY, S = 0.f, mb, rm;
                if (a.stat_max) {   // given (logit units): mb = max * log2e
                    const int64_t gi = ((int64_t)s * a.G + r / a.w) * a.stat_ld + a.stat_row0 + i;
                    rm = row_ok ? a.stat_max[gi] : 0.f;
                    S = row_ok ? a.stat_sum[gi] : 1.f;
                    mb = rm * kLog2e;
                } else {
#pragma unroll
                    for (int g4 = 0; g4 < 2 * kSets; ++g4) M = fmaxf(M, rowstat[g4 * kM + lane_idx].x);
#pragma unroll
                    for (int g4 = 0; g4 < 2 * kSets; ++g4) {
                        const float2 h = rowstat[g4 * kM + lane_idx];
                        if (h.x != -INFINITY) S += h.y * ex2((h.x - M) * c1);
                    }
                    mb = M * c1;
                    rm = M * a.inv_scale;
                }
                float* pk = reinterpret_cast<float*>(c_pk) + (lane_idx >> 1) * 4 + (lane_idx & 1);
                const float t2c = a.t_star * kLog2e;
                if (row_ok) {
                    a.row_max[(int64_t)s * R + r] = rm;
                    a.row_sum[(int64_t)s * R + r] = S;
                    pk[0] = mb + t2c;
                    pk[2] = ex2(t2c) / S;
                    c_lim[lane_idx] = (int)(a.q_base + i);
                } else {
                    pk[0] = INFINITY;   // u' = -inf: no mass
                    pk[2] = 0.f;
                    c_lim[lane_idx] = -1;         // sees no key (and is never counted)
                }
            }
            sm100::named_bar_sync(1, kEpiWarps * 32);
        }

        // ---- pass 2 (thread = key): column mass and below-threshold counts over
        //   the 64 rows of this half.  u = l*c1 - mb_r ~ log2(exp(logit - max));
        //   below <=> u < t* log2e; mass = 2^(u - log2 S_r).  Serial per key: no
        //   cross-lane reduction, and every key column follows the same order.
        //   Each half writes its own partial row of col_partial (no barrier).
        // the counters this pass accumulates into were zeroed by zero_outputs, the
        // programmatic predecessor: everything before this point overlapped it
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const int r0 = half * 64;
        const int64_t rg = r_first + r0;
        const bool one_head = rg / a.w == (rg + 63) / a.w;
        float* colp = a.col_partial + ((int64_t)s * nparts + rb * 2 + half) * a.n;
        for (int it = P1 + (set - P1 % kSets + kSets) % kSets; it < iters; it += kSets) {
            const int t = tlo + (it - P1);
            const int j = t * kN + lane_idx;                     // this thread's key
            const bool all_visible = (int64_t)t * kN + kN - 1 <= a.q_base;   // CTA-uniform
            const int acc = it % kAcc;
            sm100::mbar_wait(tfull + acc, (it / kAcc) & 1);
            sm100::tc_fence_after();
            // exact mode: an entry whose decision u' < 0 is within `band` of flipping
            // (fp32 logits vs the reference's float64 dots) is not counted here but
            // listed for a float64 re-decision.  band = 0: plain decisions.
            const float band = EXACT ? a.band : 0.f;
            float2 cs01 = make_float2(0.f, 0.f), cs23 = make_float2(0.f, 0.f);   // mass: row k -> chain k & 3
            int cnt = 0;
            uint32_t rbuf[2][kSub];
            if (kPipe) tmem_issue(lane_addr + acc * kN, rbuf[0]);
#pragma unroll
            for (int h = 0; h < kCh; ++h) {
            const int rh = r0 + h * kSub;                        // first row of this chunk
            if (kPipe) {
                tmem_wait(rbuf[h & 1]);
                if (h + 1 < kCh) tmem_issue(lane_addr + acc * kN + (h + 1) * kSub, rbuf[(h + 1) & 1]);
#pragma unroll
                for (int i = 0; i < kSub; ++i) l[i] = __uint_as_float(rbuf[h & 1][i]);
            } else {
                if (!((VLC_K1_PROBE & 8) && h > 0)) tmem_ld(lane_addr + acc * kN + h * kSub, l);
            }
            if (h == kCh - 1) {
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(tempty + acc);
            }
            if (VLC_K1_PROBE & 1) { cs01.x += l[0]; continue; }   // timing probe: no epilogue math
            // per entry: u' = l c1 - mbt_r (log2 of e_r / p-threshold), below <=> u' < 0,
            // mass += 2^u' * is_r -- packed pairs of rows: one FFMA2, two MUFU, one
            // FFMA2, two FSET + one FADD2 for the count, one FMNMX3 for the band test.
            // The same operation order in every branch, so identical key columns
            // give bit-identical mass (the reference's tie rule needs that).
            const float4* pk4 = c_pk + (rh >> 1);
            float minabs = INFINITY;                          // min |u'| over the chunk (band test)
            float2 cf = make_float2(0.f, 0.f);                // certain-below count
            const float2 c1v = make_float2(c1, c1);
            const bool all_rows = r_first + rh + kSub - 1 < R;
            if (all_visible && all_rows) {   // every row real and every key visible
#pragma unroll
                for (int q2 = 0; q2 < kSub / 2; ++q2) {
                    const float4 c = pk4[q2];
                    const float2 u = __ffma2_rn(make_float2(l[2 * q2], l[2 * q2 + 1]), c1v, make_float2(-c.x, -c.y));
                    cf = __fadd2_rn(cf, make_float2(u.x < -band ? 1.f : 0.f, u.y < -band ? 1.f : 0.f));
                    if (EXACT) minabs = fminf(minabs, fminf(fabsf(u.x), fabsf(u.y)));
#ifdef VLC_K1_NOEX2_TEST   // timing probe only: is K1 bound by the SFU?
                    const float2 e = __ffma2_rn(u, make_float2(0.01f, 0.01f), make_float2(1.f, 1.f));
#else
                    const float2 e = make_float2(ex2(u.x), ex2(u.y));
#endif
                    if (q2 & 1) cs23 = __ffma2_rn(e, make_float2(c.z, c.w), cs23);
                    else cs01 = __ffma2_rn(e, make_float2(c.z, c.w), cs01);
                }
            } else {
#pragma unroll
                for (int q2 = 0; q2 < kSub / 2; ++q2) {
                    const float4 c = pk4[q2];
                    const bool v0 = j <= c_lim[rh + 2 * q2], v1 = j <= c_lim[rh + 2 * q2 + 1];
                    const float2 u = __ffma2_rn(make_float2(l[2 * q2], l[2 * q2 + 1]), c1v, make_float2(-c.x, -c.y));
                    cf = __fadd2_rn(cf, make_float2((v0 && u.x < -band) ? 1.f : 0.f, (v1 && u.y < -band) ? 1.f : 0.f));
                    if (EXACT) minabs = fminf(minabs, fminf(v0 ? fabsf(u.x) : INFINITY, v1 ? fabsf(u.y) : INFINITY));
                    const float2 e = make_float2(v0 ? ex2(u.x) : 0.f, v1 ? ex2(u.y) : 0.f);
                    if (q2 & 1) cs23 = __ffma2_rn(e, make_float2(c.z, c.w), cs23);
                    else cs01 = __ffma2_rn(e, make_float2(c.z, c.w), cs01);
                }
            }
            float cntf = cf.x + cf.y;
            // exact mode: a lane whose chunk holds an entry within `band` of its
            // decision lists the whole chunk (key j x these kSub rows) in one record
            // and counts none of it here; the fix-up re-decides all of its entries
            // from float64 dots.  No per-entry work on this path: l[] is dead here.
            bool listed = false;
            if (EXACT && !(VLC_K1_PROBE & 16) && __any_sync(kFull, minabs < band)) {
                if (j < a.n && minabs < band) {
                    const int at = atomicAdd(a.fix_counts + 1, 1);
                    if (at < a.cap) {
                        // .w: the chunk's smallest |u| from the tensor-core logits (log2
                        // units), which the fix-up compares with the exact one
                        a.flag[at] = make_int4(s, (int)(r_first + rh), j, __float_as_int(minabs));
                        listed = true;
                        cntf = 0.f;
                    } else {   // list full: the chunk's in-band entries stay undecided
                        atomicAdd(a.fix_counts + 2, 1);   // (reported: check() raises ExactnessError)
                    }
                }
            }
            cnt += (int)cntf;
            if (!one_head) {
#pragma unroll
                for (int k = 0; k < kSub; ++k) {
                    const float u = fmaf(l[k], c1, -(reinterpret_cast<const float*>(pk4 + (k >> 1))[k & 1]));
                    const int tot = __reduce_add_sync(kFull, (!listed && j <= c_lim[rh + k] && u < -band) ? 1 : 0);
                    if (lane == 0 && tot) atomicAdd(hcnt + (int)((r_first + rh + k) / a.w - head0), tot);
                }
            }
            }
            if (j < a.n) colp[j] = (cs01.x + cs01.y) + (cs23.x + cs23.y);
            if (a.below_col && cnt && j < a.n) atomicAdd(a.below_col + (int64_t)s * a.n + j, cnt);
            // per-head totals (warp reduce, one shared atomic per warp)
            if (one_head) {   // (mixed-head halves were counted row by row above)
                const int tot = __reduce_add_sync(kFull, cnt);
                if (lane == 0 && tot) atomicAdd(hcnt + (int)(rg / a.w - head0), tot);
            }
        }
        // columns no row of this block can see
        if (set == 0 && thi == T)
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
    const int nblk = nparts / 2, units = nblk * a.slots;
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int tail = units % n_sm;
    const int n_full = (VLC_K1_SPLIT_TAIL && tail > 0 && 2 * tail <= n_sm) ? units - tail : units;
    e = VLC_K1_PDL ? launch_pdl(score_stats_tc<D, EXACT>, dim3(n_full + 2 * (units - n_full)), dim3(kThreads), sm, st,
                                qmap, kmap, a, nparts, nblk, n_full)
                   : (score_stats_tc<D, EXACT><<<n_full + 2 * (units - n_full), kThreads, sm, st>>>(
                          qmap, kmap, a, nparts, nblk, n_full), cudaSuccess);
    return e != cudaSuccess ? e : cudaGetLastError();
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
