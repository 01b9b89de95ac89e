// prefill.cu -- f2: causal prefill attention over the prompt on tcgen05, with
// the per-row softmax statistics (row max, row sum) as a by-product.
//
// reference: bench.py:196-234 (_prefill_layer: causal softmax(Q K^T / sqrt(d)) V
// over the m prompt rows of every head, float32) -- the step before the
// compression path; PAPER.md:528-553 (the post-vision statistics ride on the
// prefill's Q K^T).
//
// One pass per CTA = (query head, block of 128 prompt rows), online softmax:
// per 128-key tile, S = Q K^T lands in TMEM; the epilogue (thread = row, four
// warps per row sharing the tile's columns) takes the tile's row max through
// shared memory, forms P = 2^(S c1 - m_ref c1) as bf16 into tensor memory
// (tcgen05.st) and the MMA warp accumulates O += P V in TMEM with A = P from
// TMEM and B = V^T tiles (pre-transposed once, K-major) from shared memory.
// m_ref, the reference max, is raised only when the row max grows by more
// than 2^8; then O's row (tcgen05.ld / scale / tcgen05.st, after the previous
// P V retired) and the running sum are rescaled.  O / sum at the end; the row
// statistics emitted are the exact row max and the sum relative to it.
// VLC_PF_ONEPASS=0 builds the two-pass variant (max-only pass, then P with the
// final max: a second Q K^T per tile, no rescaling).
// Warps: 0 K producer, 1 MMA issuer, 2 TMEM allocator, 3 V^T producer,
// 4-19 epilogue (lane quarter x 32-column group).
#include <cuda.h>

#include "sm100.cuh"
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kM = 128;          // rows per CTA
constexpr int kN = 128;          // keys per tile
constexpr int kEpiWarps = 16;
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr uint32_t kTmemCols = 512;   // S: 2 x 128, O: d <= 128, P (TS mode): 2 x 64
#ifndef VLC_PF_TS
#define VLC_PF_TS 1
#endif
constexpr bool kTS = VLC_PF_TS;       // P through TMEM (A operand from tensor memory) instead of smem
constexpr int kKS = 2;
#ifndef VLC_PF_ONEPASS
#define VLC_PF_ONEPASS 1
#endif
constexpr bool kOnePass = VLC_PF_ONEPASS;   // online softmax with lazy O rescaling (one Q K^T per tile)
constexpr int kPasses = kOnePass ? 1 : 2;
#ifndef VLC_PF_S3
#define VLC_PF_S3 1
#endif
// one pass through TMEM: three S stages with P written over its own S stage
// (the lane quarter's max exchange already orders every S load before the P
// store), the stage freed by the P V MMA; S runs two tiles ahead of the epilogue
constexpr bool kS3 = kOnePass && kTS && VLC_PF_S3;
constexpr int kSSt = kS3 ? 3 : 2;                 // K tile ring (a third stage measured no faster)

template <int D>
struct PL {
    static constexpr int KB = D / 64;
    static constexpr uint32_t kQ = KB * kM * 128;        // Q block
    static constexpr uint32_t kK = KB * kN * 128;        // one K tile
    static constexpr uint32_t kV = 2 * D * 128;          // one V^T tile: D rows x 128 keys
    static constexpr uint32_t kP = 2 * kM * 128;         // P: 128 rows x 128 keys
    static constexpr uint32_t kPArea = kTS ? 4 * kM * 8 : 2 * kP;     // TS: pass 1's row statistics only
    static constexpr uint32_t kBytes = kQ + kKS * kK + 2 * kV + kPArea + 1024;
};

VLC_DEV uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// byte offset of 16-byte chunk c (8 bf16) of row r in a 128B-swizzled tile of
// `rows` rows (64-element boxes, `rows` x 128 B each) -- the TMA / UMMA layout
[[maybe_unused]] VLC_DEV uint32_t swz(int rows, int r, int c) {
    return (uint32_t)((c >> 3) * rows * 128 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
prefill_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
               const __grid_constant__ CUtensorMap vmap, PrefillArgs a) {
    using LY = PL<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sq = smem;
    uint8_t* sk = sq + LY::kQ;
    uint8_t* sv = sk + kKS * LY::kK;
    uint8_t* sp = sv + 2 * LY::kV;
    __shared__ uint64_t qfull, kfull[kKS], kempty[kKS], vfull[2], vempty[2], tfull[kSSt], tempty[kSSt], pfull[kSSt], pempty[2],
        ofull;
    __shared__ uint32_t tmem_slot;
    [[maybe_unused]] __shared__ float c_mb[kM];
    __shared__ float c_part[4 * kM];
    [[maybe_unused]] __shared__ float xmax[kOnePass ? 2 : 1][4][kM];      // one-pass: tile row max per column group
    [[maybe_unused]] float2* rowstat = reinterpret_cast<float2*>(sp);   // [4 * kM], pass 1 only (P is pass 2 only)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sq_slot = blockIdx.x;                                  // (b, l, query head)
    const int rb = gridDim.y - 1 - blockIdx.y;                       // longest blocks first, over all slots
    const int64_t kv_slot = (int64_t)(sq_slot / a.Hq) * a.Hkv + (sq_slot % a.Hq) / (a.Hq / a.Hkv);
    const int64_t r0 = (int64_t)rb * kM;
    const int64_t key_end = imin(a.m, r0 + kM);                      // keys any row here sees
    const int T = (int)((key_end + kN - 1) / kN);

    if (threadIdx.x == 0) {
        sm100::mbar_init(&qfull, 1);
        for (int i = 0; i < kKS; ++i) { sm100::mbar_init(kfull + i, 1); sm100::mbar_init(kempty + i, 1); }
        for (int i = 0; i < 2; ++i) { sm100::mbar_init(vfull + i, 1); sm100::mbar_init(vempty + i, 1); }
        for (int i = 0; i < kSSt; ++i) {   // kS3: the S stage is freed by the P V MMA (one commit)
            sm100::mbar_init(tfull + i, 1); sm100::mbar_init(tempty + i, kS3 ? 1 : kEpiWarps);
            sm100::mbar_init(pfull + i, kEpiWarps);
        }
        for (int i = 0; i < 2; ++i) sm100::mbar_init(pempty + i, 1);
        sm100::mbar_init(&ofull, 1);
        sm100::fence_barrier_init();
    }
    if (warp == 2) sm100::tmem_alloc(&tmem_slot, kTmemCols);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t tmem_o = tmem + (kS3 ? 3 : 2) * kN;
    const uint32_t tmem_p = tmem + 3 * kN;                            // TS mode: P stages, 64 columns each

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 32;\n");
        if (warp == 0 && lane == 0) {
            // ---- Q once, then the K tiles twice (pass 1, pass 2)
            sm100::tma_prefetch(&qmap);
            sm100::tma_prefetch(&kmap);
            sm100::mbar_expect_tx(&qfull, LY::kQ);
            for (int kb = 0; kb < LY::KB; ++kb)
                sm100::tma_load_2d(sq + kb * kM * 128, &qmap, &qfull, kb * 64, (int)(sq_slot * a.q_rows + r0));
            for (int it = 0; it < kPasses * T; ++it) {
                const int st = it % kKS, t = it < T ? it : it - T;
                sm100::mbar_wait(kempty + st, ((it / kKS) & 1) ^ 1);
                sm100::mbar_expect_tx(kfull + st, LY::kK);
                for (int kb = 0; kb < LY::KB; ++kb)
                    sm100::tma_load_2d(sk + st * LY::kK + kb * kN * 128, &kmap, kfull + st, kb * 64,
                                       (int)(kv_slot * a.kv_rows + (int64_t)t * kN));
            }
        } else if (warp == 3 && lane == 0) {
            // ---- V^T tiles (pass 2): D rows (dims) x 128 keys
            sm100::tma_prefetch(&vmap);
            for (int t = 0; t < T; ++t) {
                const int st = t & 1;
                sm100::mbar_wait(vempty + st, ((t >> 1) & 1) ^ 1);
                sm100::mbar_expect_tx(vfull + st, LY::kV);
                for (int kb = 0; kb < 2; ++kb)
                    sm100::tma_load_2d(sv + st * LY::kV + kb * D * 128, &vmap, vfull + st, t * kN + kb * 64,
                                       (int)(kv_slot * D));
            }
        } else if (warp == 1 && lane == 0) {
            // ---- MMA issuer
            constexpr uint32_t idesc_s = sm100::idesc_bf16_f32(kM, kN);
            constexpr uint32_t idesc_o = sm100::idesc_bf16_f32(kM, D);
            const uint32_t q_addr = sm100::smem_u32(sq), p_addr = sm100::smem_u32(sp);
            auto qk = [&](int it) {   // S[it & 1] = Q K^T of the K tile in ring stage it & 1
                const int st = it & 1, ks = it % kKS;
                sm100::mbar_wait(tempty + st, ((it >> 1) & 1) ^ 1);
                sm100::mbar_wait(kfull + ks, (it / kKS) & 1);
                sm100::tc_fence_after();
                const uint32_t k_addr = sm100::smem_u32(sk + ks * LY::kK);
#pragma unroll
                for (int kb = 0; kb < LY::KB; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        sm100::mma_bf16(tmem + st * kN, sm100::sdesc_k_sw128(q_addr + kb * kM * 128 + kk * 32),
                                        sm100::sdesc_k_sw128(k_addr + kb * kN * 128 + kk * 32), idesc_s,
                                        (kb | kk) != 0);
                sm100::mma_commit(kempty + ks);
                sm100::mma_commit(tfull + st);
            };
            auto pv = [&](int t) {    // O += P V for key tile t (P buffer and V^T stage t & 1)
                const int st = t & 1;
                sm100::mbar_wait(pfull + st, (t >> 1) & 1);
                sm100::mbar_wait(vfull + st, (t >> 1) & 1);
                sm100::tc_fence_after();
                const uint32_t v_addr = sm100::smem_u32(sv + st * LY::kV);
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t bd = sm100::sdesc_k_sw128(v_addr + kb * D * 128 + kk * 32);
                        if constexpr (kTS)   // 16 keys = 8 packed columns per instruction
                            sm100::mma_bf16_ts(tmem_o, tmem_p + st * 64 + (kb * 4 + kk) * 8, bd, idesc_o,
                                               (t | kb | kk) != 0);
                        else
                            sm100::mma_bf16(tmem_o, sm100::sdesc_k_sw128(p_addr + st * LY::kP + kb * kM * 128 + kk * 32),
                                            bd, idesc_o, (t | kb | kk) != 0);
                    }
                sm100::mma_commit(pempty + st);
                sm100::mma_commit(vempty + st);
            };
            sm100::mbar_wait(&qfull, 0);
            if constexpr (kS3) {
                auto qk3 = [&](int t) {   // S stage t % 3, free once P V of tile t - 3 retired
                    const int st = t % 3, ks = t % kKS;
                    sm100::mbar_wait(tempty + st, ((t / 3) & 1) ^ 1);
                    sm100::mbar_wait(kfull + ks, (t / kKS) & 1);
                    sm100::tc_fence_after();
                    const uint32_t k_addr = sm100::smem_u32(sk + ks * LY::kK);
#pragma unroll
                    for (int kb = 0; kb < LY::KB; ++kb)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            sm100::mma_bf16(tmem + st * kN, sm100::sdesc_k_sw128(q_addr + kb * kM * 128 + kk * 32),
                                            sm100::sdesc_k_sw128(k_addr + kb * kN * 128 + kk * 32), idesc_s,
                                            (kb | kk) != 0);
                    sm100::mma_commit(kempty + ks);
                    sm100::mma_commit(tfull + st);
                };
                auto pv3 = [&](int t) {   // O += P V, P packed over the first 64 columns of S stage t % 3
                    const int st = t % 3, vs = t & 1;
                    sm100::mbar_wait(pfull + st, (t / 3) & 1);
                    sm100::mbar_wait(vfull + vs, (t >> 1) & 1);
                    sm100::tc_fence_after();
                    const uint32_t v_addr = sm100::smem_u32(sv + vs * LY::kV);
#pragma unroll
                    for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            sm100::mma_bf16_ts(tmem_o, tmem + st * kN + (kb * 4 + kk) * 8,
                                               sm100::sdesc_k_sw128(v_addr + kb * D * 128 + kk * 32), idesc_o,
                                               (t | kb | kk) != 0);
                    sm100::mma_commit(vempty + vs);
                    sm100::mma_commit(tempty + st);
                };
                qk3(0);
                if (T > 1) qk3(1);
                for (int t = 0; t < T; ++t) {
                    pv3(t);
                    if (t + 2 < T) qk3(t + 2);
                }
                sm100::mma_commit(&ofull);
            } else {
            const int p1 = kOnePass ? 0 : T;
            for (int it = 0; it < p1; ++it) qk(it);
            for (int t = 0; t < T; ++t) {
                qk(p1 + t);
                if (t > 0) pv(t - 1);
            }
            pv(T - 1);
            sm100::mma_commit(&ofull);
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 112;\n");
        // ---- epilogue: warp -> (TMEM lane quarter `sub`, 32-column group `cg`)
        const int ew = warp - 4, sub = warp & 3, cg = ew >> 2;
        const int li = 32 * sub + lane;                               // row within the block
        const int64_t r = r0 + li;
        const bool row_ok = r < a.m;
        const int64_t row_end = row_ok ? r + 1 : 0;                   // causal: keys [0, r]
        const uint32_t lane_addr = tmem + (uint32_t(32 * sub) << 16) + cg * 32;
        const float c1 = a.inv_scale * kLog2e;
        float l[32];

        float S, il, row_M;
        if constexpr (kOnePass) {
            // one pass: per tile, the row max across the four column groups of the
            // lane quarter; P uses a reference max m_ref that is only raised when
            // the row max grows by more than 2^8 (then O and the sum are rescaled)
            const float grow_raw = 8.f / c1;
            float m_ref = -INFINITY, m_true = -INFINITY;
            float ps[4] = {0.f, 0.f, 0.f, 0.f};
            for (int t = 0; t < T; ++t) {
                const int st = kS3 ? t % 3 : t & 1, pb = t & 1;
                sm100::mbar_wait(tfull + st, (kS3 ? t / 3 : t >> 1) & 1);
                sm100::tc_fence_after();
                sm100::tmem_ld32(lane_addr + st * kN, l);
                sm100::tc_fence_before();
                __syncwarp();
                if (!kS3 && lane == 0) sm100::mbar_arrive(tempty + st);
                const int valid = (int)imax(0, imin(32, row_end - ((int64_t)t * kN + cg * 32)));
                const bool full = __all_sync(kFull, valid == 32);
                float cm = -INFINITY;
                if (full) {
#pragma unroll
                    for (int k = 0; k < 32; ++k) cm = fmaxf(cm, l[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < 32; ++k) cm = k < valid ? fmaxf(cm, l[k]) : cm;
                }
                xmax[t & 1][cg][li] = cm;
                sm100::named_bar_sync(2 + sub, 128);                  // the lane quarter's 4 warps
                const float tm = fmaxf(fmaxf(xmax[t & 1][0][li], xmax[t & 1][1][li]),
                                       fmaxf(xmax[t & 1][2][li], xmax[t & 1][3][li]));
                m_true = fmaxf(m_true, tm);
                const bool grow = tm > m_ref + grow_raw;
                if (!kS3) sm100::mbar_wait(pempty + pb, ((t >> 1) & 1) ^ 1);   // P V of tile t - 2 has read P[pb]
                if (__any_sync(kFull, grow)) {
                    const float sc = (grow && m_ref != -INFINITY) ? ex2((m_ref - tm) * c1) : 1.f;
                    if (t > 0 && cg * 32 < D) {
                        // O holds the tiles before t once P V of tile t - 1 has retired
                        if constexpr (kS3) sm100::mbar_wait(tempty + (t - 1) % 3, ((t - 1) / 3) & 1);
                        else sm100::mbar_wait(pempty + (pb ^ 1), ((t - 1) >> 1) & 1);
                        sm100::tc_fence_after();
                        float o[32];
                        const uint32_t oa = tmem_o + (uint32_t(32 * sub) << 16) + cg * 32;
                        sm100::tmem_ld32(oa, o);
#pragma unroll
                        for (int k = 0; k < 32; ++k) o[k] *= sc;
                        sm100::tmem_st32(oa, o);
                    }
                    if (grow) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) ps[k] *= sc;
                        m_ref = tm;
                    }
                }
                const float mb = m_ref * c1;
                uint32_t pk[16];
                if (full) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float p0 = ex2(fmaf(l[2 * k], c1, -mb)), p1 = ex2(fmaf(l[2 * k + 1], c1, -mb));
                        ps[(2 * k) & 3] += p0;
                        ps[(2 * k + 1) & 3] += p1;
                        pk[k] = pack_bf16(p0, p1);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float p0 = 2 * k < valid ? ex2(fmaf(l[2 * k], c1, -mb)) : 0.f;
                        const float p1 = 2 * k + 1 < valid ? ex2(fmaf(l[2 * k + 1], c1, -mb)) : 0.f;
                        ps[(2 * k) & 3] += p0;
                        ps[(2 * k + 1) & 3] += p1;
                        pk[k] = pack_bf16(p0, p1);
                    }
                }
                sm100::tc_fence_after();
                if constexpr (kS3)   // over this tile's own S stage (all of its S loads are done)
                    sm100::tmem_st16(tmem + (uint32_t(32 * sub) << 16) + st * kN + cg * 16, pk);
                else
                    sm100::tmem_st16(tmem_p + (uint32_t(32 * sub) << 16) + pb * 64 + cg * 16, pk);
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(pfull + (kS3 ? st : pb));
            }
            c_part[cg * kM + li] = (ps[0] + ps[1]) + (ps[2] + ps[3]);
            sm100::named_bar_sync(1, kEpiWarps * 32);
            const float l_ref = (c_part[li] + c_part[kM + li]) + (c_part[2 * kM + li] + c_part[3 * kM + li]);
            il = row_ok ? 1.f / l_ref : 0.f;
            S = l_ref * ex2((m_ref - m_true) * c1);                  // the sum relative to the true max
            row_M = m_true;
        } else {
            // pass 1: row max of the raw dots only (no exponentials)
            float m = -INFINITY;
            for (int it = 0; it < T; ++it) {
                const int st = it & 1;
                sm100::mbar_wait(tfull + st, (it >> 1) & 1);
                sm100::tc_fence_after();
                sm100::tmem_ld32(lane_addr + st * kN, l);
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(tempty + st);
                const int valid = (int)imax(0, imin(32, row_end - ((int64_t)it * kN + cg * 32)));
                if (__all_sync(kFull, valid == 32)) {
    #pragma unroll
                    for (int k = 0; k < 32; ++k) m = fmaxf(m, l[k]);
                } else {
    #pragma unroll
                    for (int k = 0; k < 32; ++k) m = k < valid ? fmaxf(m, l[k]) : m;
                }
            }
            rowstat[cg * kM + li] = make_float2(m, 0.f);
            sm100::named_bar_sync(1, kEpiWarps * 32);
            if (cg == 0) {
                float M = -INFINITY;
    #pragma unroll
                for (int g = 0; g < 4; ++g) M = fmaxf(M, rowstat[g * kM + li].x);
                c_mb[li] = row_ok ? M * c1 : 0.f;
                if (row_ok && a.row_max) a.row_max[(int64_t)sq_slot * a.m + r] = M * a.inv_scale;
            }
            sm100::named_bar_sync(1, kEpiWarps * 32);
            const float mb = c_mb[li];

            // pass 2: P = 2^(l c1 - mb) <= 1 (0 past the causal frontier) as bf16,
            // the row sum of the same exponentials on the side; O = (P V) / sum at the end
            float ps[4] = {0.f, 0.f, 0.f, 0.f};
            for (int t = 0; t < T; ++t) {
                const int it = T + t, st = it & 1;
                sm100::mbar_wait(tfull + st, (it >> 1) & 1);
                sm100::tc_fence_after();
                sm100::tmem_ld32(lane_addr + st * kN, l);
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(tempty + st);
                const int valid = (int)imax(0, imin(32, row_end - ((int64_t)t * kN + cg * 32)));
                uint32_t pk[16];
                if (__all_sync(kFull, valid == 32)) {
    #pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float p0 = ex2(fmaf(l[2 * k], c1, -mb)), p1 = ex2(fmaf(l[2 * k + 1], c1, -mb));
                        ps[(2 * k) & 3] += p0;
                        ps[(2 * k + 1) & 3] += p1;
                        pk[k] = pack_bf16(p0, p1);
                    }
                } else {
    #pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float p0 = 2 * k < valid ? ex2(fmaf(l[2 * k], c1, -mb)) : 0.f;
                        const float p1 = 2 * k + 1 < valid ? ex2(fmaf(l[2 * k + 1], c1, -mb)) : 0.f;
                        ps[(2 * k) & 3] += p0;
                        ps[(2 * k + 1) & 3] += p1;
                        pk[k] = pack_bf16(p0, p1);
                    }
                }
                const int pb = t & 1;
                sm100::mbar_wait(pempty + pb, ((t >> 1) & 1) ^ 1);       // P V of tile t - 2 has read this buffer
                if constexpr (kTS) {
                    // this warp's 32 keys = 16 packed columns of its lane quarter
                    sm100::tc_fence_after();
                    sm100::tmem_st16(tmem_p + (uint32_t(32 * sub) << 16) + pb * 64 + cg * 16, pk);
                    sm100::tc_fence_before();
                } else {
                    uint8_t* pdst = sp + pb * LY::kP;
    #pragma unroll
                    for (int q = 0; q < 4; ++q)
                        *reinterpret_cast<uint4*>(pdst + swz(kM, li, cg * 4 + q)) =
                            make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                    sm100::fence_proxy_async();                          // generic writes -> async proxy
                }
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(pfull + pb);
            }
            // row sums: the four column groups' partials in a fixed order
            c_part[cg * kM + li] = (ps[0] + ps[1]) + (ps[2] + ps[3]);
            sm100::named_bar_sync(1, kEpiWarps * 32);
            S = (c_part[li] + c_part[kM + li]) + (c_part[2 * kM + li] + c_part[3 * kM + li]);
            if (cg == 0 && row_ok && a.row_sum) a.row_sum[(int64_t)sq_slot * a.m + r] = S;
            il = row_ok ? 1.f / S : 0.f;
            row_M = 0.f;   // written in pass 1
        }
        if (kOnePass && cg == 0 && row_ok && a.row_max) {
            a.row_max[(int64_t)sq_slot * a.m + r] = row_M * a.inv_scale;
            a.row_sum[(int64_t)sq_slot * a.m + r] = S;
        }

        // O: thread = row, warp cg holds dims 32 cg .. 32 cg + 31
        sm100::mbar_wait(&ofull, 0);
        sm100::tc_fence_after();
        if (cg * 32 < D) {
            sm100::tmem_ld32(tmem_o + (uint32_t(32 * sub) << 16) + cg * 32, l);
            if (row_ok) {
                float4* dst = reinterpret_cast<float4*>(a.out + ((int64_t)sq_slot * a.m + r) * D + cg * 32);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    dst[q] = make_float4(l[4 * q] * il, l[4 * q + 1] * il, l[4 * q + 2] * il, l[4 * q + 3] * il);
            }
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(tmem, kTmemCols);
    }
}

// ---------------------------------------------------------------- two Q tiles per CTA
// CTA = (query head, 256 prompt rows) as two 128-row Q tiles whose softmax
// warpgroups take turns on the tensor core: S_i = Q_i K^T lands in TMEM
// columns [128 i, 128 i + 128); warpgroup i (thread = row, the whole 128-key
// row in one thread: no cross-warp max exchange) forms P_i = 2^(S c1 - m_ref c1)
// as bf16 over the first 64 columns of its own S_i, and the MMA warp issues
// O_i += P_i V (A = P_i from TMEM, O_i in columns 256 + 128 i) followed at once
// by S_i of the next key tile, then the same for tile 1 -- so one warpgroup's
// softmax overlaps the other's MMAs.  The commit that signals S_i of tile t
// also covers O_i's previous P V, so a warpgroup may rescale its O_i row (lazy,
// when the row max grows by more than 2^8) as soon as it sees S_i.
// Warps: 0 K / Q producer, 1 MMA issuer, 2 TMEM allocator, 3 V^T producer,
// 4-7 softmax of Q tile 0, 8-11 softmax of Q tile 1.
#ifndef VLC_PF_PAIR
#define VLC_PF_PAIR 1
#endif
constexpr int kPairThreads = 128 + 256;
#ifndef VLC_PF_SLEEP
#define VLC_PF_SLEEP 1
#endif
#ifndef VLC_PF_FAST
#define VLC_PF_FAST 0   // full tiles: P without per-entry causal masks (measured slower)
#endif
#ifndef VLC_PF_REG
#define VLC_PF_REG 1    // softmax keeps the 128-key S row in registers (one TMEM round trip per tile)
#endif
VLC_DEV void pair_wait(uint64_t* bar, uint32_t parity) {   // waits without spinning on the issue port
    if (VLC_PF_SLEEP) sm100::mbar_wait_sleep(bar, parity);
    else sm100::mbar_wait(bar, parity);
}

VLC_DEV float maxn(const float (&l)[32]) {   // 32 values, a balanced tree of 3-input maxima
    float m[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = fmaxf(fmaxf(l[4 * k], l[4 * k + 1]), fmaxf(l[4 * k + 2], l[4 * k + 3]));
    return fmaxf(fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3])), fmaxf(fmaxf(m[4], m[5]), fmaxf(m[6], m[7])));
}

template <int D>
struct PL2 {
    static constexpr int KB = D / 64;
    static constexpr uint32_t kQ = KB * kM * 128;     // one 128-row Q tile
    static constexpr uint32_t kK = KB * kN * 128;     // one K tile
    static constexpr uint32_t kV = 2 * D * 128;       // one V^T tile: D rows x 128 keys
    static constexpr uint32_t kBytes = 2 * kQ + 2 * kK + 2 * kV + 1024;
};

template <int D>
__global__ void __launch_bounds__(kPairThreads, 1)
prefill_pair_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                    const __grid_constant__ CUtensorMap vmap, PrefillArgs a) {
    using LY = PL2<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sq = smem;
    uint8_t* sk = sq + 2 * LY::kQ;
    uint8_t* sv = sk + 2 * LY::kK;
    __shared__ uint64_t qfull, kfull[2], kempty[2], vfull[2], vempty[2], sfull[2], pfull[2], ofull;
    __shared__ uint32_t tmem_slot;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sq_slot = blockIdx.x;                                  // (b, l, query head)
    const int rb = gridDim.y - 1 - blockIdx.y;                       // longest blocks first, over all slots
    const int64_t kv_slot = (int64_t)(sq_slot / a.Hq) * a.Hkv + (sq_slot % a.Hq) / (a.Hq / a.Hkv);
    const int64_t r0 = (int64_t)rb * 2 * kM;
    const bool two = r0 + kM < a.m;                                  // Q tile 1 has rows
    const int T0 = (int)((imin(a.m, r0 + kM) + kN - 1) / kN);       // key tiles of Q tile 0
    const int T1 = two ? (int)((imin(a.m, r0 + 2 * kM) + kN - 1) / kN) : 0;
    const int T = two ? T1 : T0;

    if (threadIdx.x == 0) {
        sm100::mbar_init(&qfull, 1);
        for (int i = 0; i < 2; ++i) {
            sm100::mbar_init(kfull + i, 1); sm100::mbar_init(kempty + i, 1);
            sm100::mbar_init(vfull + i, 1); sm100::mbar_init(vempty + i, 1);
            sm100::mbar_init(sfull + i, 1); sm100::mbar_init(pfull + i, 4);
        }
        sm100::mbar_init(&ofull, 1);
        sm100::fence_barrier_init();
    }
    if (warp == 2) sm100::tmem_alloc(&tmem_slot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tmem_slot;                                 // S_i at 128 i, O_i at 256 + 128 i

    if (warp < 4) {
        if (VLC_PF_REG) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
        if (warp == 0 && lane == 0) {
            sm100::tma_prefetch(&qmap);
            sm100::tma_prefetch(&kmap);
            sm100::mbar_expect_tx(&qfull, (two ? 2 : 1) * LY::kQ);
            for (int i = 0; i < (two ? 2 : 1); ++i)
                for (int kb = 0; kb < LY::KB; ++kb)
                    sm100::tma_load_2d(sq + i * LY::kQ + kb * kM * 128, &qmap, &qfull, kb * 64,
                                       (int)(sq_slot * a.q_rows + r0 + i * kM));
            for (int t = 0; t < T; ++t) {
                const int st = t & 1;
                pair_wait(kempty + st, ((t >> 1) & 1) ^ 1);
                sm100::mbar_expect_tx(kfull + st, LY::kK);
                for (int kb = 0; kb < LY::KB; ++kb)
                    sm100::tma_load_2d(sk + st * LY::kK + kb * kN * 128, &kmap, kfull + st, kb * 64,
                                       (int)(kv_slot * a.kv_rows + (int64_t)t * kN));
            }
        } else if (warp == 3 && lane == 0) {
            sm100::tma_prefetch(&vmap);
            for (int t = 0; t < T; ++t) {
                const int st = t & 1;
                pair_wait(vempty + st, ((t >> 1) & 1) ^ 1);
                sm100::mbar_expect_tx(vfull + st, LY::kV);
                for (int kb = 0; kb < 2; ++kb)
                    sm100::tma_load_2d(sv + st * LY::kV + kb * D * 128, &vmap, vfull + st, t * kN + kb * 64,
                                       (int)(kv_slot * D));
            }
        } else if (warp == 1 && lane == 0) {
            constexpr uint32_t idesc_s = sm100::idesc_bf16_f32(kM, kN);
            constexpr uint32_t idesc_o = sm100::idesc_bf16_f32(kM, D);
            auto mma_s = [&](int i, int t) {   // S_i = Q_i K_t^T, then signal S_i (covers O_i's P V too)
                const uint32_t q_addr = sm100::smem_u32(sq + i * LY::kQ);
                const uint32_t k_addr = sm100::smem_u32(sk + (t & 1) * LY::kK);
#pragma unroll
                for (int kb = 0; kb < LY::KB; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        sm100::mma_bf16(tmem + i * kN, sm100::sdesc_k_sw128(q_addr + kb * kM * 128 + kk * 32),
                                        sm100::sdesc_k_sw128(k_addr + kb * kN * 128 + kk * 32), idesc_s,
                                        (kb | kk) != 0);
                sm100::mma_commit(sfull + i);
            };
            auto mma_pv = [&](int i, int t) {  // O_i += P_i V_t, P_i packed over S_i's first 64 columns
                const uint32_t v_addr = sm100::smem_u32(sv + (t & 1) * LY::kV);
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        sm100::mma_bf16_ts(tmem + 2 * kN + i * kN, tmem + i * kN + (kb * 4 + kk) * 8,
                                           sm100::sdesc_k_sw128(v_addr + kb * D * 128 + kk * 32), idesc_o,
                                           (t | kb | kk) != 0);
            };
            pair_wait(&qfull, 0);
            pair_wait(kfull, 0);
            sm100::tc_fence_after();
            mma_s(0, 0);
            if (two) mma_s(1, 0);
            sm100::mma_commit(kempty);
            for (int t = 0; t < T; ++t) {
                const bool h0 = t < T0, n0 = t + 1 < T0, n1 = two && t + 1 < T1;
                if (n0 || n1) pair_wait(kfull + ((t + 1) & 1), ((t + 1) >> 1) & 1);
                pair_wait(vfull + (t & 1), (t >> 1) & 1);
                if (h0) {
                    pair_wait(pfull, t & 1);
                    sm100::tc_fence_after();
                    mma_pv(0, t);
                    if (n0) mma_s(0, t + 1);
                }
                if (two) {
                    pair_wait(pfull + 1, t & 1);
                    sm100::tc_fence_after();
                    mma_pv(1, t);
                    if (n1) mma_s(1, t + 1);
                }
                sm100::mma_commit(vempty + (t & 1));
                if (n0 || n1) sm100::mma_commit(kempty + ((t + 1) & 1));
            }
            sm100::mma_commit(&ofull);
        }
    } else {
        // ---- softmax warpgroup wg of Q tile wg: thread = row, the whole 128-key row
        if (VLC_PF_REG) asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n");
        const int wg = (warp - 4) >> 2, sub = warp & 3;
        const int li = 32 * sub + lane;
        const int Ti = wg ? T1 : T0;
        const int64_t r = r0 + wg * kM + li;
        const bool row_ok = r < a.m;
        const int64_t row_end = row_ok ? r + 1 : 0;                   // causal: keys [0, r]
        const uint32_t lq = uint32_t(32 * sub) << 16;
        const uint32_t s_addr = tmem + lq + wg * kN, o_addr = tmem + lq + 2 * kN + wg * kN;
        const float c1 = a.inv_scale * kLog2e;
        const float grow_raw = 8.f / c1;
        float m_ref = -INFINITY, m_true = -INFINITY;
        float ps[4] = {0.f, 0.f, 0.f, 0.f};
        float l[32];
#if VLC_PF_REG
        // the whole 128-key S row in registers: four loads in flight, one wait,
        // then the row max and P from the same registers
        uint32_t sr[4][32];
        for (int t = 0; t < Ti; ++t) {
            pair_wait(sfull + wg, t & 1);
            sm100::tc_fence_after();
            const int64_t k0 = (int64_t)t * kN;
            const bool full = __all_sync(kFull, k0 + kN <= row_end);
#pragma unroll
            for (int c = 0; c < 4; ++c) sm100::tmem_ld32_issue(s_addr + 32 * c, sr[c]);
#pragma unroll
            for (int c = 0; c < 4; ++c) sm100::tmem_ld32_wait(sr[c]);   // the first waits; all tie their registers
            float tm = -INFINITY;
            if (full) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float v[32];
#pragma unroll
                    for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(sr[c][k]);
                    tm = fmaxf(tm, maxn(v));
                }
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int valid = (int)imax(0, imin(32, row_end - (k0 + 32 * c)));
#pragma unroll
                    for (int k = 0; k < 32; ++k) tm = k < valid ? fmaxf(tm, __uint_as_float(sr[c][k])) : tm;
                }
            }
            m_true = fmaxf(m_true, tm);
            const bool grow = tm > m_ref + grow_raw;
            if (__any_sync(kFull, grow)) {
                const float sc = (grow && m_ref != -INFINITY) ? ex2((m_ref - tm) * c1) : 1.f;
                if (t > 0) {   // every earlier P V into O_i is complete (the S_i signal covers it)
#pragma unroll 1
                    for (int c = 0; c < D / 32; ++c) {
                        float o[32];
                        sm100::tmem_ld32(o_addr + 32 * c, o);
#pragma unroll
                        for (int k = 0; k < 32; ++k) o[k] *= sc;
                        sm100::tmem_st32(o_addr + 32 * c, o);
                    }
                }
                if (grow) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) ps[k] *= sc;
                    m_ref = tm;
                }
            }
            const float mb = m_ref * c1;
            if (full) {
                // packed pairs: FFMA2 for the exponent arguments, FADD2 for two of the
                // four sum chains (row sums only need float32 rounding)
                const float2 c1v = make_float2(c1, c1), nmb = make_float2(-mb, -mb);
                float2 s01 = make_float2(ps[0], ps[1]), s23 = make_float2(ps[2], ps[3]);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t pk[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float2 u = __ffma2_rn(make_float2(__uint_as_float(sr[c][2 * k]), __uint_as_float(sr[c][2 * k + 1])),
                                                    c1v, nmb);
                        const float2 e = make_float2(ex2(u.x), ex2(u.y));
                        if (k & 1) s23 = __fadd2_rn(s23, e);
                        else s01 = __fadd2_rn(s01, e);
                        pk[k] = pack_bf16(e.x, e.y);
                    }
                    sm100::tmem_st16_nowait(s_addr + 16 * c, pk);
                }
                ps[0] = s01.x; ps[1] = s01.y; ps[2] = s23.x; ps[3] = s23.y;
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t pk[16];
                    const int valid = (int)imax(0, imin(32, row_end - (k0 + 32 * c)));
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float p0 = 2 * k < valid ? ex2(fmaf(__uint_as_float(sr[c][2 * k]), c1, -mb)) : 0.f;
                        const float p1 = 2 * k + 1 < valid ? ex2(fmaf(__uint_as_float(sr[c][2 * k + 1]), c1, -mb)) : 0.f;
                        ps[(2 * k) & 3] += p0;
                        ps[(2 * k + 1) & 3] += p1;
                        pk[k] = pack_bf16(p0, p1);
                    }
                    sm100::tmem_st16_nowait(s_addr + 16 * c, pk);
                }
            }
            sm100::tmem_st_wait();
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(pfull + wg);
        }
#else
        for (int t = 0; t < Ti; ++t) {
            pair_wait(sfull + wg, t & 1);
            sm100::tc_fence_after();
            const int64_t k0 = (int64_t)t * kN;
            const bool full = __all_sync(kFull, k0 + kN <= row_end);
            // sweep A: the tile's row max
            float tm = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                sm100::tmem_ld32(s_addr + 32 * c, l);
                if (full) {
                    tm = fmaxf(tm, maxn(l));
                } else {
                    const int valid = (int)imax(0, imin(32, row_end - (k0 + 32 * c)));
#pragma unroll
                    for (int k = 0; k < 32; ++k) tm = k < valid ? fmaxf(tm, l[k]) : tm;
                }
            }
            m_true = fmaxf(m_true, tm);
            const bool grow = tm > m_ref + grow_raw;
            if (__any_sync(kFull, grow)) {
                const float sc = (grow && m_ref != -INFINITY) ? ex2((m_ref - tm) * c1) : 1.f;
                if (t > 0) {   // every earlier P V into O_i is complete (the S_i signal covers it)
#pragma unroll 1
                    for (int c = 0; c < D / 32; ++c) {
                        float o[32];
                        sm100::tmem_ld32(o_addr + 32 * c, o);
#pragma unroll
                        for (int k = 0; k < 32; ++k) o[k] *= sc;
                        sm100::tmem_st32(o_addr + 32 * c, o);
                    }
                }
                if (grow) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) ps[k] *= sc;
                    m_ref = tm;
                }
            }
            const float mb = m_ref * c1;
            // sweep B: P over S_i's own columns (chunk c's 16 packed columns only
            // overwrite S columns already loaded: 16 c + 15 < 32 (c + 1))
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                sm100::tmem_ld32(s_addr + 32 * c, l);
                uint32_t pk[16];
                if (VLC_PF_FAST && full) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float p0 = ex2(fmaf(l[2 * k], c1, -mb)), p1 = ex2(fmaf(l[2 * k + 1], c1, -mb));
                        ps[(2 * k) & 3] += p0;
                        ps[(2 * k + 1) & 3] += p1;
                        pk[k] = pack_bf16(p0, p1);
                    }
                } else {
                    const int valid = full ? 32 : (int)imax(0, imin(32, row_end - (k0 + 32 * c)));
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float p0 = 2 * k < valid ? ex2(fmaf(l[2 * k], c1, -mb)) : 0.f;
                        const float p1 = 2 * k + 1 < valid ? ex2(fmaf(l[2 * k + 1], c1, -mb)) : 0.f;
                        ps[(2 * k) & 3] += p0;
                        ps[(2 * k + 1) & 3] += p1;
                        pk[k] = pack_bf16(p0, p1);
                    }
                }
                sm100::tmem_st16(s_addr + 16 * c, pk);
            }
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(pfull + wg);
        }
#endif
        if (Ti > 0) {
            const float l_ref = (ps[0] + ps[1]) + (ps[2] + ps[3]);
            if (row_ok && a.row_max) {
                a.row_max[(int64_t)sq_slot * a.m + r] = m_true * a.inv_scale;
                a.row_sum[(int64_t)sq_slot * a.m + r] = l_ref * ex2((m_ref - m_true) * c1);
            }
            const float il = row_ok ? 1.f / l_ref : 0.f;
            pair_wait(&ofull, 0);
            sm100::tc_fence_after();
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                sm100::tmem_ld32(o_addr + 32 * c, l);
                if (row_ok) {
                    float4* dst = reinterpret_cast<float4*>(a.out + ((int64_t)sq_slot * a.m + r) * D + 32 * c);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        dst[q] = make_float4(l[4 * q] * il, l[4 * q + 1] * il, l[4 * q + 2] * il, l[4 * q + 3] * il);
                }
            }
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(tmem, 512);
    }
}

// V [slots, kv_rows, D] -> V^T [slots, D, tpad] (keys contiguous), zero past m
__global__ void transpose_v(const __nv_bfloat16* __restrict__ v, __nv_bfloat16* __restrict__ vt, int64_t kv_rows,
                            int d, int64_t m, int64_t tpad) {
    __shared__ __nv_bfloat16 tile[32][33];
    const int64_t s = blockIdx.z;
    const int64_t j0 = (int64_t)blockIdx.x * 32, d0 = (int64_t)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t j = j0 + i, dd = d0 + threadIdx.x;
        tile[i][threadIdx.x] = (j < m && dd < d) ? v[(s * kv_rows + j) * d + dd] : __float2bfloat16(0.f);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t dd = d0 + i, j = j0 + threadIdx.x;
        if (dd < d && j < tpad) vt[(s * d + dd) * tpad + j] = tile[threadIdx.x][i];
    }
}

template <int D>
cudaError_t launch_prefill_d(const PrefillArgs& a, cudaStream_t st) {
    const int64_t tpad = prefill_tpad(a.m);
    const int64_t kv_slots = (int64_t)a.B * a.L * a.Hkv;
    dim3 tg((unsigned)((tpad + 31) / 32), (unsigned)((D + 31) / 32), (unsigned)kv_slots);
    transpose_v<<<tg, dim3(32, 8), 0, st>>>(static_cast<const __nv_bfloat16*>(a.v), static_cast<__nv_bfloat16*>(a.vt),
                                           a.kv_rows, D, a.m, tpad);
    CUtensorMap qmap, kmap, vmap;
    const int64_t q_slots = (int64_t)a.B * a.L * a.Hq;
    if (!make_tmap_2d(&qmap, a.q, q_slots * a.q_rows, D, kM)) return cudaErrorInvalidValue;
    if (!make_tmap_2d(&kmap, a.k, kv_slots * a.kv_rows, D, kN)) return cudaErrorInvalidValue;
    if (!make_tmap_2d_strided(&vmap, a.vt, kv_slots * D, (int)tpad, tpad, D, true)) return cudaErrorInvalidValue;
    if (VLC_PF_PAIR) {
        const size_t smem = PL2<D>::kBytes;
        cudaError_t e = cudaFuncSetAttribute(prefill_pair_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        // x = slot varies fastest in launch order, so every slot's longest
        // (last) row block is issued before any shorter one: the causal work
        // is scheduled longest first and the short blocks fill the tail
        dim3 grid((unsigned)q_slots, (unsigned)((a.m + 2 * kM - 1) / (2 * kM)));
        prefill_pair_kernel<D><<<grid, kPairThreads, smem, st>>>(qmap, kmap, vmap, a);
        return cudaGetLastError();
    }
    const size_t smem = PL<D>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(prefill_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)q_slots, (unsigned)((a.m + kM - 1) / kM));
    prefill_kernel<D><<<grid, kThreads, smem, st>>>(qmap, kmap, vmap, a);
    return cudaGetLastError();
}

}  // namespace

int64_t prefill_tpad(int64_t m) { return (m + 127) / 128 * 128; }

cudaError_t launch_prefill(const PrefillArgs& a, cudaStream_t st) {
    if (a.d == 64) return launch_prefill_d<64>(a, st);
    if (a.d == 128) return launch_prefill_d<128>(a, st);
    return cudaErrorInvalidValue;
}

}  // namespace vlc
