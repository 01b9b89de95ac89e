// decode.cu -- K5: one decode step over the ragged compressed cache.
//
// reference: bench.py:356-372 (_decode_sequence: append the step's K/V row,
// then decode_step over the first k + s + 1 rows for the G query heads of each
// KV head) and _core.pyx:245-278 (decode_step: softmax(q K^T / sqrt(d)) V, fp32).
//
// One CTA per (b, l, kv) slot streams the slot's K and V rows through a
// 6-stage shared-memory ring of 16-row chunks, loaded by 2-D TMA with the
// 128-byte swizzle so tensor-core fragments come out of shared memory
// conflict-free.  Four one-warp groups take chunks round robin (group c % 4
// consumes chunk c), so four chunks are in compute at once and the serial
// chain of the slot's longest-budget layers is a quarter.  A CTA is 128
// threads and 48 KB of ring, so four fit per SM: two steps' grids (256 CTAs
// each at M7B) are resident together and the next step's prologue, loads and
// base-row chunks run under the current one (5.5 vs 6.2 us/step for two
// two-warp groups per chunk at 96 KB, 56 vs 62 at batch 8).  The G <= 8 query heads of the KV head
// are the N = 8 columns of transposed mma.sync tiles (GQA: every key row is
// read from HBM once per step for the whole group; no padding of the big M side):
//   S^T = K Q^T    m16n8k16, M = 16 keys, bf16 in, fp32 accumulate (exact products);
//   O^T += V^T P^T m16n8k16, M = 16 dims, K = 16 keys; P^T comes from the S^T
//                  accumulator through movmatrix, split into bf16 hi + lo parts
//                  (~2^-16 relative); V exact bf16, fp32 accumulate.
// Each warp keeps its own online-softmax state; the eight warps' (max, sum, O)
// partials merge once at the end.  Under programmatic dependent launch only
// the chunk holding the previous step's append (and the global writes) wait
// for the previous step: everything else is loaded and computed while it
// drains.  Each stage has two full barriers used alternately, so a group that
// runs a ring ahead of another never mistakes a stage's previous use for its
// chunk.  A stage is refilled as soon as the warps that consumed it arrive on
// its "empty" barrier.  The chunk holding row k + step takes that row from
// k_new / v_new through a small swizzled side buffer (the lanes whose ldmatrix
// row it is read there; the ring is only ever written by TMA) and appends it
// to the cache for later steps.
#include "sm100.cuh"
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

#ifndef VLC_DEC_GROUP_WARPS
#define VLC_DEC_GROUP_WARPS 1
#endif
#ifndef VLC_DEC_GROUPS
#define VLC_DEC_GROUPS 4
#endif
constexpr int kGroupWarps = VLC_DEC_GROUP_WARPS;   // warps per consumer group (16 rows each)
constexpr int kGroups = VLC_DEC_GROUPS;            // groups take chunks round-robin
constexpr int kWarps = kGroupWarps * kGroups;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxG = 8;
constexpr int kChunk = 16 * kGroupWarps;        // rows per ring stage
#ifndef VLC_DEC_STAGES
#define VLC_DEC_STAGES 6   // >= VLC_DEC_GROUPS: a group runs at most one use of a stage ahead
#endif
constexpr int kStages = VLC_DEC_STAGES;
#ifndef VLC_DEC_SCHAINS
#define VLC_DEC_SCHAINS 2   // accumulator chains of S = K Q^T (1 or 2)
#endif
#ifndef VLC_DEC_L2PF
#define VLC_DEC_L2PF 0   // L2 bulk prefetch of the rows beyond the first ring (measured slower: 7.28 vs 7.12 us/step, B8 72.5 vs 66.6)
#endif
#ifndef VLC_DEC_EARLYLAUNCH
#define VLC_DEC_EARLYLAUNCH 1
#endif
#ifndef VLC_DEC_EARLY_PERIOD
#define VLC_DEC_EARLY_PERIOD 32   // under early release, every P-th step releases late (bounds the deferred rows)
#endif
#ifndef VLC_DEC_PROBE
#define VLC_DEC_PROBE 0   // timing probes (wrong results), bits: 1 = no math, 2 = no TMA after the first ring, 4 = no wait for the previous step, 8 = no merge / output
#endif

template <int D>
struct Cfg {
    static constexpr int KB = D / 64;                        // 64-dim (128 B) swizzle boxes per row
    static constexpr uint32_t kBox = kChunk * 128;           // bytes of one box (64 rows x 128 B)
    static constexpr uint32_t kTile = KB * kBox;             // K (or V) tile of a chunk
    static constexpr uint32_t kStage = 2 * kTile;            // K + V
    static constexpr uint32_t kBytes = kStages * kStage + 1024;   // + alignment slack
    static constexpr int MT = D / 16;                        // 16-dim output tiles
};

// byte offset of 16-byte piece `c` (of the row's D/8) of row r inside a tile
template <int D>
VLC_DEV uint32_t swz(int r, int c) {
    return (uint32_t)((c >> 3) * Cfg<D>::kBox + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

VLC_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
VLC_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
// D = A(16x16) * B(16x8) + C, bf16 -> f32, full A fragment
VLC_DEV void mma16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
VLC_DEV uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
VLC_DEV uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
VLC_DEV float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

template <int D, int G>
#ifndef VLC_DEC_MINB
#define VLC_DEC_MINB (512 / kThreads)
#endif
__global__ void __launch_bounds__(kThreads, VLC_DEC_MINB)
decode_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap, DecodeArgs a) {
    using C = Cfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // two full barriers per stage, alternating by the stage's use (chunk c is
    // use c / kStages): a group running a ring ahead of the refills waits on
    // the other barrier of the pair, whose pending phase cannot be mistaken
    // for its chunk's (a parity wait alone would accept the previous use)
    __shared__ uint64_t bar[kStages][2], empty[kStages];
    __shared__ float part_m[kWarps][8], part_s[kWarps][8];
    // the step's new K / V row (one chunk per CTA holds it), laid out like its
    // row of a swizzled tile with the row term dropped: the lanes whose
    // ldmatrix row is the new row take this as their row base, so the TMA ring
    // is never written by threads
    constexpr uint32_t kNewBytes = (Cfg<D>::KB - 1) * Cfg<D>::kBox + 128;
    __shared__ __align__(128) uint8_t new_kv[2][kNewBytes];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int grp = warp / kGroupWarps, wig = warp % kGroupWarps;   // consumer group, warp in group
    const int row = lane >> 2, quad = lane & 3;              // fragment row (key / dim), column pair (heads)
    const int s = blockIdx.x;
    const int64_t n = a.base_len[s / a.Hkv] + a.step + 1;    // rows this step
    const int64_t new_row = n - 1;
    const int64_t seg = a.cache_off[s];
    const int nchunks = (int)((n + kChunk - 1) / kChunk);

    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            sm100::mbar_init(&bar[i][0], 1);
            sm100::mbar_init(&bar[i][1], 1);
            sm100::mbar_init(&empty[i], kGroupWarps);
        }
        sm100::fence_barrier_init();
        sm100::tma_prefetch(&kmap);
        sm100::tma_prefetch(&vmap);
    }
    __syncthreads();
    auto issue = [&](int c) {
        const int st = c % kStages;
        uint8_t* kdst = smem + st * C::kStage;
        const int y = (int)(seg + (int64_t)c * kChunk);
        uint64_t* fb = &bar[st][(c / kStages) & 1];
        sm100::mbar_expect_tx(fb, C::kStage);
        for (int kb = 0; kb < C::KB; ++kb) {
            sm100::tma_load_2d(kdst + kb * C::kBox, &kmap, fb, kb * 64, y);
            sm100::tma_load_2d(kdst + C::kTile + kb * C::kBox, &vmap, fb, kb * 64, y);
        }
    };
    // Programmatic dependent launch.  When the caller guarantees that the
    // previous kernel is this cache's decode step `step - 1` (a.chained), rows
    // written before it are final (that step waited for them), so only the
    // chunk holding row k + step - 1 (its append, chunk `pend`) has to wait
    // for it: the TMA of that chunk is issued after griddepcontrol.wait, and
    // every thread waits before its first global write (the append, the
    // output).  All other chunks are loaded AND computed while the previous
    // step drains.  The next step may launch once a thread of every CTA is
    // past its wait (this step's predecessor is then complete, so all the next
    // step reads early is final).  Without the guarantee (a.chained == 0)
    // everything waits up front.
    // Early release (a.early: chained, and the step fills the GPU so at most about
    // two steps are ever resident): the step releases its successor at once;
    // since earlier steps may then still be running, every chunk holding rows
    // they appended is loaded only after griddepcontrol.wait.  Otherwise the
    // step releases its successor after that wait and only the chunk holding the
    // previous step's append waits.
    const int pend = a.chained ? (int)((n - 2) / kChunk) : -1;
    constexpr int kPeriod = VLC_DEC_EARLY_PERIOD;
    const bool early = a.chained && a.early && (a.step % kPeriod) != 0;   // this step releases at once
    // rows whose appends may still be in flight: those of steps t .. step-1, t the
    // latest step that released late (it had waited, so every step before t is complete)
    int first_dep = pend;
    if (a.chained && a.early) {
        const int64_t prev = a.step - 1, t = prev - prev % kPeriod;
        first_dep = (int)((a.base_len[s / a.Hkv] + t) / kChunk);
    }
    auto deferred = [&](int c) { return c >= 0 && pend >= 0 && c >= first_dep && c <= pend; };
    bool waited = !a.chained;
    auto wait_prev = [&]() {
        if (!waited) {
            if (!(VLC_DEC_PROBE & 4)) asm volatile("griddepcontrol.wait;" ::: "memory");   // probe 4: no wait (racy)
            if (!early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
            waited = true;
        }
    };
    if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (!a.chained) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    if (tid == 0) {
        for (int c = 0; c < kStages && c < nchunks; ++c)
            if (!deferred(c)) issue(c);
        // rows beyond the ring: start their HBM reads now (into L2), so the
        // refills that follow wait for L2, not HBM (a no-op when resident)
        if (VLC_DEC_L2PF && nchunks > kStages) {
            const int64_t r0 = seg + (int64_t)kStages * kChunk, nr = seg + n - 1 - r0;   // the new row excluded
            if (nr > 0) {
                const uint32_t bytes = (uint32_t)(nr * D * 2);
                sm100::prefetch_l2_bulk(static_cast<const __nv_bfloat16*>(a.k_cache) + r0 * D, bytes);
                sm100::prefetch_l2_bulk(static_cast<const __nv_bfloat16*>(a.v_cache) + r0 * D, bytes);
            }
        }
    }

    // Q^T as B fragments per 16-dim k-step: b0 = Q[head row][dims 2q, 2q+1], b1 = dims + 8
    const uint32_t* qw = reinterpret_cast<const uint32_t*>(a.q);
    uint32_t qb[D / 16][2];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
        if (row < G) {
            const int64_t base = (((int64_t)s * G + row) * a.q_stride + kk * 16) / 2;
            qb[kk][0] = qw[base + quad];
            qb[kk][1] = qw[base + 4 + quad];
        } else {
            qb[kk][0] = qb[kk][1] = 0u;
        }
    }
    if (tid == 0) {   // initial chunks that wait for the previous step
        for (int c = 0; c < kStages && c < nchunks; ++c)
            if (deferred(c)) {
                wait_prev();
                issue(c);
            }
    }
    // O^T accumulators: tile t covers dims 16t..16t+15; c0,c1 = (dim 16t+row, heads 2q, 2q+1),
    // c2,c3 = (dim 16t+row+8, heads 2q, 2q+1)
    float o[C::MT][4];
#pragma unroll
    for (int t = 0; t < C::MT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
    float run_m[2] = {-INFINITY, -INFINITY}, run_s[2] = {0.f, 0.f};   // heads 2q, 2q+1
    const float c1 = a.inv_scale * kLog2e;

    for (int c = grp; c < nchunks; c += kGroups) {
        const int st = c % kStages;
        const int64_t j0 = (int64_t)c * kChunk;
        uint8_t* ks = smem + st * C::kStage;
        uint8_t* vs = ks + C::kTile;
        // chunk c is use c / kStages of its stage: wait on that use's barrier
        if (!((VLC_DEC_PROBE & 2) && c >= kStages))
            sm100::mbar_wait(&bar[st][(c / kStages) & 1], (c / (2 * kStages)) & 1);
        const bool has_new = new_row < j0 + kChunk;   // last chunk (group-uniform)
        if (has_new) {   // the new row: into this group's row buffer and appended to the cache
            wait_prev();                                           // the append is a global write
            for (int gt = tid % (kGroupWarps * 32); gt < 2 * (D / 8); gt += kGroupWarps * 32) {
                const bool isv = gt >= D / 8;
                const int piece = gt % (D / 8);
                const uint4 val = reinterpret_cast<const uint4*>(
                    static_cast<const __nv_bfloat16*>(isv ? a.v_new : a.k_new) + (int64_t)s * a.kv_stride)[piece];
                *reinterpret_cast<uint4*>(new_kv[isv] + (piece >> 3) * C::kBox +
                                          (((piece & 7) ^ (int)((new_row - j0) & 7)) << 4)) = val;
                reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(isv ? a.v_cache : a.k_cache) +
                                         (seg + new_row) * D)[piece] = val;
            }
            if (kGroupWarps == 1) __syncwarp();   // a one-warp group: the warp's own barrier
            else sm100::named_bar_sync(1 + grp, kGroupWarps * 32);
        }
        if (VLC_DEC_PROBE & 1) {   // timing probe: no math
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&empty[st]);
            if (wig == 0 && lane == 0 && c + kStages < nchunks) {
                sm100::mbar_wait(&empty[st], (c / kStages) & 1);
                if (deferred(c + kStages)) wait_prev();
                issue(c + kStages);
            }
            continue;
        }
        // ---- S^T = K Q^T for this warp's 16 keys
        const int kr = wig * 16;                               // first key of the warp
        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t kbase = sm100::smem_u32(ks);
        const int arow = kr + (lane & 7) + ((lane >> 3) & 1) * 8;   // ldmatrix row of this lane
        const uint32_t krow = (has_new && j0 + arow == new_row) ? sm100::smem_u32(new_kv[0]) : kbase + arow * 128;
        auto kaddr = [&](int piece) { return krow + swz<D>(arow, piece) - arow * 128; };
#if VLC_DEC_SCHAINS == 2
        // two independent accumulator chains over the k-steps (half the HMMA latency chain)
        float sacc2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < D / 16; kk += 2) {
            uint32_t af[4], ag[4];
            ldsm_x4(kaddr(kk * 2 + (lane >> 4)), af[0], af[1], af[2], af[3]);
            ldsm_x4(kaddr((kk + 1) * 2 + (lane >> 4)), ag[0], ag[1], ag[2], ag[3]);
            mma16(sacc, af, qb[kk][0], qb[kk][1]);
            mma16(sacc2, ag, qb[kk + 1][0], qb[kk + 1][1]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) sacc[i] += sacc2[i];
#else
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
            uint32_t af[4];
            ldsm_x4(kaddr(kk * 2 + (lane >> 4)), af[0], af[1], af[2], af[3]);
            mma16(sacc, af, qb[kk][0], qb[kk][1]);
        }
#endif
        // ---- online softmax per head over the warp's keys: thread holds keys
        //      kr+row (c0, c1) and kr+row+8 (c2, c3) for heads 2q (c0, c2), 2q+1 (c1, c3)
        const int64_t ja = j0 + kr + row, jb = ja + 8;
        const float l00 = ja < n ? sacc[0] : -INFINITY, l01 = ja < n ? sacc[1] : -INFINITY;
        const float l10 = jb < n ? sacc[2] : -INFINITY, l11 = jb < n ? sacc[3] : -INFINITY;
        float tm0 = fmaxf(l00, l10), tm1 = fmaxf(l01, l11);
#pragma unroll
        for (int o2 = 4; o2 < 32; o2 <<= 1) {
            tm0 = fmaxf(tm0, __shfl_xor_sync(kFull, tm0, o2));
            tm1 = fmaxf(tm1, __shfl_xor_sync(kFull, tm1, o2));
        }
        const float mn0 = fmaxf(run_m[0], tm0), mn1 = fmaxf(run_m[1], tm1);
        const float mb0 = mn0 == -INFINITY ? 0.f : mn0 * c1, mb1 = mn1 == -INFINITY ? 0.f : mn1 * c1;
        const float p00 = ex2(fmaf(l00, c1, -mb0)), p10 = ex2(fmaf(l10, c1, -mb0));
        const float p01 = ex2(fmaf(l01, c1, -mb1)), p11 = ex2(fmaf(l11, c1, -mb1));
        if (__any_sync(kFull, mn0 != run_m[0] || mn1 != run_m[1])) {
            const float sc0 = run_m[0] == -INFINITY ? 0.f : ex2(fmaf(run_m[0], c1, -mb0));
            const float sc1 = run_m[1] == -INFINITY ? 0.f : ex2(fmaf(run_m[1], c1, -mb1));
#pragma unroll
            for (int t = 0; t < C::MT; ++t) { o[t][0] *= sc0; o[t][1] *= sc1; o[t][2] *= sc0; o[t][3] *= sc1; }
            run_s[0] *= sc0;
            run_s[1] *= sc1;
        }
        run_m[0] = mn0;
        run_m[1] = mn1;
        run_s[0] += p00 + p10;
        run_s[1] += p01 + p11;
        // P^T as B fragments (keys x heads): transpose the two 8x8 key blocks;
        // hi + lo bf16 parts
        const float h00 = bf16_round(p00), h01 = bf16_round(p01), h10 = bf16_round(p10), h11 = bf16_round(p11);
        const uint32_t bh0 = movmatrix_t(pack_bf16(h00, h01)), bh1 = movmatrix_t(pack_bf16(h10, h11));
        const uint32_t bl0 = movmatrix_t(pack_bf16(p00 - h00, p01 - h01));
        const uint32_t bl1 = movmatrix_t(pack_bf16(p10 - h10, p11 - h11));
        // ---- O^T += V^T P^T: V^T A fragments by transposed ldmatrix of the warp's 16 rows
        const uint32_t vbase = sm100::smem_u32(vs);
        const int vrow = kr + (lane & 7) + (lane >> 4) * 8;
        const uint32_t vrowb = (has_new && j0 + vrow == new_row) ? sm100::smem_u32(new_kv[1]) : vbase + vrow * 128;
#pragma unroll
        for (int t = 0; t < C::MT; ++t) {
            uint32_t af[4];
            const int piece = t * 2 + ((lane >> 3) & 1);
            ldsm_x4_t(vrowb + swz<D>(vrow, piece) - vrow * 128, af[0], af[1], af[2], af[3]);
            mma16(o[t], af, bh0, bh1);
            mma16(o[t], af, bl0, bl1);
        }
        // stage consumed by this group's warps -> refill it (the group leader)
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&empty[st]);
        if (wig == 0 && lane == 0 && c + kStages < nchunks && !(VLC_DEC_PROBE & 2)) {
            sm100::mbar_wait(&empty[st], (c / kStages) & 1);
            if (deferred(c + kStages)) wait_prev();           // holds rows earlier steps appended
            issue(c + kStages);
        }
    }

    wait_prev();                                              // before the output writes
    if (VLC_DEC_PROBE & 8) return;                            // probe 8: no merge, no output
    // ---- merge the warps: per head, (max, sum) then O, through shared memory
#pragma unroll
    for (int o2 = 4; o2 < 32; o2 <<= 1) {
        run_s[0] += __shfl_xor_sync(kFull, run_s[0], o2);
        run_s[1] += __shfl_xor_sync(kFull, run_s[1], o2);
    }
    if (row == 0) {
        part_m[warp][2 * quad] = run_m[0]; part_s[warp][2 * quad] = run_s[0];
        part_m[warp][2 * quad + 1] = run_m[1]; part_s[warp][2 * quad + 1] = run_s[1];
    }
    __syncthreads();                                          // both groups are done with the ring
    if (VLC_DEC_PROBE & 32) return;                           // probe 32: only the first merge barrier
    // O partials as [warp][dim][8 heads]: a thread's two adjacent heads are one
    // 8-byte store and a warp's stores cover 64 consecutive floats (no bank
    // conflicts); the padding heads >= G are not stored at all
    float* po = reinterpret_cast<float*>(smem);               // ring is idle now
    __shared__ float f_s[kWarps][8], is_s[8];                 // per (warp, head) rescale, 1 / sum per head
    if (tid < G) {   // the merge's scalars once per head, not once per output
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, part_m[w][tid]);
        float S = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float f = part_m[w][tid] == -INFINITY ? 0.f : ex2((part_m[w][tid] - M) * c1);
            f_s[w][tid] = f;
            S = fmaf(part_s[w][tid], f, S);
        }
        is_s[tid] = 1.f / S;
    }
    if (2 * quad < G) {
#pragma unroll
        for (int t = 0; t < C::MT; ++t) {
            const int d0 = 16 * t + row;
            *reinterpret_cast<float2*>(po + (warp * D + d0) * 8 + 2 * quad) = make_float2(o[t][0], o[t][1]);
            *reinterpret_cast<float2*>(po + (warp * D + d0 + 8) * 8 + 2 * quad) = make_float2(o[t][2], o[t][3]);
        }
    }
    __syncthreads();
    if (VLC_DEC_PROBE & 16) return;                           // probe 16: no final combine / output
    for (int idx = tid; idx < G * D; idx += kThreads) {
        const int g = idx % G, dim = idx / G;
        float O = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) O = fmaf(po[(w * D + dim) * 8 + g], f_s[w][g], O);
        a.out[((int64_t)s * G + g) * D + dim] = O * is_s[g];
    }
}

template <int D, int G>
cudaError_t launch_dg(const DecodeArgs& a, const CUtensorMap& km, const CUtensorMap& vm, cudaStream_t st) {
    using C = Cfg<D>;
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::kBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.slots);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kBytes;
    cfg.stream = st;
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    DecodeArgs b = a;
    b.early = (VLC_DEC_EARLYLAUNCH && a.slots >= n_sm) ? 1 : 0;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (see kernel)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, decode_kernel<D, G>, km, vm, b);
}

template <int D>
cudaError_t launch_d(const DecodeArgs& a, cudaStream_t st) {
    CUtensorMap km, vm;
    if (!make_tmap_2d(&km, a.k_cache, a.cache_rows, D, kChunk) ||
        !make_tmap_2d(&vm, a.v_cache, a.cache_rows, D, kChunk))
        return cudaErrorInvalidValue;
    switch (a.G) {
        case 1: return launch_dg<D, 1>(a, km, vm, st);
        case 2: return launch_dg<D, 2>(a, km, vm, st);
        case 3: return launch_dg<D, 3>(a, km, vm, st);
        case 4: return launch_dg<D, 4>(a, km, vm, st);
        case 5: return launch_dg<D, 5>(a, km, vm, st);
        case 6: return launch_dg<D, 6>(a, km, vm, st);
        case 7: return launch_dg<D, 7>(a, km, vm, st);
        case 8: return launch_dg<D, 8>(a, km, vm, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

#ifdef VLC_DEC_LAUNCH   // a second build of this file with another CTA shape (decode_wide.cu)
cudaError_t VLC_DEC_LAUNCH(const DecodeArgs& a, cudaStream_t st) {
    if (a.G < 1 || a.G > kMaxG) return cudaErrorInvalidValue;
    if (a.d == 64) return launch_d<64>(a, st);
    if (a.d == 128) return launch_d<128>(a, st);
    return cudaErrorInvalidValue;
}
#else
// Grids smaller than the GPU (fewer slots than SMs) gain nothing from small
// CTAs -- no second step needs the room -- and each slot's stream is then the
// whole step: they take the wide CTA (two-warp groups, 32-row tiles, 256
// threads; decode_wide.cu).
cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t st) {
    if (a.G < 1 || a.G > kMaxG) return cudaErrorInvalidValue;
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (a.slots < n_sm) return launch_decode_wide(a, st);
    if (a.d == 64) return launch_d<64>(a, st);
    if (a.d == 128) return launch_d<128>(a, st);
    return cudaErrorInvalidValue;
}
#endif

}  // namespace vlc
