// decode.cu -- K5: one decode step over the ragged compressed cache.
//
// reference: bench.py:356-372 (_decode_sequence: append the step's K/V row,
// then decode_step over the first k + s + 1 rows for the G query heads of each
// KV head) and _core.pyx:245-278 (decode_step: softmax(q K^T / sqrt(d)) V, fp32).
//
// One CTA per (b, l, kv) slot streams the slot's K and V rows (contiguous in
// its cache segment) through a kStages-deep shared-memory ring filled by 1-D
// TMA bulk copies, so ~kStages*16 KB per CTA are always in flight without
// occupying registers.  Each 32-row chunk is reduced in three short phases:
// (A) logits, one K-row load shared by all G query heads (GQA-aware: every key
// row is read from HBM once per step for the whole group); (B) per-head online
// softmax update, one warp per head; (C) P.V with threads over (head, dims).
// No workspace and no cross-CTA merge.  The chunk holding row k + step takes it
// from k_new / v_new and also appends it to the cache for later steps.
#include "sm100.cuh"
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxG = 8;
constexpr int kChunk = 32;     // rows per ring stage
constexpr int kStages = 4;

template <int D, int G>
struct Cfg {
    static constexpr int LPK = D / 8;                  // lanes per key row (16-byte pieces)
    static constexpr int KPI = 32 / LPK;               // keys per warp instruction
    static constexpr int UNITS = kChunk / KPI;         // key groups per chunk
    static constexpr int UPW = UNITS / kWarps;         // key groups per warp
    static constexpr int DP = D / 2;                   // dim pairs
    static constexpr int HSTRIDE = kThreads / DP;      // heads covered per thread sweep
    static constexpr int HPT = (G + HSTRIDE - 1) / HSTRIDE;   // heads per thread in phase C
    static constexpr uint32_t kRowBytes = D * 2;
    static constexpr uint32_t kStageBytes = kChunk * kRowBytes;
    static constexpr uint32_t kBytes = 2 * kStages * kStageBytes;
    static_assert(UNITS % kWarps == 0, "chunk must split evenly over the warps");
};

VLC_DEV void unpack8(const uint4& u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) { f[2 * e] = bf16_lo(w[e]); f[2 * e + 1] = bf16_hi(w[e]); }
}

template <int D, int G>
__global__ void __launch_bounds__(kThreads) decode_kernel(DecodeArgs a) {
    using C = Cfg<D, G>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* kring = smem;                                   // [kStages][kChunk][D] bf16
    uint8_t* vring = smem + kStages * C::kStageBytes;        // [kStages][kChunk][D] bf16
    __shared__ float lg[G][kChunk];                          // logits, then probabilities
    __shared__ float h_scale[G], h_sum[G];
    __shared__ uint64_t bar[kStages];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int pc = lane % C::LPK, sub = lane / C::LPK;
    const int s = blockIdx.x;
    const int64_t n = a.base_len[s / a.Hkv] + a.step + 1;   // rows this step
    const int64_t new_row = n - 1;
    const int nchunks = (int)((n + kChunk - 1) / kChunk);
    const size_t seg = (size_t)a.cache_off[s] * C::kRowBytes;
    const uint8_t* kc = static_cast<const uint8_t*>(a.k_cache) + seg;
    const uint8_t* vc = static_cast<const uint8_t*>(a.v_cache) + seg;

    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) sm100::mbar_init(&bar[i], 1);
        sm100::fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int c) {   // rows of chunk c already in the cache (not the new row)
        const int st = c % kStages;
        const int64_t j0 = (int64_t)c * kChunk;
        const int64_t j1 = imin(j0 + kChunk, new_row);
        const uint32_t bytes = j1 > j0 ? (uint32_t)(j1 - j0) * C::kRowBytes : 0u;
        sm100::fence_proxy_async();
        sm100::mbar_expect_tx(&bar[st], 2 * bytes);
        if (bytes) {
            sm100::bulk_load(kring + st * C::kStageBytes, kc + j0 * C::kRowBytes, bytes, &bar[st]);
            sm100::bulk_load(vring + st * C::kStageBytes, vc + j0 * C::kRowBytes, bytes, &bar[st]);
        }
    };
    if (tid == 0)
        for (int c = 0; c < kStages && c < nchunks; ++c) issue(c);

    // query pieces of every head for phase A (this lane's 8 dims)
    const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(a.q);
    float q[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(qb + ((int64_t)s * G + g) * a.q_stride + pc * 8), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) q[g][e] = f[e] * a.inv_scale;
    }
    // phase-C ownership: dim pair dp, heads gb, gb + HSTRIDE, ...
    const int dp = tid % C::DP, gb = tid / C::DP;
    float acc[C::HPT][2];
#pragma unroll
    for (int h = 0; h < C::HPT; ++h) acc[h][0] = acc[h][1] = 0.f;
    // phase-B state (warp g owns head g)
    float run_m = -INFINITY, run_s = 0.f;

    for (int c = 0; c < nchunks; ++c) {
        const int st = c % kStages;
        const int64_t j0 = (int64_t)c * kChunk;
        const int nk = (int)imin(kChunk, n - j0);
        uint8_t* ks = kring + st * C::kStageBytes;
        uint8_t* vs = vring + st * C::kStageBytes;
        if (new_row < j0 + kChunk) {   // last chunk: bring in the new row (CTA-uniform)
            if (tid < 2 * C::LPK) {
                const bool isv = tid >= C::LPK;
                const int piece = tid % C::LPK;
                const uint4 val = reinterpret_cast<const uint4*>(
                    static_cast<const __nv_bfloat16*>(isv ? a.v_new : a.k_new) + (int64_t)s * a.kv_stride)[piece];
                reinterpret_cast<uint4*>((isv ? vs : ks) + (new_row - j0) * C::kRowBytes)[piece] = val;
                reinterpret_cast<uint4*>(static_cast<uint8_t*>(isv ? a.v_cache : a.k_cache) + seg +
                                         new_row * C::kRowBytes)[piece] = val;
            }
            __syncthreads();
        }
        sm100::mbar_wait(&bar[st], (c / kStages) & 1);

        // ---- A: logits; each K-row piece is loaded once for all G heads
#pragma unroll
        for (int u = 0; u < C::UPW; ++u) {
            const int kk = (warp + u * kWarps) * C::KPI + sub;
            float kf[8];
            unpack8(reinterpret_cast<const uint4*>(ks + kk * C::kRowBytes)[pc], kf);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float dot = 0.f;
#pragma unroll
                for (int e = 0; e < 8; ++e) dot = fmaf(q[g][e], kf[e], dot);
#pragma unroll
                for (int o = C::LPK / 2; o >= 1; o >>= 1) dot += __shfl_xor_sync(kFull, dot, o);
                if (pc == 0) lg[g][kk] = kk < nk ? dot : -INFINITY;
            }
        }
        __syncthreads();
        // ---- B: online softmax update per head (warp g)
        if (warp < G) {
            const float l = lg[warp][lane];
            const float mn = fmaxf(run_m, warp_max(l));      // finite: row 0 of the chunk is valid
            const float p = ex2((l - mn) * kLog2e);
            const float sc = ex2((run_m - mn) * kLog2e);       // 0 on the first chunk
            lg[warp][lane] = p;
            run_s = run_s * sc + warp_sum(p);
            run_m = mn;
            if (lane == 0) { h_scale[warp] = sc; h_sum[warp] = run_s; }
        }
        __syncthreads();
        // ---- C: acc = acc * scale + P.V over the chunk
#pragma unroll
        for (int h = 0; h < C::HPT; ++h) {
            const int g = gb + h * C::HSTRIDE;
            if (g < G) {
                const float sc = h_scale[g];
                float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
                if (nk == kChunk) {
#pragma unroll 8
                    for (int kk = 0; kk < kChunk; kk += 2) {
                        const uint32_t u0 = reinterpret_cast<const uint32_t*>(vs + kk * C::kRowBytes)[dp];
                        const uint32_t u1 = reinterpret_cast<const uint32_t*>(vs + (kk + 1) * C::kRowBytes)[dp];
                        const float p0 = lg[g][kk], p1 = lg[g][kk + 1];
                        a0 = fmaf(p0, bf16_lo(u0), a0);
                        a1 = fmaf(p0, bf16_hi(u0), a1);
                        b0 = fmaf(p1, bf16_lo(u1), b0);
                        b1 = fmaf(p1, bf16_hi(u1), b1);
                    }
                } else {   // rows past nk hold stale bytes: never touch them
                    for (int kk = 0; kk < nk; ++kk) {
                        const uint32_t u0 = reinterpret_cast<const uint32_t*>(vs + kk * C::kRowBytes)[dp];
                        const float p0 = lg[g][kk];
                        a0 = fmaf(p0, bf16_lo(u0), a0);
                        a1 = fmaf(p0, bf16_hi(u0), a1);
                    }
                }
                acc[h][0] = fmaf(acc[h][0], sc, a0 + b0);
                acc[h][1] = fmaf(acc[h][1], sc, a1 + b1);
            }
        }
        __syncthreads();   // stage and logits free
        if (tid == 0 && c + kStages < nchunks) issue(c + kStages);
    }
#pragma unroll
    for (int h = 0; h < C::HPT; ++h) {
        const int g = gb + h * C::HSTRIDE;
        if (g < G) {
            const float inv = 1.f / h_sum[g];
            float2 o = make_float2(acc[h][0] * inv, acc[h][1] * inv);
            reinterpret_cast<float2*>(a.out + ((int64_t)s * G + g) * D)[dp] = o;
        }
    }
}

template <int D, int G>
cudaError_t launch_dg(const DecodeArgs& a, cudaStream_t st) {
    using C = Cfg<D, G>;
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::kBytes);
    if (e != cudaSuccess) return e;
    decode_kernel<D, G><<<a.slots, kThreads, C::kBytes, st>>>(a);
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_d(const DecodeArgs& a, cudaStream_t st) {
    switch (a.G) {
        case 1: return launch_dg<D, 1>(a, st);
        case 2: return launch_dg<D, 2>(a, st);
        case 3: return launch_dg<D, 3>(a, st);
        case 4: return launch_dg<D, 4>(a, st);
        case 5: return launch_dg<D, 5>(a, st);
        case 6: return launch_dg<D, 6>(a, st);
        case 7: return launch_dg<D, 7>(a, st);
        case 8: return launch_dg<D, 8>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t st) {
    if (a.G < 1 || a.G > kMaxG) return cudaErrorInvalidValue;
    if (a.d == 64) return launch_d<64>(a, st);
    if (a.d == 128) return launch_d<128>(a, st);
    return cudaErrorInvalidValue;
}

}  // namespace vlc
