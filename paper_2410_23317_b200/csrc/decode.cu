// decode.cu -- K5: one decode step over the ragged compressed cache.
//
// reference: bench.py:356-372 (_decode_sequence: append the step's K/V row,
// then decode_step over the first k + s + 1 rows for the G query heads of each
// KV head) and _core.pyx:245-278 (decode_step: softmax(q K^T / sqrt(d)) V in
// fp32).  The G query rows of a KV head share one pass over its keys: each key
// row is read once from HBM for the whole group (GQA-aware), with lanes
// covering 8 bf16 (16 bytes) of a row each.  Cache reads use the coherent
// path: the appended row is written by this same launch.
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxG = 8;

template <int D>
__global__ void __launch_bounds__(kWarps * 32) decode_kernel(DecodeArgs a) {
    constexpr int LPK = D / 8;            // lanes per key row
    constexpr int KPW = 32 / LPK;         // keys per warp iteration
    __shared__ float s_m[kWarps][kMaxG], s_s[kWarps][kMaxG];
    __shared__ float s_acc[kWarps][kMaxG][D];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s = blockIdx.x;
    const int G = a.G;
    const int64_t n0 = a.base_len[s / a.Hkv];
    const int64_t n = n0 + a.step + 1;
    const int64_t seg = a.cache_off[s];
    uint4* kc = static_cast<uint4*>(a.k_cache) + seg * LPK;
    uint4* vc = static_cast<uint4*>(a.v_cache) + seg * LPK;

    // append this step's K/V row at position n0 + step (bench.py:368-371)
    if (tid < LPK) {
        const uint4* kn = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.k_new) + (int64_t)s * a.kv_stride);
        const uint4* vn = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.v_new) + (int64_t)s * a.kv_stride);
        kc[(n - 1) * LPK + tid] = kn[tid];
        vc[(n - 1) * LPK + tid] = vn[tid];
    }
    __syncthreads();

    // this lane's 8 query components for each of the G heads
    const int part = lane % LPK, sub = lane / LPK;
    float q[kMaxG][8];
    const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(a.q);
#pragma unroll
    for (int g = 0; g < kMaxG; ++g) {
        if (g < G) {
            const uint4 u = *reinterpret_cast<const uint4*>(qb + ((int64_t)s * G + g) * a.q_stride + part * 8);
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                q[g][2 * e] = bf16_lo(w4[e]) * a.inv_scale;
                q[g][2 * e + 1] = bf16_hi(w4[e]) * a.inv_scale;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) q[g][e] = 0.f;
        }
    }

    float m[kMaxG], ssum[kMaxG], acc[kMaxG][8];
#pragma unroll
    for (int g = 0; g < kMaxG; ++g) {
        m[g] = -INFINITY; ssum[g] = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[g][e] = 0.f;
    }

    // contiguous key range per warp
    const int64_t per_warp = (n + kWarps - 1) / kWarps;
    const int64_t j_begin = warp * per_warp, j_end = imin(n, j_begin + per_warp);
    constexpr int kUnroll = 2;
    for (int64_t j0 = j_begin; j0 < j_end; j0 += KPW * kUnroll) {
        uint4 kv[kUnroll], vv[kUnroll];
        bool ok[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t j = j0 + u * KPW + sub;
            ok[u] = j < j_end;
            kv[u] = ok[u] ? kc[j * LPK + part] : make_uint4(0, 0, 0, 0);
            vv[u] = ok[u] ? vc[j * LPK + part] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            float kf[8], vf[8];
            const uint32_t kw[4] = {kv[u].x, kv[u].y, kv[u].z, kv[u].w};
            const uint32_t vw[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                kf[2 * e] = bf16_lo(kw[e]); kf[2 * e + 1] = bf16_hi(kw[e]);
                vf[2 * e] = bf16_lo(vw[e]); vf[2 * e + 1] = bf16_hi(vw[e]);
            }
#pragma unroll
            for (int g = 0; g < kMaxG; ++g) {
                if (g >= G) continue;
                float dot = 0.f;
#pragma unroll
                for (int e = 0; e < 8; ++e) dot = fmaf(q[g][e], kf[e], dot);
#pragma unroll
                for (int o = LPK / 2; o >= 1; o >>= 1) dot += __shfl_xor_sync(kFull, dot, o);
                // every lane of a key group now holds that key's logit; other
                // key groups of the warp hold their own keys' logits
                const float l = ok[u] ? dot : -INFINITY;
                // warp-wide max over the KPW keys of this iteration
                float lm = l;
#pragma unroll
                for (int o = LPK; o < 32; o <<= 1) lm = fmaxf(lm, __shfl_xor_sync(kFull, lm, o));
                const float mnew = fmaxf(m[g], lm);
                if (mnew == -INFINITY) continue;
                const float scale = ex2((m[g] - mnew) * kLog2e);
                const float pj = ex2((l - mnew) * kLog2e);
                float psum = pj;
#pragma unroll
                for (int o = LPK; o < 32; o <<= 1) psum += __shfl_xor_sync(kFull, psum, o);
                ssum[g] = ssum[g] * scale + psum;
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[g][e] = fmaf(pj, vf[e], acc[g][e] * scale);
                m[g] = mnew;
            }
        }
    }
    // acc holds this lane's key group's partial; fold the KPW key groups
#pragma unroll
    for (int g = 0; g < kMaxG; ++g) {
        if (g >= G) continue;
#pragma unroll
        for (int e = 0; e < 8; ++e)
#pragma unroll
            for (int o = LPK; o < 32; o <<= 1) acc[g][e] += __shfl_xor_sync(kFull, acc[g][e], o);
        if (lane < LPK) {
#pragma unroll
            for (int e = 0; e < 8; ++e) s_acc[warp][g][part * 8 + e] = acc[g][e];
        }
        if (lane == 0) { s_m[warp][g] = m[g]; s_s[warp][g] = ssum[g]; }
    }
    __syncthreads();
    // combine warps: thread t handles (g, dim) pairs
    for (int idx = tid; idx < G * D; idx += kWarps * 32) {
        const int g = idx / D, dim = idx % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_m[w][g]);
        float S = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            if (s_m[w][g] == -INFINITY) continue;
            const float f = ex2((s_m[w][g] - M) * kLog2e);
            S = fmaf(s_s[w][g], f, S);
            O = fmaf(s_acc[w][g][dim], f, O);
        }
        a.out[((int64_t)s * G + g) * D + dim] = O / S;
    }
}

}  // namespace

cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t st) {
    if (a.G > kMaxG) return cudaErrorInvalidValue;
    switch (a.d) {
        case 64: decode_kernel<64><<<a.slots, kWarps * 32, 0, st>>>(a); break;
        case 128: decode_kernel<128><<<a.slots, kWarps * 32, 0, st>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace vlc
