// decode.cu -- K5: one decode step over the ragged compressed cache.
//
// reference: bench.py:356-372 (_decode_sequence: append the step's K/V row,
// then decode_step over the first k + s + 1 rows for the G query heads of each
// KV head) and _core.pyx:245-278 (decode_step: softmax(q K^T / sqrt(d)) V, fp32).
//
// Split-K flash-decoding over a fixed work list: slot s owns
// chunk_off[s+1] - chunk_off[s] chunks of kDecodeChunk keys (sized for its
// final length k_s + n_steps, built by K2).  A persistent grid walks the list;
// each CTA loads a whole chunk (K and V, 16-byte lanes, every load in flight
// before any math), reduces it to a (max, sum, acc[D]) partial per query head,
// and the last CTA to finish a slot (atomic ticket) merges the partials.  Each
// key row is read once per step for all G query heads (GQA-aware).  The chunk
// holding row k + step takes the new row from k_new / v_new and also appends
// it to the cache for later steps.
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kWarps = 4;
constexpr int kMaxG = 8;

template <int D>
struct DecodeCfg {
    static constexpr int LPK = D / 8;                          // lanes per key row (16-byte pieces)
    static constexpr int KPI = 32 / LPK;                       // keys per warp instruction
    static constexpr int IT = kDecodeChunk / (kWarps * KPI);   // iterations per warp
};

VLC_DEV void unpack8(const uint4& u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) { f[2 * e] = bf16_lo(w[e]); f[2 * e + 1] = bf16_hi(w[e]); }
}

template <int D, int G>
__global__ void __launch_bounds__(kWarps * 32) decode_kernel(DecodeArgs a) {
    using C = DecodeCfg<D>;
    __shared__ float s_part[kWarps][G][D + 2];
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int part = lane % C::LPK, sub = lane / C::LPK;
    const int total = (int)a.chunk_off[a.slots];
    const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(a.q);

    for (int item = blockIdx.x; item < total; item += gridDim.x) {
        // slot of this item: last s with chunk_off[s] <= item
        int lo = 0, hi = a.slots - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (a.chunk_off[mid] <= item) lo = mid; else hi = mid - 1;
        }
        const int s = lo;
        const int c = item - (int)a.chunk_off[s];
        const int64_t n = a.base_len[s / a.Hkv] + a.step + 1;     // keys this step
        const int64_t new_row = n - 1;
        const int64_t j_begin = (int64_t)c * kDecodeChunk;
        const int64_t j_end = imin(n, j_begin + kDecodeChunk);
        uint4* kc = static_cast<uint4*>(a.k_cache) + a.cache_off[s] * C::LPK;
        uint4* vc = static_cast<uint4*>(a.v_cache) + a.cache_off[s] * C::LPK;
        const uint4* kn = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.k_new) + (int64_t)s * a.kv_stride);
        const uint4* vn = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.v_new) + (int64_t)s * a.kv_stride);

        // ---- all loads of this warp's keys first
        uint4 kr[C::IT], vr[C::IT];
        bool ok[C::IT];
#pragma unroll
        for (int it = 0; it < C::IT; ++it) {
            const int64_t j = j_begin + (int64_t)(warp * C::IT + it) * C::KPI + sub;
            ok[it] = j < j_end;
            if (ok[it] && j == new_row) {
                kr[it] = kn[part];
                vr[it] = vn[part];
                kc[j * C::LPK + part] = kr[it];   // append for later steps
                vc[j * C::LPK + part] = vr[it];
            } else if (ok[it]) {
                kr[it] = kc[j * C::LPK + part];
                vr[it] = vc[j * C::LPK + part];
            } else {
                kr[it] = make_uint4(0, 0, 0, 0);
                vr[it] = make_uint4(0, 0, 0, 0);
            }
        }
        float q[G][8];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float f[8];
            unpack8(*reinterpret_cast<const uint4*>(qb + ((int64_t)s * G + g) * a.q_stride + part * 8), f);
#pragma unroll
            for (int e = 0; e < 8; ++e) q[g][e] = f[e] * a.inv_scale;
        }
        // ---- logits (every lane of a key group holds its key's logit)
        float lg[C::IT][G];
#pragma unroll
        for (int it = 0; it < C::IT; ++it) {
            float kf[8];
            unpack8(kr[it], kf);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float dot = 0.f;
#pragma unroll
                for (int e = 0; e < 8; ++e) dot = fmaf(q[g][e], kf[e], dot);
#pragma unroll
                for (int o = C::LPK / 2; o >= 1; o >>= 1) dot += __shfl_xor_sync(kFull, dot, o);
                lg[it][g] = ok[it] ? dot : -INFINITY;
            }
        }
        // ---- warp-local softmax partial over its keys
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float m = -INFINITY;
#pragma unroll
            for (int it = 0; it < C::IT; ++it) m = fmaxf(m, lg[it][g]);
#pragma unroll
            for (int o = C::LPK; o < 32; o <<= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
            float ssum = 0.f, acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (m != -INFINITY) {
#pragma unroll
                for (int it = 0; it < C::IT; ++it) {
                    const float pj = ex2((lg[it][g] - m) * kLog2e);
                    ssum += pj;
                    float vf[8];
                    unpack8(vr[it], vf);
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[e] = fmaf(pj, vf[e], acc[e]);
                }
            }
#pragma unroll
            for (int o = C::LPK; o < 32; o <<= 1) {
                ssum += __shfl_xor_sync(kFull, ssum, o);
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(kFull, acc[e], o);
            }
            if (lane < C::LPK) {
#pragma unroll
                for (int e = 0; e < 8; ++e) s_part[warp][g][part * 8 + e] = acc[e];
            }
            if (lane == 0) { s_part[warp][g][D] = m; s_part[warp][g][D + 1] = ssum; }
        }
        __syncthreads();
        // ---- chunk partial (combine the warps) -> workspace
        float* ws = a.partials + (int64_t)item * G * (D + 2);
        for (int idx = tid; idx < G * D; idx += kWarps * 32) {
            const int g = idx / D, dim = idx % D;
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_part[w][g][D]);
            float S = 0.f, O = 0.f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const float mw = s_part[w][g][D];
                if (mw == -INFINITY) continue;
                const float f = ex2((mw - M) * kLog2e);
                S = fmaf(s_part[w][g][D + 1], f, S);
                O = fmaf(s_part[w][g][dim], f, O);
            }
            ws[g * (D + 2) + dim] = O;
            if (dim == 0) { ws[g * (D + 2) + D] = M; ws[g * (D + 2) + D + 1] = S; }
        }
        // ---- ticket: the last chunk of the slot merges
        __threadfence();
        __syncthreads();
        const int nchunks = (int)(a.chunk_off[s + 1] - a.chunk_off[s]);
        if (tid == 0) {
            const int prev = atomicAdd(a.tickets + s, 1);
            s_last = (prev == nchunks - 1);
            if (s_last) a.tickets[s] = 0;   // ready for the next step
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            const float* base = a.partials + a.chunk_off[s] * G * (D + 2);
            for (int idx = tid; idx < G * D; idx += kWarps * 32) {
                const int g = idx / D, dim = idx % D;
                float M = -INFINITY;
                for (int cc = 0; cc < nchunks; ++cc) M = fmaxf(M, __ldcg(base + (cc * G + g) * (D + 2) + D));
                float S = 0.f, O = 0.f;
                for (int cc = 0; cc < nchunks; ++cc) {
                    const float* pc = base + (cc * G + g) * (D + 2);
                    const float mc = __ldcg(pc + D);
                    if (mc == -INFINITY) continue;
                    const float f = ex2((mc - M) * kLog2e);
                    S = fmaf(__ldcg(pc + D + 1), f, S);
                    O = fmaf(__ldcg(pc + dim), f, O);
                }
                a.out[((int64_t)s * G + g) * D + dim] = O / S;
            }
        }
        __syncthreads();   // s_part / s_last reuse
    }
}

template <int D>
cudaError_t launch_d(const DecodeArgs& a, cudaStream_t st) {
    const int blocks = (int)imax(1, imin(a.max_items, 148 * 8));
    switch (a.G) {
#define VLC_CASE(g) case g: decode_kernel<D, g><<<blocks, kWarps * 32, 0, st>>>(a); break;
        VLC_CASE(1) VLC_CASE(2) VLC_CASE(3) VLC_CASE(4) VLC_CASE(5) VLC_CASE(6) VLC_CASE(7) VLC_CASE(8)
#undef VLC_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t st) {
    if (a.G < 1 || a.G > kMaxG) return cudaErrorInvalidValue;
    if (a.d == 64) return launch_d<64>(a, st);
    if (a.d == 128) return launch_d<128>(a, st);
    return cudaErrorInvalidValue;
}

}  // namespace vlc
