// score_stats.cu -- K1: post-vision attention statistics (reference
// pkg/src/vlcache/_kernels/_core.pyx:110-242 / attention.py:93-132).
//
// CTA = (slot, 128-row block).  Thread t owns window row rb*128 + t; keys are
// streamed 32 per chunk through shared memory.  Logits come from CUDA-core
// FMAs in this first version; the softmax/threshold/column epilogue
// (score_epilogue.cuh) is the one the tcgen05 producer feeds.
#include <cstdlib>

#include "score_epilogue.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kRows = 128;   // window rows per CTA
constexpr int kChunk = 32;   // keys per chunk

template <int D>
__global__ void __launch_bounds__(kRows) score_stats_cc(ScoreArgs a, int nrb) {
    extern __shared__ float4 smem4[];
    float* qT = reinterpret_cast<float*>(smem4);   // [D][kRows]
    float* ks = qT + D * kRows;                    // [kChunk][D]
    __shared__ float colw[kRows / 32][kChunk];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s = blockIdx.y, rb = blockIdx.x;
    const int64_t R = (int64_t)a.G * a.w;
    const int64_t r = (int64_t)rb * kRows + tid;
    const bool row_ok = r < R;
    const int64_t i = row_ok ? r % a.w : 0;
    const int64_t row_end = row_ok ? imin(a.n, a.q_base + i + 1) : 0;   // keys [0, row_end)
    const int64_t r_last = imin(R, (int64_t)rb * kRows + kRows) - 1;
    // the largest window position of any row in this block bounds the keys
    const int64_t i_max = (r_last / a.w == (int64_t)rb * kRows / a.w) ? r_last % a.w : a.w - 1;
    const int64_t blk_end = imin(a.n, a.q_base + i_max + 1);

    const __nv_bfloat16* qg = static_cast<const __nv_bfloat16*>(a.q);
    const __nv_bfloat16* kg = static_cast<const __nv_bfloat16*>(a.k) + (int64_t)s * a.T * a.d;
    for (int idx = tid; idx < kRows * D; idx += kRows) {
        const int row = idx / D, c = idx % D;
        const int64_t rr = (int64_t)rb * kRows + row;
        float v = 0.f;
        if (rr < R && c < a.d) v = __bfloat162float(qg[((int64_t)s * R + rr) * a.d + c]);
        qT[c * kRows + row] = v;
    }

    auto load_chunk = [&](int64_t j0) {
        for (int idx = tid; idx < kChunk * D; idx += kRows) {
            const int j = idx / D, c = idx % D;
            float v = 0.f;
            if (j0 + j < blk_end && c < a.d) v = __bfloat162float(kg[(j0 + j) * a.d + c]);
            ks[j * D + c] = v;
        }
    };
    auto dots = [&](float (&l)[32]) {
#pragma unroll
        for (int c = 0; c < 32; ++c) l[c] = 0.f;
#pragma unroll 2
        for (int k = 0; k < D; k += 4) {
            const float q0 = qT[(k + 0) * kRows + tid], q1 = qT[(k + 1) * kRows + tid];
            const float q2 = qT[(k + 2) * kRows + tid], q3 = qT[(k + 3) * kRows + tid];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const float4 kv = *reinterpret_cast<const float4*>(&ks[c * D + k]);
                l[c] = fmaf(q0, kv.x, l[c]);
                l[c] = fmaf(q1, kv.y, l[c]);
                l[c] = fmaf(q2, kv.z, l[c]);
                l[c] = fmaf(q3, kv.w, l[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) l[c] *= a.inv_scale;
    };

    // ---- pass 1: row max / sum
    RowStats st{-INFINITY, 0.f};
    float l[32];
    for (int64_t j0 = 0; j0 < blk_end; j0 += kChunk) {
        __syncthreads();
        load_chunk(j0);
        __syncthreads();
        dots(l);
        const int valid = (int)imax(0, imin(kChunk, row_end - j0));
        pass1_chunk(l, valid, st);
    }
    const float log2s = row_ok ? __log2f(st.s) : 0.f;

    // ---- pass 2: column mass, below-threshold counts
    int below = 0;
    float* colp = a.col_partial + ((int64_t)s * nrb + rb) * a.n;
    for (int64_t j0 = 0; j0 < blk_end; j0 += kChunk) {
        __syncthreads();
        load_chunk(j0);
        __syncthreads();
        dots(l);
        const int valid = (int)imax(0, imin(kChunk, row_end - j0));
        float e[32];
        const int nb = pass2_chunk(l, valid, st.m, log2s, a.t_star, e);
        below += nb;
        const float csum = transpose_reduce32(e, lane);
        colw[warp][lane] = csum;
        if (a.below_col) {
            int bc[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const float t = l[c] - st.m;
                bc[c] = (c < valid && t < a.t_star) ? 1 : 0;
            }
            const int cnt = transpose_reduce32(bc, lane);
            if (cnt && j0 + lane < a.n) atomicAdd(a.below_col + (int64_t)s * a.n + j0 + lane, cnt);
        }
        __syncthreads();
        if (tid < kChunk && j0 + tid < a.n) {
            float v = 0.f;
#pragma unroll
            for (int wv = 0; wv < kRows / 32; ++wv) v += colw[wv][tid];
            colp[j0 + tid] = v;
        }
    }
    // columns no row of this block can see
    for (int64_t j = ((blk_end + kChunk - 1) / kChunk) * kChunk + tid; j < a.n; j += kRows) colp[j] = 0.f;

    if (row_ok) {
        a.row_max[(int64_t)s * R + r] = st.m;
        a.row_sum[(int64_t)s * R + r] = st.s;
        if (below) atomicAdd(a.below_head + (int64_t)s * a.G + r / a.w, (unsigned long long)below);
    }
}

}  // namespace

int score_row_blocks(int64_t rows) { return (int)((rows + kRows - 1) / kRows); }

cudaError_t launch_score_stats(const ScoreArgs& a, cudaStream_t st) {
    const int nrb = score_row_blocks((int64_t)a.G * a.w);
    cudaError_t e = cudaMemsetAsync(a.below_head, 0, sizeof(unsigned long long) * a.slots * a.G, st);
    if (e != cudaSuccess) return e;
    if (a.below_col) {
        e = cudaMemsetAsync(a.below_col, 0, sizeof(int) * a.slots * a.n, st);
        if (e != cudaSuccess) return e;
    }
    // tcgen05 path (score_stats_tc.cu); the CUDA-core kernel above is kept only
    // as a debugging cross-check behind VLC_K1_CUDA_CORE=1
    static const bool cuda_core = [] {
        const char* v = getenv("VLC_K1_CUDA_CORE");
        return v && v[0] == '1';
    }();
    if (!cuda_core) return launch_score_stats_tc(a, nrb, st);
    dim3 grid(nrb, a.slots);
    if (a.d <= 64) {
        const size_t sm = sizeof(float) * (64 * kRows + kChunk * 64);
        cudaFuncSetAttribute(score_stats_cc<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        score_stats_cc<64><<<grid, kRows, sm, st>>>(a, nrb);
    } else {
        const size_t sm = sizeof(float) * (128 * kRows + kChunk * 128);
        cudaFuncSetAttribute(score_stats_cc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        score_stats_cc<128><<<grid, kRows, sm, st>>>(a, nrb);
    }
    return cudaGetLastError();
}

}  // namespace vlc
