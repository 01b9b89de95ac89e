// eval_rows.cu -- dense causal softmax rows for the analysis / evaluation API
// (SURVEY.md section 8 row f4), over float32 trace rows.
//
// reference: attention.py:72-90 (dense_attention_rows), evaluate.py:78-104
// (oracle_scores: the same rows restricted to the prompt keys), and the
// threshold filter + modality sums of evaluate.py:161-185 / sparsity.py:46-66.
//
// One CTA per (query head, row).  The reference computes
//   l_j = float32(float64 dot(q, k_j) * (1 / sqrt(d)))      (fp32 Q/K widened)
//   e_j = float32 exp(l_j - max_j l_j);  prob_j = double(e_j) / sum_j double(e_j)
// Products of two fp32 values are exact in float64, so the per-thread sequential
// fp64 dot differs from BLAS only in sum rounding (far below a float32 ulp of
// the logit); exp is taken in double and rounded once to float32 (a correctly
// rounded expf).  Logits and then e live in shared memory (key span <= ~55K).
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kRowThreads = 256;

template <typename T, typename Op>
VLC_DEV T block_reduce(T v, T* red, Op op) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = op(v, __shfl_xor_sync(kFull, v, o));
    __syncthreads();   // red[] may still be read by a previous reduction
    if (lane == 0) red[warp] = v;
    __syncthreads();
    T r = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = op(r, red[w]);   // fixed order
    return r;
}

__global__ void __launch_bounds__(kRowThreads) attention_rows_kernel(RowsArgs a) {
    extern __shared__ double rows_smem[];
    double* qs = rows_smem;                               // [d] the query row, widened
    float* lg = reinterpret_cast<float*>(qs + a.d);       // [lim] logits, then e
    __shared__ float redf[32];
    __shared__ double redd[32];
    const int tid = threadIdx.x;
    const int64_t hr = blockIdx.x;                        // head * rows + r
    const int64_t head = hr / a.rows, r = hr % a.rows;
    const float* q = a.q + hr * a.d;
    const float* k = a.k + (head / a.group) * a.key_rows * a.d;
    const int64_t lim = imin(a.key_limit, a.first_row + r + 1);   // visible keys [0, lim)

    for (int i = tid; i < a.d; i += blockDim.x) qs[i] = (double)q[i];
    __syncthreads();
    float mx = -INFINITY;
    for (int64_t j = tid; j < lim; j += blockDim.x) {
        double acc = 0.0;
        if ((a.d & 3) == 0) {
            const float4* kr = reinterpret_cast<const float4*>(k + j * a.d);
            for (int c = 0; c < a.d / 4; ++c) {
                const float4 v = kr[c];
                acc = fma((double)v.x, qs[4 * c], acc);
                acc = fma((double)v.y, qs[4 * c + 1], acc);
                acc = fma((double)v.z, qs[4 * c + 2], acc);
                acc = fma((double)v.w, qs[4 * c + 3], acc);
            }
        } else {
            for (int c = 0; c < a.d; ++c) acc = fma((double)k[j * a.d + c], qs[c], acc);
        }
        const float l = (float)(acc * a.inv_scale);
        lg[j] = l;
        mx = fmaxf(mx, l);
    }
    const float M = block_reduce(mx, redf, [](float x, float y) { return fmaxf(x, y); });
    double s = 0.0;
    for (int64_t j = tid; j < lim; j += blockDim.x) {
        const float e = (float)exp((double)(lg[j] - M));   // float32 difference, as numpy
        lg[j] = e;
        s += (double)e;
    }
    const double S = block_reduce(s, redd, [](double x, double y) { return x + y; });
    __syncthreads();
    if (a.probs) {
        double* out = a.probs + hr * a.out_cols;
        for (int64_t j = tid; j < a.out_cols; j += blockDim.x) out[j] = j < lim ? (double)lg[j] / S : 0.0;
    }
    if (a.mass) {
        // threshold_filter: keep prob >= p * row max; the max is e = 1 at the argmax
        const double cut = a.filter_p * (1.0 / S);
        double vis = 0.0, lang = 0.0;
        const int64_t pend = imin(lim, a.prompt_len);
        for (int64_t j = tid; j < pend; j += blockDim.x) {
            const double pj = (double)lg[j] / S;
            if (pj >= cut) {
                if (j >= a.vis_start && j < a.vis_end) vis += pj;
                else lang += pj;
            }
        }
        const auto add = [](double x, double y) { return x + y; };
        const double V = block_reduce(vis, redd, add);
        const double Lg = block_reduce(lang, redd, add);
        if (tid == 0) {
            a.mass[hr * 3 + 0] = V;
            a.mass[hr * 3 + 1] = Lg;
            a.mass[hr * 3 + 2] = V + Lg;
        }
    }
}

}  // namespace

int64_t attention_rows_smem(int64_t d, int64_t span) { return d * 8 + span * 4; }

cudaError_t launch_attention_rows(const RowsArgs& a, cudaStream_t st) {
    const int64_t span = imin(a.key_limit, a.first_row + a.rows);
    const size_t smem = (size_t)attention_rows_smem(a.d, span);
    cudaError_t e = cudaFuncSetAttribute(attention_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attention_rows_kernel<<<(unsigned)(a.heads * a.rows), kRowThreads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace vlc
