// seam_f32.cu -- the reference kernel seam's float32 contract on the device.
//
// reference: pkg/src/vlcache/_kernels/_core.pyx:210-242 (stats_tiled) and
// :245-278 (decode_step), with their arithmetic restated operation by
// operation: logits float32(float64 dot * (1/sqrt(d))) from a 16-chain
// float64 dot (_core.pyx:34-62), pass 1 online float32 row max with a float64
// row sum rescaled by exp(double) per key tile (:110-157), pass 2 float32
// exps against the final row max, float64 column mass and the `(double)e < p`
// count (:160-207); decode with 16-chain float32 dots, float64 denominator and
// float32 accumulation in key order (:245-278).
//
// This is the drop-in for vlcache._kernels (numpy-in / numpy-out, one
// (layer, head) per call): float32 operands as the reference takes them, so
// the reference's own tests run unmodified over it.  It is deliberately the
// reference's serial order per row / per key column (one thread each) -- the
// seam is launch-bound by design; the batched bf16 hot path is K1..K5.
#include <cfloat>

#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

// expf as glibc computes it (correctly rounded in practice): the float64 exp
// rounded once to float32
VLC_DEV float expf_ref(float x) { return (float)exp((double)x); }

// fp64 dot with sixteen interleaved accumulators combined as a balanced tree
// (reference _core.pyx:34-62); FMA-contracted like the reference's -O3 build
VLC_DEV double dot16_f64(const float* __restrict__ x, const float* __restrict__ y, int n) {
    double acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = 0.0;
    int t = 0;
    for (; t + 16 <= n; t += 16)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = fma((double)x[t + c], (double)y[t + c], acc[c]);
    for (; t < n; ++t) acc[0] = fma((double)x[t], (double)y[t], acc[0]);
    const double lo = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    const double hi = ((acc[8] + acc[9]) + (acc[10] + acc[11])) + ((acc[12] + acc[13]) + (acc[14] + acc[15]));
    return lo + hi;
}

// same shape in float32 (reference _core.pyx:64-92)
VLC_DEV float dot16_f32(const float* __restrict__ x, const float* __restrict__ y, int n) {
    float acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = 0.f;
    int t = 0;
    for (; t + 16 <= n; t += 16)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = fmaf(x[t + c], y[t + c], acc[c]);
    for (; t < n; ++t) acc[0] = fmaf(x[t], y[t], acc[0]);
    const float lo = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    const float hi = ((acc[8] + acc[9]) + (acc[10] + acc[11])) + ((acc[12] + acc[13]) + (acc[14] + acc[15]));
    return lo + hi;
}

// pass 1: thread = window row r; key tiles of `tile` keys in order
__global__ void seam_pass1(SeamStatsArgs a) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= a.w) return;
    const float* q = a.q + r * a.d;
    const int64_t lim = imin(a.n, a.q_base + r + 1);   // keys [0, lim) visible
    float rmax = -INFINITY;
    double rsum = 0.0;
    for (int64_t k0 = 0; k0 < lim; k0 += a.tile) {
        const int64_t k1 = imin(k0 + a.tile, lim);
        float tmax = -FLT_MAX;
        for (int64_t j = k0; j < k1; ++j) {
            const float l = (float)(dot16_f64(q, a.k + j * a.d, a.d) * a.inv);
            tmax = l > tmax ? l : tmax;
        }
        if (tmax > rmax) {
            rsum *= exp((double)rmax - (double)tmax);
            rmax = tmax;
        }
        double s = 0.0;
        for (int64_t j = k0; j < k1; ++j) {
            const float l = (float)(dot16_f64(q, a.k + j * a.d, a.d) * a.inv);
            s += (double)expf_ref(l - rmax);
        }
        rsum += s;
    }
    a.row_max[r] = rmax;
    a.row_sum[r] = rsum;
}

// pass 2: thread = key j; rows ascending (the reference's column order)
__global__ void seam_pass2(SeamStatsArgs a) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.n) return;
    const float* k = a.k + j * a.d;
    double col = 0.0;
    int64_t below = 0, causal = 0;
    for (int64_t r = imax(0, j - a.q_base); r < a.w; ++r) {   // rows with j <= q_base + r
        const float l = (float)(dot16_f64(a.q + r * a.d, k, a.d) * a.inv);
        const float e = expf_ref(l - a.row_max[r]);
        col += (double)e * (1.0 / a.row_sum[r]);
        below += (double)e < a.p;
        causal += 1;
    }
    a.col_score[j] = col;
    a.below[j] = below;
    if (a.causal) a.causal[j] = causal;
}

// decode: logits (thread per key), then per head one thread for the max and
// the float64 denominator in key order, then thread per output dim
__global__ void seam_logits(SeamDecodeArgs a) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int h = blockIdx.y;
    if (j >= a.n) return;
    a.scratch[(int64_t)h * a.n + j] = dot16_f32(a.q + (int64_t)h * a.d, a.k + j * a.d, a.d) * a.inv;
}

__global__ void seam_softmax(SeamDecodeArgs a) {
    const int h = blockIdx.x;
    float* e = a.scratch + (int64_t)h * a.n;
    __shared__ float smx[256];
    float mx = -FLT_MAX;
    for (int64_t j = threadIdx.x; j < a.n; j += blockDim.x) mx = fmaxf(mx, e[j]);
    smx[threadIdx.x] = mx;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) smx[threadIdx.x] = fmaxf(smx[threadIdx.x], smx[threadIdx.x + w]);
        __syncthreads();
    }
    mx = smx[0];
    for (int64_t j = threadIdx.x; j < a.n; j += blockDim.x) e[j] = expf_ref(e[j] - mx);
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int64_t j = 0; j < a.n; ++j) s += (double)e[j];
        a.denom[h] = s;
    }
}

__global__ void seam_weighted(SeamDecodeArgs a) {
    const int h = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.d) return;
    const float* e = a.scratch + (int64_t)h * a.n;
    const double s = a.denom[h];
    float o = 0.f;
    for (int64_t j = 0; j < a.n; ++j) o = fmaf((float)((double)e[j] / s), a.v[j * a.d + t], o);
    a.out[(int64_t)h * a.d + t] = o;
}

}  // namespace

cudaError_t launch_seam_stats(const SeamStatsArgs& a, cudaStream_t st) {
    seam_pass1<<<(unsigned)((a.w + 127) / 128), 128, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    seam_pass2<<<(unsigned)((a.n + 127) / 128), 128, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_seam_decode(const SeamDecodeArgs& a, cudaStream_t st) {
    seam_logits<<<dim3((unsigned)((a.n + 127) / 128), a.g), 128, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    seam_softmax<<<a.g, 256, 0, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    seam_weighted<<<dim3((unsigned)((a.d + 127) / 128), a.g), 128, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace vlc
