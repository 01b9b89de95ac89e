// budget.cu -- K2: layer-adaptive budget allocation on the device, numpy-exact.
//
// reference: sparsity.py:79 (gamma = below.sum() / causal.sum()),
//            sparsity.py:41-43 (gamma' = gamma.mean(axis=1)),
//            budget.py:107-110 (Z = sum(1 - gamma'); pre = (1 - gamma') / Z * (alpha*L)),
//            budget.py:75 (beta = clip(pre, beta_min, beta_max)),
//            budget.py:70-71 (k = clip(ceil(beta*m), 1, m)).
// numpy reduces contiguous float64 rows with pairwise summation
// (8 strided accumulators for n <= 128, recursive halving above); the same
// association is reproduced here with round-to-nearest intrinsics so that no
// FMA contraction can creep in.  Bit-exact given equal integer counts.
#include "vlc_kernels.h"

namespace vlc {
namespace {

__device__ double pairwise_sum(const double* a, int64_t n, int64_t stride) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i * stride]);
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[(i + j) * stride]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
        return res;
    }
    // numpy halves, rounding the split down to a multiple of the unroll (8)
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    const double left = pairwise_sum(a, n2, stride);
    return __dadd_rn(left, pairwise_sum(a + n2 * stride, n - n2, stride));
}

// One block, one thread per batch element for the per-batch arithmetic, then a
// serial prefix over slots by thread 0.
__global__ void allocate_kernel(BudgetArgs a) {
    const int b = threadIdx.x;
    if (b < a.B && !a.below_head) {
        for (int l = 0; l < a.L; ++l)
            a.gamma_mean[(int64_t)b * a.L + l] = a.gamma_mean_in[(int64_t)b * a.L + l];
    }
    if (b < a.B && a.below_head) {
        const double causal = (double)a.causal_per_head;
        double* g = a.gamma + (int64_t)b * a.L * a.Hq;
        for (int l = 0; l < a.L; ++l) {
            for (int h = 0; h < a.Hq; ++h) {
                const int64_t idx = ((int64_t)b * a.L + l) * a.Hq + h;
                g[(int64_t)l * a.Hq + h] = __ddiv_rn((double)a.below_head[idx], causal);
            }
            a.gamma_mean[(int64_t)b * a.L + l] =
                __ddiv_rn(pairwise_sum(g + (int64_t)l * a.Hq, a.Hq, 1), (double)a.Hq);
        }
    }
    if (b < a.B) {
        double* gm = a.gamma_mean + (int64_t)b * a.L;
        // 1 - gamma' into beta_pre as scratch, then Z by pairwise sum
        double* pre = a.beta_pre + (int64_t)b * a.L;
        for (int l = 0; l < a.L; ++l) pre[l] = __dadd_rn(1.0, -gm[l]);
        const double z = pairwise_sum(pre, a.L, 1);
        a.status[b] = (z == 0.0) ? 1 : 0;
        for (int l = 0; l < a.L; ++l) {
            const double p = __dmul_rn(__ddiv_rn(pre[l], z), a.alpha_times_L);
            pre[l] = p;
            const double be = fmin(fmax(p, a.beta_min), a.beta_max);
            a.beta[(int64_t)b * a.L + l] = be;
            double kc = ceil(__dmul_rn(be, (double)a.prompt_len));
            int64_t k = (z == 0.0) ? 1 : (int64_t)kc;
            if (k < 1) k = 1;
            if (k > a.prompt_len) k = a.prompt_len;
            a.kept_counts[(int64_t)b * a.L + l] = k;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t ko = 0, co = 0;
        const int64_t slots = (int64_t)a.B * a.L * a.Hkv;
        for (int64_t s = 0; s < slots; ++s) {
            const int64_t k = a.kept_counts[s / a.Hkv];
            a.kept_off[s] = ko;
            a.cache_off[s] = co;
            ko += k;
            co += k + a.cache_extra;
        }
        a.kept_off[slots] = ko;
        a.cache_off[slots] = co;
    }
}

}  // namespace

cudaError_t launch_allocate(const BudgetArgs& a, cudaStream_t st) {
    if (a.B > 1024) return cudaErrorInvalidValue;
    const int threads = ((a.B + 31) / 32) * 32;
    allocate_kernel<<<1, threads, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace vlc
